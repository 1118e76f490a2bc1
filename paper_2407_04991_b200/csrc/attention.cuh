// Masked attention over the preallocated KV cache (reference kernels.py:148-233,
// model.py:429-437, 475-478).
//
// Query row t of sequence b attends cache slots [start[b], qbase + t]
// (start = left-pad offset); an empty window produces zeros. Scores are
// (q . k) * (1/sqrt(D)) in f32, softmax with max subtraction, output rounded
// to f16 (model.py:476-477). Cache layout [B, NH, cap, D] per layer (N14).
//
// * attn_decode_kernel — one CTA per (head, sequence), one query row: exact
//   two-pass softmax with every score kept in smem (the reference's order of
//   operations: max, exp, sum, w = e * inv, sum_s w_s v_s), 16-byte K/V loads.
// * attn_prefill_kernel — one CTA per (16 query rows, head, sequence); keys
//   streamed through smem in chunks of 64 with an online (flash-style) softmax.
//   Key chunks are aligned to start[b], so a row's arithmetic does not depend on
//   how much left padding its batch carries (batched == single, bitwise).
#pragma once

#include "common.cuh"

namespace tf {

struct AttnArgs {
  int B, NH, D, cap, T;
  const __half* q;  // [B*T, ldq], head h at columns h*D
  int ldq;
  const __half* kc;  // layer base [B, NH, cap, D]
  const __half* vc;
  const int* start;    // [B] first valid slot (left pad)
  const int* qbase_dev;  // slot of query row t=0
  float scale;
  __half* out;  // [B*T, ldo]
  int ldo;
  // beam search: slot s of row b lives in row (b / beam) * beam + indir[b * cap + s]
  const int* indir;
  int beam;
  // split-KV decode: per (b, h, chunk) partial states + per-(b, h) arrival counters
  float* ws;
  int* cnt;
  int max_chunks;
};

// ------------------------------------------------------------------ decode
// blockDim = kDecThreads. Dynamic smem: (D + cap + max(2 * kDecThreads, kDecWarps * D)) floats.
constexpr int kDecThreads = 256;
constexpr int kDecWarps = kDecThreads / 32;
__global__ void __launch_bounds__(256, 3) attn_decode_kernel(const AttnArgs a) {
  extern __shared__ float sm[];
  pdl_wait();
  pdl_trigger();
  const int h = blockIdx.x, b = blockIdx.y;
  const int D = a.D;
  float* qs = sm;               // [D]
  float* sc = sm + D;           // [cap] scores / weights
  float* red = sc + a.cap;      // [2 * kDecThreads] partial outputs / reduction scratch
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b], hi = qbase;  // inclusive window [lo, hi]
  const int n = hi - lo + 1;
  const __half* qrow = a.q + (size_t)b * a.ldq + (size_t)h * D;  // T == 1
  for (int d = tid; d < D; d += kDecThreads) qs[d] = __half2float(qrow[d]);
  __syncthreads();
  __half* orow = a.out + (size_t)b * a.ldo + (size_t)h * D;
  if (n <= 0) {
    for (int d = tid; d < D; d += kDecThreads) orow[d] = __float2half_rn(0.0f);
    return;
  }
  const size_t head_stride = (size_t)a.cap * D;        // one (row, head) block
  const size_t row_stride = (size_t)a.NH * head_stride;  // one batch row
  const int* ind = a.indir ? a.indir + (size_t)b * a.cap : nullptr;
  const int beam0 = a.indir ? (b / a.beam) * a.beam : b;
  // K/V row of slot s (through the beam indirection when present)
  auto kv_off = [&](int s) -> size_t {
    const int src = ind ? beam0 + ind[s] : b;
    return (size_t)src * row_stride + (size_t)h * head_stride + (size_t)s * D;
  };
  const __half* K = a.kc;
  const __half* V = a.vc;

  // ---- scores
  if ((D & 7) == 0 && D <= 256) {
    const int G = D >> 3;                 // lanes per key (16 B each)
    const int kpw = 32 / G > 0 ? 32 / G : 1;  // keys per warp load
    const int sub = lane / G, gl = lane - sub * G;
    // 8 loads in flight per lane: each warp covers 8 * kpw keys per round
    for (int base = warp * 8 * kpw; base < n; base += 64 * kpw) {
      uint4 raw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = base + u * kpw + sub;
        raw[u] = (sub < kpw && j < n) ? *reinterpret_cast<const uint4*>(K + kv_off(lo + j) + gl * 8)
                                      : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = base + u * kpw + sub;
        float acc = 0.0f;
        const __half2* kh = reinterpret_cast<const __half2*>(&raw[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = __half22float2(kh[e]);
          acc = __fadd_rn(acc, __fmul_rn(qs[gl * 8 + 2 * e], kf.x));
          acc = __fadd_rn(acc, __fmul_rn(qs[gl * 8 + 2 * e + 1], kf.y));
        }
        for (int o = G >> 1; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        if (sub < kpw && gl == 0 && j < n) sc[j] = __fmul_rn(acc, a.scale);
      }
    }
  } else {
    for (int j = tid; j < n; j += kDecThreads) {
      const __half* kr = K + kv_off(lo + j);
      float acc = 0.0f;
      for (int d = 0; d < D; ++d) acc = __fadd_rn(acc, __fmul_rn(qs[d], __half2float(kr[d])));
      sc[j] = __fmul_rn(acc, a.scale);
    }
  }
  __syncthreads();
  // ---- max, exp, sum
  float m = -INFINITY;
  for (int j = tid; j < n; j += kDecThreads) m = fmaxf(m, sc[j]);
  m = warp_max(m);
  if (lane == 0) red[warp] = m;
  __syncthreads();
  m = red[0];
  for (int w = 1; w < kDecWarps; ++w) m = fmaxf(m, red[w]);
  __syncthreads();
  float z = 0.0f;
  for (int j = tid; j < n; j += kDecThreads) {
    const float e = expf(__fsub_rn(sc[j], m));
    sc[j] = e;
    z += e;
  }
  z = warp_sum(z);
  if (lane == 0) red[warp] = z;
  __syncthreads();
  z = 0.0f;
  for (int w = 0; w < kDecWarps; ++w) z += red[w];
  const float inv = __fdiv_rn(1.0f, z);
  __syncthreads();
  // ---- weighted sum of V
  if ((D & 7) == 0 && D <= 256) {
    // G lanes per value row (8 dims each, 16-byte loads), kpw rows per warp
    // load, 8 loads in flight; sub-groups and warps combined in a fixed order
    const int G = D >> 3;
    const int kpw = 32 / G > 0 ? 32 / G : 1;
    const int sub = lane / G, gl = lane - sub * G;
    float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    for (int base = warp * 8 * kpw; base < n; base += 8 * kpw * kDecWarps) {
      uint4 raw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = base + u * kpw + sub;
        raw[u] = (sub < kpw && j < n) ? *reinterpret_cast<const uint4*>(V + kv_off(lo + j) + gl * 8)
                                      : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int j = base + u * kpw + sub;
        if (sub < kpw && j < n) {
          const float w = __fmul_rn(sc[j], inv);
          float vf[8];
          unpack8(raw[u], vf);
#pragma unroll
          for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(o[e], __fmul_rn(w, vf[e]));
        }
      }
    }
    // sub-groups of this warp (lanes gl, gl + G, ...)
    for (int off = G; off < 32; off <<= 1)
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], off));
    if (sub == 0)
#pragma unroll
      for (int e = 0; e < 8; ++e) red[warp * D + gl * 8 + e] = o[e];
    __syncthreads();
    for (int d = tid; d < D; d += kDecThreads) {
      float v = 0.0f;
      for (int w = 0; w < kDecWarps; ++w) v = __fadd_rn(v, red[w * D + d]);
      orow[d] = f16_sat(v);
    }
    return;
  }
  // generic head_dim: threads = (dim pair, key group)
  const int DP = (D + 1) >> 1;  // dim pairs
  const int groups = kDecThreads / DP > 0 ? kDecThreads / DP : 1;
  const int g = tid / DP, dp = tid - g * DP;
  float o0 = 0.0f, o1 = 0.0f;
  if (g < groups) {
    const int d0 = 2 * dp;
    for (int j = g; j < n; j += groups) {
      const float w = __fmul_rn(sc[j], inv);
      o0 = __fadd_rn(o0, __fmul_rn(w, __half2float(V[kv_off(lo + j) + d0])));
      if (d0 + 1 < D) o1 = __fadd_rn(o1, __fmul_rn(w, __half2float(V[kv_off(lo + j) + d0 + 1])));
    }
  }
  if (g < groups) {
    red[g * 2 * DP + 2 * dp] = o0;
    red[g * 2 * DP + 2 * dp + 1] = o1;
  }
  __syncthreads();
  for (int d = tid; d < D; d += kDecThreads) {
    float v = 0.0f;
    for (int gg = 0; gg < groups; ++gg) v = __fadd_rn(v, red[gg * 2 * DP + d]);
    orow[d] = f16_sat(v);
  }
}

// ------------------------------------------------------------------ split-KV decode
// grid (max_chunks, NH, B), 128 threads; chunk c covers window slots
// [lo + 64c, lo + 64c + 64) (aligned to the row's first valid slot). Each CTA
// writes its partial softmax state (max m, sum z, unnormalised o[64]); the last
// chunk of a (b, h) to finish merges them in chunk order (deterministic).
constexpr int kSplitKeys = 64;
constexpr int kSplitThreads = 128;

__global__ void __launch_bounds__(kSplitThreads) attn_decode_split_kernel(const AttnArgs a) {
  __shared__ float qs[64], sc[kSplitKeys], red[4 * 64 + 8];
  __shared__ int s_last;
  pdl_wait();
  pdl_trigger();
  constexpr int D = 64;
  const int c = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b], hi = qbase;  // window [lo, hi]
  const int n = hi - lo + 1;
  const int nch = n > 0 ? (n + kSplitKeys - 1) / kSplitKeys : 0;
  if (c >= nch && !(n <= 0 && c == 0)) return;
  __half* orow = a.out + (size_t)b * a.ldo + (size_t)h * D;
  if (n <= 0) {  // empty window: zeros
    if (tid < D) orow[tid] = __float2half_rn(0.0f);
    return;
  }
  const size_t row_stride = (size_t)a.NH * a.cap * D, head_stride = (size_t)a.cap * D;
  const int* ind = a.indir ? a.indir + (size_t)b * a.cap : nullptr;
  const int beam0 = a.indir ? (b / a.beam) * a.beam : b;
  auto kv_off = [&](int s) -> size_t {
    const int src = ind ? beam0 + ind[s] : b;
    return (size_t)src * row_stride + (size_t)h * head_stride + (size_t)s * D;
  };
  if (tid < D) qs[tid] = __half2float(a.q[(size_t)b * a.ldq + (size_t)h * D + tid]);
  const int j0 = c * kSplitKeys, cnt_keys = min(kSplitKeys, n - j0);
  const int sub = lane >> 3, gl = lane & 7;
  // K rows: 4 warps x 4 rows per load x 4 loads in flight = 64 keys
  uint4 kr[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = warp * 16 + u * 4 + sub;
    kr[u] = j < cnt_keys ? *reinterpret_cast<const uint4*>(a.kc + kv_off(lo + j0 + j) + gl * 8)
                         : make_uint4(0, 0, 0, 0);
  }
  // V rows issued now too (independent of the scores)
  uint4 vr[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = warp * 16 + u * 4 + sub;
    vr[u] = j < cnt_keys ? *reinterpret_cast<const uint4*>(a.vc + kv_off(lo + j0 + j) + gl * 8)
                         : make_uint4(0, 0, 0, 0);
  }
  __syncthreads();  // qs
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = warp * 16 + u * 4 + sub;
    float kf[8], acc = 0.0f;
    unpack8(kr[u], kf);
#pragma unroll
    for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, __fmul_rn(qs[gl * 8 + e], kf[e]));
    acc += __shfl_xor_sync(0xffffffffu, acc, 4);
    acc += __shfl_xor_sync(0xffffffffu, acc, 2);
    acc += __shfl_xor_sync(0xffffffffu, acc, 1);
    if (gl == 0 && j < cnt_keys) sc[j] = __fmul_rn(acc, a.scale);
  }
  __syncthreads();
  // chunk max / exp / sum (64 scores: 2 per lane of warp 0.. handled by all)
  float m = -INFINITY;
  for (int j = tid; j < cnt_keys; j += kSplitThreads) m = fmaxf(m, sc[j]);
  m = warp_max(m);
  if (lane == 0) red[4 * 64 + warp] = m;
  __syncthreads();
  m = fmaxf(fmaxf(red[256], red[257]), fmaxf(red[258], red[259]));
  float z = 0.0f;
  __syncthreads();
  for (int j = tid; j < cnt_keys; j += kSplitThreads) {
    const float e = expf(__fsub_rn(sc[j], m));
    sc[j] = e;
    z += e;
  }
  z = warp_sum(z);
  if (lane == 0) red[4 * 64 + 4 + warp] = z;
  __syncthreads();
  z = (red[260] + red[261]) + (red[262] + red[263]);
  // unnormalised o = sum_j e_j v_j
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int j = warp * 16 + u * 4 + sub;
    if (j < cnt_keys) {
      float vf[8];
      unpack8(vr[u], vf);
      const float w = sc[j];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(o[e], __fmul_rn(w, vf[e]));
    }
  }
#pragma unroll
  for (int e = 0; e < 8; ++e) {
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 8));
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 16));
  }
  if (sub == 0)
#pragma unroll
    for (int e = 0; e < 8; ++e) red[warp * 64 + gl * 8 + e] = o[e];
  __syncthreads();
  // partial state [b][h][chunk] = {m, z, o[64]}
  float* part = a.ws + (((size_t)b * a.NH + h) * a.max_chunks) * 66;
  if (tid < D) {
    const float ov = __fadd_rn(__fadd_rn(red[tid], red[64 + tid]), __fadd_rn(red[128 + tid], red[192 + tid]));
    if (nch == 1) {
      orow[tid] = f16_sat(__fdiv_rn(ov, z));
      return;
    }
    __stcg(part + (size_t)c * 66 + 2 + tid, ov);
    if (tid == 0) {
      __stcg(part + (size_t)c * 66, m);
      __stcg(part + (size_t)c * 66 + 1, z);
    }
  }
  if (nch == 1) return;
  __threadfence();
  __syncthreads();
  if (tid == 0) {
    const int prev = atomicAdd(a.cnt + (size_t)b * a.NH + h, 1);
    s_last = (prev == nch - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // merge in chunk order: M = max m_c, Z = sum z_c e^(m_c - M), O = sum o_c e^(m_c - M)
  if (tid < D) {
    float M = -INFINITY;
    for (int cc = 0; cc < nch; ++cc) M = fmaxf(M, __ldcg(part + (size_t)cc * 66));
    float Z = 0.0f, O = 0.0f;
    for (int cc = 0; cc < nch; ++cc) {
      const float f = expf(__fsub_rn(__ldcg(part + (size_t)cc * 66), M));
      Z = __fadd_rn(Z, __fmul_rn(__ldcg(part + (size_t)cc * 66 + 1), f));
      O = __fadd_rn(O, __fmul_rn(__ldcg(part + (size_t)cc * 66 + 2 + tid), f));
    }
    orow[tid] = f16_sat(__fdiv_rn(O, Z));
  }
  if (tid == 0) a.cnt[(size_t)b * a.NH + h] = 0;  // ready for the next launch / replay
}

// ------------------------------------------------------------------ prefill
// blockDim = 128 (4 warps x 4 query rows). Dynamic smem: 16 * D floats (q rows)
// + 2 * 64 * (D + 1) halves (K/V chunk).
constexpr int kPfRows = 16;
constexpr int kPfKeys = 64;

__global__ void __launch_bounds__(128) attn_prefill_kernel(const AttnArgs a) {
  extern __shared__ float sm[];
  pdl_wait();
  pdl_trigger();
  const int qblk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int D = a.D;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  float* qs = sm;                                             // [16][D]
  const int KS = D + 1;  // odd row pitch (halves): lanes reading different keys hit different banks
  __half* ks = reinterpret_cast<__half*>(qs + kPfRows * D);   // [64][KS]
  __half* vs = ks + kPfKeys * KS;                             // [64][KS]
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b];
  const int t0 = qblk * kPfRows;
  const int rows = min(kPfRows, a.T - t0);
  for (int i = tid; i < kPfRows * D; i += 128) {
    const int r = i / D, d = i - r * D;
    qs[i] = (r < rows) ? __half2float(a.q[(size_t)(b * a.T + t0 + r) * a.ldq + h * D + d]) : 0.0f;
  }
  const size_t head_off = ((size_t)b * a.NH + h) * a.cap * D;
  const __half* K = a.kc + head_off;
  const __half* V = a.vc + head_off;
  // per-warp rows r = warp*4 + i; per-lane output dims d = lane + 32*k
  constexpr int MAXDL = 4;  // D <= 128
  float mrow[4], lrow[4], o[4][MAXDL];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    mrow[i] = -INFINITY;
    lrow[i] = 0.0f;
#pragma unroll
    for (int k = 0; k < MAXDL; ++k) o[i][k] = 0.0f;
  }
  const int hi_blk = qbase + t0 + rows - 1;  // last slot any row of this block sees
  for (int c0 = lo; c0 <= hi_blk; c0 += kPfKeys) {
    const int nk = min(kPfKeys, hi_blk - c0 + 1);
    __syncthreads();
    for (int i = tid; i < nk * D; i += 128) {
      const int j = i / D, d = i - j * D;
      ks[j * KS + d] = K[(size_t)c0 * D + i];
      vs[j * KS + d] = V[(size_t)c0 * D + i];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int r = warp * 4 + i;
      if (r >= rows) continue;
      const int hi = qbase + t0 + r;  // inclusive
      const float* qr = qs + r * D;
      float s[2];
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int j = lane + 32 * u;
        const int slot = c0 + j;
        float acc = -INFINITY;
        if (j < nk && slot <= hi) {
          acc = 0.0f;
          const __half* kr = ks + j * KS;
          for (int d = 0; d < D; ++d) acc = __fadd_rn(acc, __fmul_rn(qr[d], __half2float(kr[d])));
          acc = __fmul_rn(acc, a.scale);
        }
        s[u] = acc;
      }
      const float cmax = warp_max(fmaxf(s[0], s[1]));
      if (cmax == -INFINITY) continue;  // no visible key in this chunk
      const float mnew = fmaxf(mrow[i], cmax);
      const float alpha = (mrow[i] == -INFINITY) ? 0.0f : expf(mrow[i] - mnew);
      float p0 = (s[0] == -INFINITY) ? 0.0f : expf(s[0] - mnew);
      float p1 = (s[1] == -INFINITY) ? 0.0f : expf(s[1] - mnew);
      lrow[i] = lrow[i] * alpha + warp_sum(p0 + p1);
      mrow[i] = mnew;
#pragma unroll
      for (int k = 0; k < MAXDL; ++k) o[i][k] *= alpha;
      for (int j = 0; j < nk; ++j) {
        const float pj = __shfl_sync(0xffffffffu, j < 32 ? p0 : p1, j & 31);
        if (pj == 0.0f) continue;
        const __half* vr = vs + j * KS;
#pragma unroll
        for (int k = 0; k < MAXDL; ++k) {
          const int d = lane + 32 * k;
          if (d < D) o[i][k] += pj * __half2float(vr[d]);
        }
      }
    }
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = warp * 4 + i;
    if (r >= rows) continue;
    __half* orow = a.out + (size_t)(b * a.T + t0 + r) * a.ldo + h * D;
    const float inv = lrow[i] > 0.0f ? 1.0f / lrow[i] : 0.0f;
#pragma unroll
    for (int k = 0; k < MAXDL; ++k) {
      const int d = lane + 32 * k;
      if (d < D) orow[d] = f16_sat(o[i][k] * inv);
    }
  }
}

}  // namespace tf
