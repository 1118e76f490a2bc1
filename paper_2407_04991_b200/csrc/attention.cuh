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
};

// ------------------------------------------------------------------ decode
// blockDim = kDecThreads. Dynamic smem: (D + cap + 2 * kDecThreads) floats.
constexpr int kDecThreads = 256;
constexpr int kDecWarps = kDecThreads / 32;
__global__ void __launch_bounds__(256) attn_decode_kernel(const AttnArgs a) {
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
  // ---- weighted sum of V: threads = (dim pair, key group)
  const int DP = (D + 1) >> 1;  // dim pairs
  const int groups = kDecThreads / DP > 0 ? kDecThreads / DP : 1;
  const int g = tid / DP, dp = tid - g * DP;
  float o0 = 0.0f, o1 = 0.0f;
  if (g < groups) {
    const int d0 = 2 * dp;
    if ((D & 1) == 0) {
      for (int j0 = g; j0 < n; j0 += 4 * groups) {
        __half2 vr[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * groups;
          vr[u] = j < n ? *reinterpret_cast<const __half2*>(V + kv_off(lo + j) + d0) : __floats2half2_rn(0.f, 0.f);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * groups;
          if (j < n) {
            const float w = __fmul_rn(sc[j], inv);
            const float2 vf = __half22float2(vr[u]);
            o0 = __fadd_rn(o0, __fmul_rn(w, vf.x));
            o1 = __fadd_rn(o1, __fmul_rn(w, vf.y));
          }
        }
      }
    } else {
      for (int j = g; j < n; j += groups) {
        const float w = __fmul_rn(sc[j], inv);
        o0 = __fadd_rn(o0, __fmul_rn(w, __half2float(V[kv_off(lo + j) + d0])));
        if (d0 + 1 < D) o1 = __fadd_rn(o1, __fmul_rn(w, __half2float(V[kv_off(lo + j) + d0 + 1])));
      }
    }
  }
  // partials land in red[g][2*DP]; thread d sums the groups in a fixed order
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
