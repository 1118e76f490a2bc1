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
  int group;  // decode prefetch kernel: 64-slot chunks per CTA
  int trace;  // diagnostics slot (0 = off)
  // decode prefetch kernel: the next layer's caches (same layout); each CTA
  // streams its own window of them HBM -> L2 (null = off)
  const __half* pf_kc;
  const __half* pf_vc;
  const uint8_t* plan;  // beam: per-request plans (kBeamPlanBytes each) from the select, or null
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
// release/acquire ordering for the last-arriver merges (cheaper than the
// sequentially consistent fence __threadfence() emits)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}

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
  // vector path: G = D / 8 lanes per key must be a power of two (the xor
  // reductions below pair lanes inside aligned groups of G)
  const bool vec = (D & 7) == 0 && D <= 256 && (((D >> 3) & ((D >> 3) - 1)) == 0);
  if (vec) {
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
  if (vec) {
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

// ------------------------------------------------------------------ decode, prefetching
// head_dim 64. CTA (g, h, b) owns chunks [g*G, g*G+G) of the 64-slot chunks of
// row b's window [start_b, len] (aligned to start_b, as in the split kernel).
// Every slot but the newest (slot len, written by the QKV GEMM this step) is
// already in the cache, so the CTA copies its chunks' K/V into shared memory
// with cp.async BEFORE griddepcontrol.wait: the KV stream overlaps the QKV GEMM
// instead of following it. After the wait it loads only q and the newest slot.
// Per-chunk arithmetic and the fixed-order merge are those of
// attn_decode_split_kernel, so the result does not depend on G (a function of
// the session capacity) or on the batch. When one CTA owns the whole window
// the merge is local; otherwise partials go to the workspace and the
// last-arriving CTA merges them.
constexpr int kPfKeysPerChunk = 64, kPfChunkBytes = 2 * 64 * 64 * 2;  // K + V, f16
constexpr int kPfMaxG = 8;  // chunks per CTA at most
__host__ __device__ inline size_t attn_pf_smem_bytes(int G) {
  return (size_t)G * kPfChunkBytes + (size_t)G * (66 + 64) * sizeof(float);
}
// 128 threads (4 CTAs per SM: a batch-32 step is one wave)

template <int kPfThreads>
__global__ void __launch_bounds__(kPfThreads, 1) attn_decode_pf_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t pf_smem[];
  __shared__ __align__(16) float qs[64];
  __shared__ float sc_all[kPfMaxG * 64];
  __shared__ float ew_all[kPfMaxG * 64];
  __shared__ int s_last;
  constexpr int D = 64;
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(a.trace, 0);
  const int G = a.group;
  __half* kvs = reinterpret_cast<__half*>(pf_smem);                           // [G][K|V][64][64]
  float* part_s = reinterpret_cast<float*>(pf_smem + (size_t)G * kPfChunkBytes);  // [G][66]
  float* part_h = part_s + (size_t)G * 66;  // [G][64]: second key half of each chunk's PV
  const int g = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  // the cache length and left pad were written by earlier steps (complete)
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b], hi = qbase;  // window [lo, hi]
  const int n = hi - lo + 1;
  const int nch = n > 0 ? (n + 63) / 64 : 0;
  const int ngr = (nch + G - 1) / G;
  if (g >= (ngr > 0 ? ngr : 1)) {
    pdl_trigger();
    return;
  }
  const int c0 = g * G, nc = n > 0 ? min(G, nch - c0) : 0;
  const size_t row_stride = (size_t)a.NH * a.cap * D, head_stride = (size_t)a.cap * D;
  const int* ind = a.indir ? a.indir + (size_t)b * a.cap : nullptr;
  const int beam0 = a.indir ? (b / a.beam) * a.beam : b;
  // beam: this CTA's slice of the indirection row staged in smem once (one
  // coalesced load instead of a dependent global load per copied segment)
  __shared__ int s_ind[kPfMaxG * 64];
  const int slot0 = lo + c0 * 64;
  if (ind != nullptr) {
    for (int i = tid; i < nc * 64; i += kPfThreads) s_ind[i] = slot0 + i < hi ? ind[slot0 + i] : 0;
    __syncthreads();
  }
  auto kv_off = [&](int s) -> size_t {
    const int src = ind ? beam0 + (s - slot0 < nc * 64 && s >= slot0 && s < hi ? s_ind[s - slot0] : ind[s]) : b;
    return (size_t)src * row_stride + (size_t)h * head_stride + (size_t)s * D;
  };
  // ---- before the wait: K/V of every slot < hi in this CTA's chunks
  for (int seg = tid; seg < nc * 64 * 8; seg += kPfThreads) {
    const int i = seg >> 9, j = (seg >> 3) & 63, part = seg & 7;
    const int slot = lo + (c0 + i) * 64 + j;
    if (slot != hi) {  // slots past the window are zero-filled (src-size 0)
      const bool ok = slot < hi;
      const size_t off = ok ? kv_off(slot) + part * 8 : 0;
      // K rows are stored with their 16-byte segments rotated by the row index
      // (segment g of row j at position (g + j) & 7): the QK^T loop then reads
      // logical segment g of 8 consecutive rows from 8 distinct bank groups
      // while indexing q with the compile-time g
      __half* kd = kvs + ((size_t)(2 * i) * 64 + j) * 64 + ((part + j) & 7) * 8;
      __half* vd = kvs + ((size_t)(2 * i + 1) * 64 + j) * 64 + part * 8;
      cp_async16(smem_u32(kd), a.kc + off, ok);
      cp_async16(smem_u32(vd), a.vc + off, ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (a.pf_kc != nullptr && ind == nullptr && tid < 2 && nc > 0) {
    // next layer's copy of this CTA's window (contiguous slots of one (b, h))
    const int s0 = lo + c0 * 64, s1 = min(lo + (c0 + nc) * 64, hi + 1);
    const size_t off = kv_off(s0);
    l2_prefetch_bulk((tid == 0 ? a.pf_kc : a.pf_vc) + off, (uint32_t)((s1 - s0) * D * 2));
  }
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) tr.mark(a.trace, 1);
  __half* orow = a.out + (size_t)b * a.ldo + (size_t)h * D;
  if (n <= 0) {  // empty window: zeros
    if (tid < D) orow[tid] = __float2half_rn(0.0f);
    return;
  }
  // ---- after the wait: q and the newest slot
  if (tid < D) qs[tid] = __half2float(a.q[(size_t)b * a.ldq + (size_t)h * D + tid]);
  {
    const int i = (hi - lo) / 64 - c0, j = (hi - lo) % 64;
    if (i >= 0 && i < nc && tid < 16) {
      const int part = tid & 7;
      const size_t off = kv_off(hi) + part * 8;
      const __half* src = (tid < 8 ? a.kc : a.vc) + off;
      __half* dst = kvs + ((size_t)(2 * i + (tid < 8 ? 0 : 1)) * 64 + j) * 64 + (tid < 8 ? ((part + j) & 7) : part) * 8;
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>(src);
    }
  }
  cp_async_commit_wait_all();
  __syncthreads();
  if (threadIdx.x == 0) tr.mark(a.trace, 2);
  const long long clk0 = clock64();
  // scores: one thread per key. Thread reads its K row in 16-B segments in
  // the order (s + key) & 7, so the 8 threads of each LDS.128 phase hit
  // distinct bank groups; 8 independent partial dot products, summed in that
  // order (fixed by the key's position in its chunk -> batch-invariant)
  const int n_keys = min(nc * 64, n - c0 * 64);
  // q in registers (logical segment g = dims 8g .. 8g+7); per key 8 partial dot
  // products (one per segment, fixed order within), summed as a fixed tree
  float qr[64];
#pragma unroll
  for (int e = 0; e < 64; e += 4) {
    const float4 q4 = *reinterpret_cast<const float4*>(qs + e);
    qr[e] = q4.x;
    qr[e + 1] = q4.y;
    qr[e + 2] = q4.z;
    qr[e + 3] = q4.w;
  }
  for (int key = tid; key < n_keys; key += kPfThreads) {
    const int i = key >> 6, j = key & 63;
    const __half* kr = kvs + ((size_t)(2 * i) * 64 + j) * 64;
    uint4 raw[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) raw[g] = *reinterpret_cast<const uint4*>(kr + ((g + j) & 7) * 8);
    float ps[8];
#pragma unroll
    for (int g = 0; g < 8; ++g) {
      float kf[8];
      unpack8(raw[g], kf);
      float acc = __fmul_rn(qr[8 * g], kf[0]);
#pragma unroll
      for (int e = 1; e < 8; ++e) acc = __fmaf_rn(qr[8 * g + e], kf[e], acc);
      ps[g] = acc;
    }
    const float d = __fadd_rn(__fadd_rn(__fadd_rn(ps[0], ps[1]), __fadd_rn(ps[2], ps[3])),
                              __fadd_rn(__fadd_rn(ps[4], ps[5]), __fadd_rn(ps[6], ps[7])));
    sc_all[key] = __fmul_rn(d, a.scale);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    tr.mark(a.trace, 4);
    if (a.trace > 0) tr.t[6] = (unsigned long long)(clock64() - clk0);
  }
  // WPC warps per chunk (1 with 128 threads; 2 with 256: key halves 0-31 and
  // 32-63). Each warp computes the chunk max / exp / sum over all 64 keys (the
  // same values in every warp of the chunk), writes the weights of its keys, and
  // o = sum_j e_j v_j over its 64/WPC keys with each lane owning dims (2 lane,
  // 2 lane + 1), 4 accumulators (keys j % 4) combined pairwise; key halves are
  // added in order before the merge
  constexpr int WPC = kPfThreads >= 256 ? 2 : 1, KPW = 64 / WPC;
  for (int wi = warp; wi < WPC * nc; wi += kPfThreads / 32) {
    const int i = wi / WPC, hf = wi % WPC;
    const int cnt_keys = min(64, n - (c0 + i) * 64);
    const float* sci = sc_all + i * 64;
    const float s0 = lane < cnt_keys ? sci[lane] : -INFINITY;
    const float s1 = lane + 32 < cnt_keys ? sci[lane + 32] : -INFINITY;
    const float m = warp_max(fmaxf(s0, s1));
    const float e0 = lane < cnt_keys ? expf(__fsub_rn(s0, m)) : 0.0f;
    const float e1 = lane + 32 < cnt_keys ? expf(__fsub_rn(s1, m)) : 0.0f;
    const float z = warp_sum(__fadd_rn(e0, e1));
    // weights go to their own array: another warp of the chunk may still be
    // reading the scores
    float* wts = ew_all + i * 64;
    if (WPC == 1 || hf == 0) wts[lane] = e0;
    if (WPC == 1 || hf == 1) wts[lane + 32] = e1;
    __syncwarp();
    const __half* Vs = kvs + (size_t)(2 * i + 1) * 64 * 64 + (size_t)hf * KPW * 64;
    const float* w0 = wts + hf * KPW;
    float o0[4] = {0.f, 0.f, 0.f, 0.f}, o1[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 4
    for (int j = 0; j < KPW; j += 4) {
#pragma unroll
      for (int r = 0; r < 4; ++r) {
        const float2 v = __half22float2(*reinterpret_cast<const __half2*>(Vs + (j + r) * 64 + 2 * lane));
        const float w = w0[j + r];
        o0[r] = __fmaf_rn(w, v.x, o0[r]);
        o1[r] = __fmaf_rn(w, v.y, o1[r]);
      }
    }
    float* dst = hf ? part_h + i * 64 : part_s + i * 66 + 2;
    dst[2 * lane] = __fadd_rn(__fadd_rn(o0[0], o0[1]), __fadd_rn(o0[2], o0[3]));
    dst[2 * lane + 1] = __fadd_rn(__fadd_rn(o1[0], o1[1]), __fadd_rn(o1[2], o1[3]));
    if (lane == 0 && hf == 0) {
      part_s[i * 66] = m;
      part_s[i * 66 + 1] = z;
    }
  }
  __syncthreads();
  if constexpr (WPC == 2) {
    for (int e = tid; e < nc * 64; e += kPfThreads) {
      const int i = e >> 6, d = e & 63;
      part_s[i * 66 + 2 + d] = __fadd_rn(part_s[i * 66 + 2 + d], part_h[i * 64 + d]);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) tr.mark(a.trace, 5);
  if (threadIdx.x == 0) tr.mark(a.trace, 3);
  // merge in chunk order: M = max m_c, Z = sum z_c e^(m_c - M), O = sum o_c e^(m_c - M)
  auto merge = [&](const float* P, int count) {
    if (tid < D) {
      float M = -INFINITY;
      for (int cc = 0; cc < count; ++cc) M = fmaxf(M, P[(size_t)cc * 66]);
      float Z = 0.0f, O = 0.0f;
      for (int cc = 0; cc < count; ++cc) {
        const float f = expf(__fsub_rn(P[(size_t)cc * 66], M));
        Z = __fadd_rn(Z, __fmul_rn(P[(size_t)cc * 66 + 1], f));
        O = __fadd_rn(O, __fmul_rn(P[(size_t)cc * 66 + 2 + tid], f));
      }
      orow[tid] = f16_sat(__fdiv_rn(O, Z));
    }
  };
  if (ngr == 1) {
    merge(part_s, nch);
  } else {
    float* part = a.ws + (((size_t)b * a.NH + h) * a.max_chunks) * 66;
    for (int e = tid; e < nc * 66; e += kPfThreads) __stcg(part + (size_t)c0 * 66 + e, part_s[e]);
    fence_acq_rel_gpu();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(a.cnt + (size_t)b * a.NH + h, 1);
      s_last = (prev == ngr - 1);
    }
    __syncthreads();
    if (s_last) {
      fence_acq_rel_gpu();
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
      if (tid == 0) a.cnt[(size_t)b * a.NH + h] = 0;
    }
  }
  if (threadIdx.x == 0) {
    tr.mark(a.trace, 7);
    tr.flush(a.trace);
  }
}

// ------------------------------------------------------------------ mma.sync helpers
// ldmatrix / m16n8k16 (f16 in, f32 accumulate) for the decode attention kernels,
// whose per-row tiles (one query row, or the R beams of a request) are far below
// the 64-128-row minimum of a tcgen05 MMA.

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void ldsm_x2_t(uint32_t addr, uint32_t& r0, uint32_t& r1) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x2.trans.shared.b16 {%0,%1}, [%2];" : "=r"(r0), "=r"(r1) : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_h2(float x, float y) {
  __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<uint32_t*>(&h);
}


// ------------------------------------------------------------------ decode, beam groups (tensor cores)
// head_dim 64, beam search. One CTA (4 warps) per (head, request) over the whole
// window. The window's 64-slot chunks (aligned to the request's first valid
// slot) are split into 32-slot work units: a chunk whose slots resolve to the
// same source row for every beam (read off the indirection table: the prompt
// and any shared ancestry) gives units serving all R beams, any other chunk
// one unit per beam (its own rows). Units are dealt round-robin to the warps; a
// warp streams its next unit's K and V rows (cp.async, 128-byte XOR swizzle,
// two 8 KB buffers) while it runs the current one on mma.sync m16n8k16 with the
// beams as the M rows:
//   S[beams x 32] = Q K^T  (16 MMAs), scale, mask (slots past the newest, beams
//                           the unit does not serve), online softmax per beam in
//                           registers (flash form, running max / sum),
//   O[beams x 64] += P V   (16 MMAs; P reused from the S fragments as f16).
// Each warp's first unit (all but the newest slot) is staged before the PDL
// wait. The warps' partial states are merged per beam in warp order
// (deterministic), the output rounded once.
constexpr int kBtThreads = 128, kBtMaxUnits = 128;  // <= 16 half-chunks x <= 8 beams
// Per-request beam plan, written by the beam select of the previous step (which
// has just rewritten the request's indirection rows) for the next step's
// attention, so its 12 head CTAs read it instead of each re-deriving it:
// [0, 4096) source beam per window slot, u8 [beam][4096 / beam] (slot lo + k at
// k); [4096] unit count; [4112, +4 * kBtMaxUnits) units, (half-chunk << 8) |
// (beam + 1), beam + 1 = 0 for a unit shared by all beams.
constexpr int kBeamPlanBytes = 4096 + 16 + 4 * kBtMaxUnits;
__host__ __device__ constexpr size_t attn_beam_mma_smem(int R, int nbuf) {
  // q [16][72] f16 | s_ind [R][4096 / R] u8 | 4 warps x nbuf x (K 4 KB + V 4 KB) | merge [4][8][66] f32 (aliases K/V)
  return 16 * 72 * 2 + 4096 + (size_t)4 * nbuf * 8192 + 64 + 0 * R;
}

__device__ __forceinline__ uint32_t xsw(int row, int chunk16) {  // 128-B rows, 16-B chunks XOR-swizzled
  return (uint32_t)(row * 128 + ((chunk16 ^ (row & 7)) << 4));
}

// ------------------------------------------------------------------ decode, prefetching, tensor cores
// The per-row prefetching decode kernel (attn_decode_pf_kernel's staging, grid
// and fixed chunk-order merge) with the per-chunk arithmetic on mma.sync:
// warp w owns chunk w (G <= 4), q is the single nonzero row of the m16n8k16 A
// operand (lanes 0-3 hold it, straight from the QKV output), S = q K^T is 32
// MMAs per chunk, the chunk softmax runs on lanes 0-3 (quad shuffles), and
// O = P V takes P rounded to f16 (as the beam kernel; 32 MMAs). K and V chunks
// are staged with the 128-B XOR swizzle (xsw), conflict-free for ldmatrix.
// Results depend only on the row's own window. Used for every greedy batch
// (the choice must not depend on the batch): on multi-wave grids the 50 KB
// footprint and shorter CTA lifetime let the next CTAs start sooner (C3 538 vs
// 560 us/step); at one wave it is level with the CUDA-core form (C2 311 vs 312).
__global__ void __launch_bounds__(128, 1) attn_decode_pfm_kernel(const AttnArgs a) {
  extern __shared__ __align__(128) uint8_t pfm_smem[];
  __shared__ int s_last;
  constexpr int D = 64;
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(a.trace, 0);
  const int G = a.group;
  uint8_t* kvs = pfm_smem;                                                    // [G][K 8 KB | V 8 KB]
  float* part_s = reinterpret_cast<float*>(pfm_smem + (size_t)G * kPfChunkBytes);  // [G][66]
  const int g = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b], hi = qbase;  // window [lo, hi]
  const int n = hi - lo + 1;
  const int nch = n > 0 ? (n + 63) / 64 : 0;
  const int ngr = (nch + G - 1) / G;
  if (g >= (ngr > 0 ? ngr : 1)) {
    pdl_trigger();
    return;
  }
  const int c0 = g * G, nc = n > 0 ? min(G, nch - c0) : 0;
  const size_t row_off = (size_t)b * a.NH * a.cap * D + (size_t)h * a.cap * D;
  // ---- before the wait: K/V of every slot < hi in this CTA's chunks
  for (int seg = tid; seg < nc * 64 * 8; seg += 128) {
    const int i = seg >> 9, j = (seg >> 3) & 63, part = seg & 7;
    const int slot = lo + (c0 + i) * 64 + j;
    if (slot != hi) {  // slots past the window are zero-filled (src-size 0)
      const bool ok = slot < hi;
      const size_t off = ok ? row_off + (size_t)slot * D + part * 8 : 0;
      uint8_t* kb = kvs + (size_t)i * kPfChunkBytes;
      cp_async16(smem_u32(kb + xsw(j, part)), a.kc + off, ok);
      cp_async16(smem_u32(kb + 8192 + xsw(j, part)), a.vc + off, ok);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  if (a.pf_kc != nullptr && tid < 2 && nc > 0) {
    // next layer's copy of this CTA's window (contiguous slots of one (b, h))
    const int s0 = lo + c0 * 64, s1 = min(lo + (c0 + nc) * 64, hi + 1);
    l2_prefetch_bulk((tid == 0 ? a.pf_kc : a.pf_vc) + row_off + (size_t)s0 * D, (uint32_t)((s1 - s0) * D * 2));
  }
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) tr.mark(a.trace, 1);
  __half* orow = a.out + (size_t)b * a.ldo + (size_t)h * D;
  if (n <= 0) {  // empty window: zeros
    if (tid < D) orow[tid] = __float2half_rn(0.0f);
    return;
  }
  // ---- after the wait: the newest slot, and q (A operand row 0: lanes 0-3)
  {
    const int i = (hi - lo) / 64 - c0, j = (hi - lo) % 64;
    if (i >= 0 && i < nc && tid < 16) {
      const int part = tid & 7;
      const size_t off = row_off + (size_t)hi * D + part * 8;
      uint8_t* dst = kvs + (size_t)i * kPfChunkBytes + (tid < 8 ? 0 : 8192) + xsw(j, part);
      *reinterpret_cast<uint4*>(dst) = *reinterpret_cast<const uint4*>((tid < 8 ? a.kc : a.vc) + off);
    }
  }
  const int gq = lane >> 2, tq = lane & 3;
  uint32_t qa0[4], qa2[4];  // k-step ks: dims ks*16 + 2tq (+1) and ks*16 + 8 + 2tq (+1) of q, row 0 only
  {
    const uint32_t* q32 = reinterpret_cast<const uint32_t*>(a.q + (size_t)b * a.ldq + (size_t)h * D);
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      qa0[ks] = gq == 0 ? q32[ks * 8 + tq] : 0u;
      qa2[ks] = gq == 0 ? q32[ks * 8 + 4 + tq] : 0u;
    }
  }
  cp_async_commit_wait_all();
  __syncthreads();
  if (threadIdx.x == 0) tr.mark(a.trace, 2);
  if (warp < nc) {
    const int i = warp;
    const uint8_t* kb = kvs + (size_t)i * kPfChunkBytes;
    const uint8_t* vb = kb + 8192;
    const int cnt_keys = min(64, n - (c0 + i) * 64);
    // S = q K^T over the chunk's 64 keys: 8 n-tiles x 4 k-steps
    float sc[8][4];
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.0f;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t b0, b1;
        ldsm_x2(smem_u32(kb + xsw(nt * 8 + (lane & 7), ks * 2 + ((lane >> 3) & 1))), b0, b1);
        mma16816(sc[nt], qa0[ks], 0u, qa2[ks], 0u, b0, b1);
      }
    }
    // chunk softmax on row 0 (lanes 0-3 hold keys nt*8 + 2tq, +1)
    float m = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int key = nt * 8 + 2 * tq + e;
        sc[nt][e] = key < cnt_keys ? __fmul_rn(sc[nt][e], a.scale) : -INFINITY;
        m = fmaxf(m, sc[nt][e]);
      }
    }
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, 2));
    float z = 0.0f;
    uint32_t ph[8];  // P as f16 pairs (z sums the f32 weights)
#pragma unroll
    for (int nt = 0; nt < 8; ++nt) {
      const float p0 = sc[nt][0] == -INFINITY ? 0.0f : expf(__fsub_rn(sc[nt][0], m));
      const float p1 = sc[nt][1] == -INFINITY ? 0.0f : expf(__fsub_rn(sc[nt][1], m));
      z = __fadd_rn(z, __fadd_rn(p0, p1));
      ph[nt] = gq == 0 ? pack_h2(p0, p1) : 0u;
    }
    z = __fadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 1));
    z = __fadd_rn(z, __shfl_xor_sync(0xffffffffu, z, 2));
    // O = P V: 4 key k-steps of 16, 8 dim n-tiles of 8
    float o[8][4];
#pragma unroll
    for (int nd = 0; nd < 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.0f;
#pragma unroll
    for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
      for (int nd = 0; nd < 8; ++nd) {
        uint32_t b0, b1;
        const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x2_t(smem_u32(vb + xsw(key, nd)), b0, b1);
        mma16816(o[nd], ph[2 * kk], 0u, ph[2 * kk + 1], 0u, b0, b1);
      }
    }
    if (gq == 0) {
      float* dst = part_s + i * 66;
      if (tq == 0) {
        dst[0] = m;
        dst[1] = z;
      }
#pragma unroll
      for (int nd = 0; nd < 8; ++nd) {
        dst[2 + nd * 8 + 2 * tq] = o[nd][0];
        dst[2 + nd * 8 + 2 * tq + 1] = o[nd][1];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) tr.mark(a.trace, 5);
  // merge in chunk order: M = max m_c, Z = sum z_c e^(m_c - M), O = sum o_c e^(m_c - M)
  auto merge_into = [&](auto ld, int count) {
    if (tid < D) {
      float M = -INFINITY;
      for (int cc = 0; cc < count; ++cc) M = fmaxf(M, ld(cc * 66));
      float Z = 0.0f, O = 0.0f;
      for (int cc = 0; cc < count; ++cc) {
        const float f = expf(__fsub_rn(ld(cc * 66), M));
        Z = __fadd_rn(Z, __fmul_rn(ld(cc * 66 + 1), f));
        O = __fadd_rn(O, __fmul_rn(ld(cc * 66 + 2 + tid), f));
      }
      orow[tid] = f16_sat(__fdiv_rn(O, Z));
    }
  };
  if (ngr == 1) {
    merge_into([&](int e) { return part_s[e]; }, nch);
  } else {
    float* part = a.ws + (((size_t)b * a.NH + h) * a.max_chunks) * 66;
    for (int e = tid; e < nc * 66; e += 128) __stcg(part + (size_t)c0 * 66 + e, part_s[e]);
    fence_acq_rel_gpu();
    __syncthreads();
    if (tid == 0) {
      const int prev = atomicAdd(a.cnt + (size_t)b * a.NH + h, 1);
      s_last = (prev == ngr - 1);
    }
    __syncthreads();
    if (s_last) {
      fence_acq_rel_gpu();
      merge_into([&](int e) { return __ldcg(part + e); }, nch);
      if (tid == 0) a.cnt[(size_t)b * a.NH + h] = 0;
    }
  }
  if (threadIdx.x == 0) {
    tr.mark(a.trace, 7);
    tr.flush(a.trace);
  }
}
__host__ __device__ inline size_t attn_pfm_smem_bytes(int G) {
  return (size_t)G * kPfChunkBytes + (size_t)G * 66 * sizeof(float);
}

// (one buffer per warp at 6 CTAs per SM, one wave at C4, measured slower: 816 vs 789 us per beam step)
__global__ void __launch_bounds__(kBtThreads, 3) attn_decode_beam_mma_kernel(const AttnArgs a) {
  constexpr int NBUF = 2;
  extern __shared__ __align__(128) uint8_t bt_smem[];
  __half* qs = reinterpret_cast<__half*>(bt_smem);                 // [16][72]
  uint8_t* s_ind = bt_smem + 16 * 72 * 2;                           // [R][istr] source beam per slot
  uint8_t* kv = s_ind + 4096;                                       // [4 warps][NBUF][K 4 KB | V 4 KB]
  __shared__ int s_sh[64];  // per 64-slot chunk: all beams share it (window <= 4096 / R slots)
  __shared__ int s_units, s_unit_c[kBtMaxUnits], s_unit_r[kBtMaxUnits];
  constexpr int D = 64;
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(a.trace, 0);
  const int R = a.beam;
  const int istr = 4096 / R;  // slots per indirection row (window <= 4096 / R slots)
  const int h = blockIdx.y, rq = blockIdx.z, beam0 = rq * R;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, tq = lane & 3;
  // the select's plan (if any) is requested before the window scalars: the two
  // loads are independent, so a late-starting CTA waits for one round trip
  uint4 pv[2] = {make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
  int pu = 0, pcnt = 0;
  if (a.plan != nullptr) {
    const uint8_t* P = a.plan + (size_t)rq * kBeamPlanBytes;
#pragma unroll
    for (int e = 0; e < 2; ++e) pv[e] = reinterpret_cast<const uint4*>(P)[tid + e * kBtThreads];
    pu = reinterpret_cast<const int*>(P + 4112)[tid];
    pcnt = *reinterpret_cast<const int*>(P + 4096);
  }
  const int qbase = *a.qbase_dev;
  const int lo = a.start[beam0], hi = qbase;  // the beams of a request share the left pad
  const int n = hi - lo + 1;
  const int nch = n > 0 ? (n + 63) / 64 : 0;
  const size_t row_stride = (size_t)a.NH * a.cap * D, head_stride = (size_t)a.cap * D;
  // ---- before the wait: indirection rows, shared chunks, the unit list (from
  // the select's plan when there is one)
  if (a.plan != nullptr) {
    static_assert(4096 / 16 == 2 * kBtThreads && kBtMaxUnits == kBtThreads, "plan staging: 2 + 1 loads per thread");
#pragma unroll
    for (int e = 0; e < 2; ++e) reinterpret_cast<uint4*>(s_ind)[tid + e * kBtThreads] = pv[e];
    s_unit_c[tid] = pu >> 8;
    s_unit_r[tid] = (pu & 255) - 1;
    if (tid == 0) s_units = pcnt;
    __syncthreads();
  } else {
  {
    // indirection rows: the first 4 rows x 512 slots with 16 loads in flight per
    // thread (late-wave CTAs start while the other CTAs saturate L2; a dependent
    // load per slot made this staging ~4 us of their critical path), the rest
    // (beam > 4 or windows > 512) by the plain loop
    const int per = nch * 64;
    int v[16];
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int r = e >> 2, k = tid + (e & 3) * kBtThreads;
      v[e] = (r < R && k < per) ? ((lo + k < hi && a.indir) ? a.indir[(size_t)(beam0 + r) * a.cap + lo + k] : r) : 0;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int r = e >> 2, k = tid + (e & 3) * kBtThreads;
      if (r < R && k < per) s_ind[r * istr + k] = (uint8_t)v[e];
    }
    if (R > 4 || per > 4 * kBtThreads) {
      for (int i = tid; i < R * per; i += kBtThreads) {
        const int r = i / per, k = i - r * per;
        if (r >= 4 || k >= 4 * kBtThreads)
          s_ind[r * istr + k] = (uint8_t)((lo + k < hi && a.indir) ? a.indir[(size_t)(beam0 + r) * a.cap + lo + k] : r);
      }
    }
  }
  __syncthreads();
  for (int c = warp; c < nch; c += 4) {
    bool same = true;
    for (int kk = c * 64 + lane; kk < c * 64 + 64; kk += 32) {
      const int s = lo + kk;
      if (s == hi) same = false;  // the newest slot: each beam's own row
      for (int r = 1; r < R && s < hi; ++r) same = same && s_ind[r * istr + kk] == s_ind[kk];
    }
    same = __all_sync(0xffffffffu, same);
    if (lane == 0) s_sh[c] = same;
  }
  __syncthreads();
  if (warp == 0) {
    // units: 32-slot halves of the chunks in order (shared: one unit for all
    // beams; else one per beam), placed by a warp prefix sum over the halves
    int base = 0;
    for (int h0 = 0; h0 < 2 * nch; h0 += 32) {
      const int h = h0 + lane;
      const bool live = h < 2 * nch && h * 32 < n;
      const bool sh = live && s_sh[h >> 1];
      const int cnt = live ? (sh ? 1 : R) : 0;
      int incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      const int u0 = base + incl - cnt;
      if (live) {
        if (sh) {
          s_unit_c[u0] = h;
          s_unit_r[u0] = -1;  // all beams
        } else {
          for (int r = 0; r < R; ++r) {
            s_unit_c[u0 + r] = h;
            s_unit_r[u0 + r] = r;
          }
        }
      }
      base += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (lane == 0) s_units = base;
  }
  __syncthreads();
  }
  const int units = s_units;
  // two 8 KB unit buffers per warp (K 4 KB | V 4 KB): the next unit streams in
  // while the current one is computed
  uint8_t* wb = kv + warp * (NBUF * 8192);
  // stage unit u's 32 slots into buffer `buf` (all but the newest slot before the wait)
  auto stage = [&](int u, int buf, bool after_wait) {
    const int hc = s_unit_c[u], ur = s_unit_r[u];
    uint8_t* kb = wb + buf * 8192;
    uint8_t* vb = kb + 4096;
    for (int i = lane; i < 32 * 8; i += 32) {
      const int j = i >> 3, prt = i & 7, k = hc * 32 + j, slot = lo + k;
      if (slot == hi && !after_wait) continue;
      const bool ok = slot <= hi;
      const int rr = ur < 0 ? 0 : ur;
      const int src = beam0 + (slot == hi ? (a.indir ? a.indir[(size_t)(beam0 + rr) * a.cap + hi] : rr)
                                          : s_ind[rr * istr + k]);
      const size_t off = ok ? (size_t)src * row_stride + (size_t)h * head_stride + (size_t)slot * D + prt * 8 : 0;
      cp_async16(smem_u32(kb + xsw(j, prt)), a.kc + off, ok);
      cp_async16(smem_u32(vb + xsw(j, prt)), a.vc + off, ok);
    }
  };
  if (warp < units) stage(warp, 0, false);
  asm volatile("cp.async.commit_group;" ::: "memory");
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) tr.mark(a.trace, 1);
  // the unit staged early may hold the newest slot (written by this layer's QKV GEMM)
  if (warp < units) {
    const int hc = s_unit_c[warp], ur = s_unit_r[warp];
    const int j = hi - lo - hc * 32;
    if (j >= 0 && j < 32 && lane < 8) {
      const int rr = ur < 0 ? 0 : ur;
      const int src = beam0 + (a.indir ? a.indir[(size_t)(beam0 + rr) * a.cap + hi] : rr);
      const size_t off = (size_t)src * row_stride + (size_t)h * head_stride + (size_t)hi * D + lane * 8;
      cp_async16(smem_u32(wb + xsw(j, lane)), a.kc + off, true);
      cp_async16(smem_u32(wb + 4096 + xsw(j, lane)), a.vc + off, true);
    }
  }
  asm volatile("cp.async.commit_group;" ::: "memory");
  // q rows (beams; rows >= R zero), f16 as stored by the QKV epilogue
  for (int i = tid; i < 16 * 8; i += kBtThreads) {
    const int r = i >> 3, prt = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (r < R) v = *reinterpret_cast<const uint4*>(a.q + (size_t)(beam0 + r) * a.ldq + (size_t)h * D + prt * 8);
    *reinterpret_cast<uint4*>(qs + r * 72 + prt * 8) = v;
  }
  __syncthreads();
  uint32_t qa[4][4];  // A fragments of Q: rows g / g+8, 4 k-steps of 16 dims
  {
    const int r = (lane & 7) + ((lane >> 3) & 1) * 8;
#pragma unroll
    for (int ks = 0; ks < 4; ++ks)
      ldsm_x4(smem_u32(qs + r * 72 + ks * 16 + (lane >> 4) * 8), qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3]);
  }
  float m0 = -INFINITY, l0 = 0.0f;  // beam g (rows g + 8 are padding)
  float o[8][4];
#pragma unroll
  for (int nd = 0; nd < 8; ++nd) o[nd][0] = o[nd][1] = o[nd][2] = o[nd][3] = 0.0f;
  int buf = 0;
  for (int u = warp; u < units; u += 4, buf ^= 1) {
    if (u + 4 < units) stage(u + 4, buf ^ 1, true);  // the next unit streams in while this one computes
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    const uint8_t* kb = wb + buf * 8192;
    const uint8_t* vb = kb + 4096;
    const int hc = s_unit_c[u], ur = s_unit_r[u];
    // S = Q K^T: 4 key n-tiles of 8
    float sc[4][4];
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      sc[nt][0] = sc[nt][1] = sc[nt][2] = sc[nt][3] = 0.0f;
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        uint32_t b0, b1;
        ldsm_x2(smem_u32(kb + xsw(nt * 8 + (lane & 7), ks * 2 + ((lane >> 3) & 1))), b0, b1);
        mma16816(sc[nt], qa[ks][0], qa[ks][1], qa[ks][2], qa[ks][3], b0, b1);
      }
    }
    // scale + mask (rows: beam g; the unit serves beam ur, or all), unit max
    const bool row_in = g < R && (ur < 0 || ur == g);
    float mx = -INFINITY;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int slot = lo + hc * 32 + nt * 8 + 2 * tq + e;
        sc[nt][e] = (row_in && slot <= hi) ? __fmul_rn(sc[nt][e], a.scale) : -INFINITY;
        mx = fmaxf(mx, sc[nt][e]);
      }
    }
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 1));
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 2));
    const float mn = fmaxf(m0, mx);
    const float al = (m0 == -INFINITY) ? 0.0f : expf(__fsub_rn(m0, mn));
    float ps = 0.0f;
    uint32_t pa[4];  // P as f16 pairs: row g (rows g+8 are zero)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
      const float p0 = sc[nt][0] == -INFINITY ? 0.0f : expf(__fsub_rn(sc[nt][0], mn));
      const float p1 = sc[nt][1] == -INFINITY ? 0.0f : expf(__fsub_rn(sc[nt][1], mn));
      ps = __fadd_rn(ps, __fadd_rn(p0, p1));
      pa[nt] = pack_h2(p0, p1);
    }
    if (mx != -INFINITY) {  // this unit has visible keys for beam g
      l0 = __fadd_rn(__fmul_rn(l0, al), ps);
      m0 = mn;
#pragma unroll
      for (int nd = 0; nd < 8; ++nd) {
        o[nd][0] = __fmul_rn(o[nd][0], al);
        o[nd][1] = __fmul_rn(o[nd][1], al);
      }
    }
    // O += P V: 2 key k-steps of 16, 8 dim n-tiles of 8
#pragma unroll
    for (int kk = 0; kk < 2; ++kk) {
#pragma unroll
      for (int nd = 0; nd < 8; ++nd) {
        uint32_t b0, b1;
        const int key = kk * 16 + (lane & 7) + ((lane >> 3) & 1) * 8;
        ldsm_x2_t(smem_u32(vb + xsw(key, nd)), b0, b1);
        mma16816(o[nd], pa[2 * kk], 0u, pa[2 * kk + 1], 0u, b0, b1);
      }
    }
    __syncwarp();  // every lane's ldmatrix done before this buffer is restaged
  }
  if (threadIdx.x == 0) tr.mark(a.trace, 5);
  // per-beam merge of the 4 warps' states, in warp order
  l0 = __fadd_rn(l0, __shfl_xor_sync(0xffffffffu, l0, 1));
  l0 = __fadd_rn(l0, __shfl_xor_sync(0xffffffffu, l0, 2));
  __syncthreads();  // all warps done with their K/V buffers (reused for the merge)
  float* mrg = reinterpret_cast<float*>(kv);  // [4 warps][8 beams][66]: m, l, O[64]
  if (g < R) {
    float* dst = mrg + ((size_t)warp * 8 + g) * 66;
    if (tq == 0) {
      dst[0] = m0;
      dst[1] = l0;
    }
#pragma unroll
    for (int nd = 0; nd < 8; ++nd) {
      dst[2 + nd * 8 + 2 * tq] = o[nd][0];
      dst[2 + nd * 8 + 2 * tq + 1] = o[nd][1];
    }
  }
  __syncthreads();
  for (int i = tid; i < R * D; i += kBtThreads) {
    const int r = i / D, d = i - r * D;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, mrg[((size_t)w * 8 + r) * 66]);
    float Z = 0.0f, O = 0.0f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float* P = mrg + ((size_t)w * 8 + r) * 66;
      if (P[0] == -INFINITY) continue;
      const float f = expf(__fsub_rn(P[0], M));
      Z = __fadd_rn(Z, __fmul_rn(P[1], f));
      O = __fadd_rn(O, __fmul_rn(P[2 + d], f));
    }
    a.out[(size_t)(beam0 + r) * a.ldo + (size_t)h * D + d] = f16_sat(Z > 0.0f ? __fdiv_rn(O, Z) : 0.0f);
  }
  if (threadIdx.x == 0) {
    tr.mark(a.trace, 7);
    tr.flush(a.trace);
  }
}

// ------------------------------------------------------------------ prefill, tcgen05
// head_dim 64. One CTA = 128 query rows of one (head, sequence); query row r =
// TMEM lane r. Key chunks of 64 slots aligned to start[b] (as in every other
// attention kernel: a row's arithmetic never depends on its batch's padding).
// One pass over the chunks (flash form):
//   S_j = Q K_j^T   tcgen05.mma kind::f16 M=128 N=64 K=64, f32 in TMEM (issued
//                   as soon as every thread has read S_{j-1}, so it runs while
//                   chunk j-1's P is computed; 128 TMEM columns per CTA keep
//                   three CTAs per SM);
//   P_j = exp(s - m) with a per-row reference max m that is raised only when a
//        chunk's max exceeds it by more than kTcRescale (then O and the sums
//        are rescaled in place: tcgen05.ld / st of the O columns), rounded to
//        f16 into a K-major SW128 tile;
//   O  += P_j V_j   tcgen05.mma with V read MN-major (the cache's [slot][d]
//                   rows, no transpose);
//   out = q16(O / sum).
// 8 warps: warps w and w + 4 share TMEM lane quadrant w % 4 and take the column
// halves w / 4 of every chunk (and of O); the halves of a row agree on m
// through shared memory once per chunk.
constexpr int kTcRows = 128, kTcKeys = 64, kTcThreads = 256;
constexpr int kTcTile = 128 * 128;  // Q or P tile bytes (128 rows x 64 f16)
constexpr int kTcChunk = 64 * 128;  // K or V chunk bytes (64 slots x 64 f16)
constexpr size_t kTcSmem = 1024 + 2 * kTcTile + 4 * kTcChunk + 64 + 2 * 128 * 8;
constexpr float kTcRescale = 5.0f;  // P <= e^5 between rescales

__device__ __forceinline__ uint32_t sw128_off(int row, int chunk16) {  // byte offset of 16-B chunk
  return (uint32_t)((row >> 3) * 1024 + (row & 7) * 128 + ((chunk16 ^ (row & 7)) << 4));
}

__global__ void __launch_bounds__(kTcThreads) attn_prefill_tc_kernel(const AttnArgs a) {
  extern __shared__ uint8_t tc_smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(tc_smem_raw) + 1023) & ~(uintptr_t)1023);
  uint8_t* qs = sm;
  uint8_t* ps = sm + kTcTile;
  uint8_t* kbuf = sm + 2 * kTcTile;                // [2][kTcChunk]
  uint8_t* vbuf = sm + 2 * kTcTile + 2 * kTcChunk;  // [2][kTcChunk]
  uint64_t* bar = reinterpret_cast<uint64_t*>(sm + 2 * kTcTile + 4 * kTcChunk);  // [0]: S, [2]: PV
  float* stat = reinterpret_cast<float*>(sm + 2 * kTcTile + 4 * kTcChunk + 64);   // [2 halves][128 rows]
  __shared__ uint32_t tmem_slot;
  constexpr int D = 64;
  const int qblk = blockIdx.x, h = blockIdx.y, b = blockIdx.z;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const uint32_t sbar0 = smem_u32(bar), pvbar = smem_u32(bar + 2);
  if (tid == 0) {
    mbar_init(sbar0, 1);
    mbar_init(sbar0 + 8, 1);
    mbar_init(pvbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(smem_u32(&tmem_slot), 128);  // S [0,64) O [64,128)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_slot;
  pdl_wait();
  pdl_trigger();
  const int qbase = *a.qbase_dev;
  const int lo = a.start[b];
  const int t0 = qblk * kTcRows;
  const int rows = min(kTcRows, a.T - t0);
  const int hi_blk = qbase + t0 + rows - 1;
  const int nch = hi_blk >= lo ? (hi_blk - lo) / kTcKeys + 1 : 0;
  const size_t head_off = ((size_t)b * a.NH + h) * a.cap * D;
  const __half* K = a.kc + head_off;
  const __half* V = a.vc + head_off;
  for (int i = tid; i < kTcRows * 8; i += kTcThreads) {
    const int r = i >> 3, c = i & 7;
    const bool ok = r < rows;
    cp_async16(smem_u32(qs + sw128_off(r, c)),
               ok ? (const void*)(a.q + (size_t)(b * a.T + t0 + r) * a.ldq + h * D + c * 8) : (const void*)a.q, ok);
  }
  auto load = [&](const __half* src, uint8_t* base, int j) {  // one 64-slot chunk, rows = slots
    for (int i = tid; i < kTcKeys * 8; i += kTcThreads) {
      const int kk = i >> 3, c = i & 7, slot = lo + j * kTcKeys + kk;
      const bool ok = slot <= hi_blk && slot < a.cap;
      cp_async16(smem_u32(base + sw128_off(kk, c)), ok ? (const void*)(src + (size_t)slot * D + c * 8) : (const void*)src,
                 ok);
    }
  };
  const int r = (warp & 3) * 32 + lane;  // query row = TMEM lane
  const int half = warp >> 2;            // column half of each chunk and of O
  const bool row_ok = r < rows;
  const int hi_r = qbase + t0 + r;  // last visible slot of this row
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(32 * half);
  const uint32_t idesc = idesc_f16_m128(64);
  const uint32_t idesc_pv = idesc | (1u << 16);  // B (= V [slot][d]) MN-major
  uint32_t sph = 0u, pvph = 0u;
  auto issue_qk = [&](int j) {  // S = Q K_j^T (tid 0)
    if (tid == 0) {
      tc_fence_after();
      const uint64_t da = umma_desc_sw128(smem_u32(qs));
      const uint64_t db = umma_desc_sw128(smem_u32(kbuf + (j & 1) * kTcChunk));
#pragma unroll
      for (int k = 0; k < D / 16; ++k) tc_mma_f16(tmem, da + 2 * k, db + 2 * k, idesc, k != 0 ? 1u : 0u);
      tc_commit(sbar0);
    }
  };
  auto publish = [&]() {  // this thread's cp.async data and smem stores -> visible to the tensor core
    asm volatile("cp.async.commit_group;\n\tcp.async.wait_group 0;" ::: "memory");
    fence_proxy_async_smem();
    tc_fence_before();
    __syncthreads();
  };
  int pv_waited = 0;  // PV commits observed
  auto wait_pv = [&](int k) {
    while (pv_waited <= k) {
      mbar_wait(pvbar, pvph);
      pvph ^= 1u;
      ++pv_waited;
    }
    tc_fence_after();
  };
  float m = -INFINITY, l = 0.0f;  // reference max of the row; exp-sum of this half's columns
  if (nch > 0) {
    load(K, kbuf, 0);
    load(V, vbuf, 0);
  }
  if (nch > 1) load(K, kbuf + kTcChunk, 1);
  publish();
  if (nch > 0) issue_qk(0);
  for (int j = 0; j < nch; ++j) {
    mbar_wait(sbar0, sph);
    sph ^= 1u;
    tc_fence_after();
    float s[32];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      float v[16];
      tmem_ld16(trow + (uint32_t)(16 * q), v);
#pragma unroll
      for (int e = 0; e < 16; ++e) {
        const int slot = lo + j * kTcKeys + 32 * half + 16 * q + e;
        s[16 * q + e] = (row_ok && slot <= hi_r) ? __fmul_rn(v[e], a.scale) : -INFINITY;
      }
    }
    float cm = -INFINITY;
#pragma unroll
    for (int e = 0; e < 32; ++e) cm = fmaxf(cm, s[e]);
    stat[half * 128 + r] = cm;
    if (j > 0) wait_pv(j - 1);  // the P tile, V buffer (j - 1) & 1 and O are stable
    publish();                  // S read by all; K(j+1) and V(j) landed
    if (j + 1 < nch) issue_qk(j + 1);  // runs while P(j) is computed
    cm = fmaxf(cm, stat[(half ^ 1) * 128 + r]);  // the row's chunk max (both halves)
    const bool raise = cm != -INFINITY && (m == -INFINITY || cm > m + kTcRescale);
    float alpha = 1.0f;
    if (raise) {
      alpha = m == -INFINITY ? 0.0f : expf(__fsub_rn(m, cm));
      l = __fmul_rn(l, alpha);
      m = cm;
    }
    if (j > 0 && __any_sync(0xffffffffu, raise)) {  // rescale this warp's O rows (warp-collective TMEM ops)
#pragma unroll
      for (int q = 0; q < 2; ++q) {
        float v[16];
        tmem_ld16(trow + 64u + (uint32_t)(16 * q), v);
#pragma unroll
        for (int e = 0; e < 16; ++e) v[e] = __fmul_rn(v[e], alpha);
        tmem_st16(trow + 64u + (uint32_t)(16 * q), v);
      }
    }
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      float pv[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float x = s[8 * c + e];
        pv[e] = x == -INFINITY ? 0.0f : expf(__fsub_rn(x, m));
        l = __fadd_rn(l, pv[e]);
      }
      *reinterpret_cast<uint4*>(ps + sw128_off(r, 4 * half + c)) = pack8(pv);
    }
    publish();  // P(j) written, V(j) landed, O rescaled
    if (tid == 0) {
      tc_fence_after();
      const uint64_t da = umma_desc_sw128(smem_u32(ps));
      const uint64_t db = umma_desc_sw128(smem_u32(vbuf + (j & 1) * kTcChunk));
#pragma unroll
      for (int k = 0; k < kTcKeys / 16; ++k)  // 16 slots = two 1024-B row groups of the MN-major V tile
        tc_mma_f16(tmem + 64, da + 2 * k, db + (uint64_t)(128 * k), idesc_pv, (j | k) != 0 ? 1u : 0u);
      tc_commit(pvbar);
    }
    if (j + 2 < nch) load(K, kbuf + (j & 1) * kTcChunk, j + 2);        // QK(j) done
    if (j + 1 < nch) load(V, vbuf + ((j + 1) & 1) * kTcChunk, j + 1);  // PV(j-1) done
  }
  // the row's exp-sum: both halves (half 0's term first in both threads)
  stat[half * 128 + r] = l;
  if (nch > 0) wait_pv(nch - 1);
  __syncthreads();
  const float lo_sum = stat[r], hi_sum = stat[128 + r];
  const float tot = __fadd_rn(lo_sum, hi_sum);
  const float inv = tot > 0.0f ? __fdiv_rn(1.0f, tot) : 0.0f;
  __half* orow = a.out + (size_t)(b * a.T + t0 + r) * a.ldo + h * D + 32 * half;
#pragma unroll
  for (int q = 0; q < 2; ++q) {
    float v[16];
    if (nch > 0) {  // CTA-uniform: tcgen05.ld is warp-collective, every lane takes part
      tmem_ld16(trow + 64u + (uint32_t)(16 * q), v);
    } else {
#pragma unroll
      for (int e = 0; e < 16; ++e) v[e] = 0.0f;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = __fmul_rn(v[e], inv);
    if (row_ok) {
      *reinterpret_cast<uint4*>(orow + 16 * q) = pack8(v);
      *reinterpret_cast<uint4*>(orow + 16 * q + 8) = pack8(v + 8);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 128);
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
