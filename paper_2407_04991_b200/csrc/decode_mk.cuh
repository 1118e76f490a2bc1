// Persistent decode megakernel (sm_100a): every greedy decode step of a session
// in ONE launch, one CTA per SM, dataflow-synchronised through device counters.
//
// Why: a C2 decode step moves ~420 MB (floor ~65 us at 6.45 TB/s) but is a chain
// of ~7 dependent phases per layer x 12 layers; as separate kernels the fixed
// launch/ramp/tail costs dominate (~800 us/step). Here weights never wait for
// data: each CTA's weight producer streams its static list of weight tiles
// through a TMA ring as fast as the ring drains, across phase, layer and step
// boundaries; only the tiny activation operands wait on dependency counters.
//
// Decomposition (H, F multiples of 128; D == 64; batch <= bn <= 128):
//   GEMM items — 128 output features x 128 K (two 64-wide K blocks), swap-AB
//   tcgen05 (weights on MMA-M, batch on MMA-N), f32 partial tile to global:
//     QKV(l, t, c)  t < 3H/128, c < H/128     input h1 (TMA)
//     WO (l, t, c)  t < H/128,  c < H/128     input attn (TMA), needs heads 2c, 2c+1
//     W1 (l, t, c)  t < F/128,  c < H/128     input h2 (TMA)
//     W2 (l, t, c)  t < H/128,  c < F/128     input gelu(sum of W1 partials of tile c)
//                                             built in smem by the helper warps
//     LM (t)        t < V/128, full K         input hf (TMA), argmax epilogue
//   aux tasks (4-warp group):
//     ATT(l, b, h)  reduce q/k/v partials (+bias, f16), append k/v to the cache,
//                   exact two-pass softmax over slots [pad_b, len]
//     R2 (l, b)     x += q16(sum Wo partials + bo); h2 = LN2(x)
//     R1 (l, b)     x += q16(sum W2 partials + b2); h1 = LN1'(x) (next layer / final)
//     EMB(b)        token = argmax key of the previous step; append; x, h1 = LN(emb)
// Every reduction sums its partials in a fixed order (deterministic).
// Counters are monotonic within a launch (zeroed by the host before it): the
// consumer of step s waits for (s + 1) x per-step count.
#pragma once

#include "common.cuh"

namespace tf {
namespace mk {

constexpr int kMaxLayers = 24;
constexpr int kThreads = 384;  // 12 warps
constexpr int kKC = 128;       // K per GEMM item (two 64-wide blocks)
constexpr int kWSlot = 128 * 64 * 2;

enum GemmType : int { G_QKV = 0, G_WO = 1, G_W1 = 2, G_W2 = 3, G_LM = 4 };
enum AuxType : int { A_ATT = 0, A_R2 = 1, A_R1 = 2, A_EMB = 3 };

struct Layer {
  const float *ln1_g, *ln1_b, *bqkv, *bo, *ln2_g, *ln2_b, *b1, *b2;
};

struct Maps {
  CUtensorMap w[4 * kMaxLayers + 1];  // per layer: qkv, wo, w1, w2; then lm_head
  CUtensorMap act[4];                 // h1, attn, h2, hf   (box 64 x bn)
};

struct Params {
  int L, H, F, NH, V, B, bn, cap, n_steps, ws, bs;  // ws/bs: weight / B ring stages
  int nck, ncf, nqkv, lm_tiles;                       // H/128, F/128, 3H/128, ceil(V/128)
  const Layer* layers;
  const float *fin_g, *fin_b;
  const __half *tok_emb, *pos_emb;
  int ldw;
  __half *x, *h1, *h2, *attn, *hf;
  int ldx;
  float *p_qkv, *p_wo, *p_w1, *p_w2;
  __half *kc, *vc;
  const int* pads;
  int* len_dev;
  int* step_dev;
  unsigned long long* keys;
  int* out_tokens;
  int max_new;
  int* ctr;
  const int4* items;
  const int* item_off;  // [gridDim.x + 1]
  const int4* aux;
  const int* aux_off;
  float scale;
  long long* trace;  // optional: [items + aux][3] globaltimer stamps of step `trace_step`
  int trace_step;
  int flags;     // bit0: L2 evict_first on weight loads; bit1: relaxed polling + fence
  int sleep_ns;  // poll back-off
};

// ---------------------------------------------------------------- counters
struct Ctr {
  int *h1, *qkv, *att, *wo, *h2, *w1, *w2, *lm;
  __device__ Ctr(const Params& p) {
    int* c = p.ctr;
    h1 = c;
    qkv = h1 + (p.L + 1);
    att = qkv + p.L * p.nqkv;
    wo = att + p.L * p.NH;
    h2 = wo + p.L;
    w1 = h2 + p.L;
    w2 = w1 + p.L * p.ncf;
    lm = w2 + p.L;
  }
};
__host__ __device__ inline int ctr_count(int L, int nqkv, int NH, int ncf) {
  return (L + 1) + L * nqkv + L * NH + L + L + L * ncf + L + 1;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ int g_poll_mode = 0;     // set by the host before each launch (Params.flags bit1)
__device__ int g_poll_sleep = 128;  // ns
__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (g_poll_mode) {
    if (ld_relaxed(p) < target) {
      unsigned ns = 32;
      while (ld_relaxed(p) < target) {
        __nanosleep(ns);
        ns = ns < (unsigned)g_poll_sleep ? ns * 2 : ns;
      }
    }
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    return;
  }
  if (ld_acquire(p) >= target) return;
  while (ld_acquire(p) < target) __nanosleep(g_poll_sleep);
}
__device__ __forceinline__ void signal_add(int* p) {
  __threadfence();
  atomicAdd(p, 1);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void group_bar(int id) {  // named barrier over one 4-warp group
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
__device__ __forceinline__ float ldcg(const float* p) { return __ldcg(p); }
__device__ __forceinline__ float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }

// sum of `n` partial values base[ch * stride] in chunk order, loads batched 8 at a
// time so one round trip covers up to 8 chunks
__device__ __forceinline__ float sum_parts(const float* base, size_t stride, int n) {
  float acc = 0.0f;
  for (int c0 = 0; c0 < n; c0 += 8) {
    float t[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) t[u] = (c0 + u < n) ? __ldcg(base + (size_t)(c0 + u) * stride) : 0.0f;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (c0 + u < n) acc = __fadd_rn(acc, t[u]);
  }
  return acc;
}

__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes >= 16)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15u) : "memory");
}

__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// partial tile base: [tile][chunk][bn][128]
__device__ __forceinline__ float* part_ptr(float* base, int tile, int nchunks, int chunk, int bn) {
  return base + ((size_t)tile * nchunks + chunk) * bn * 128;
}

__device__ __forceinline__ int item_nkb(const Params& p, int type) {
  return type == G_LM ? p.nck * 2 : 2;
}

// weight map index and K-block offset of a GEMM item
__device__ __forceinline__ const CUtensorMap* item_wmap(const Maps& m, const Params& p, const int4& it) {
  return it.x == G_LM ? &m.w[4 * p.L] : &m.w[4 * it.y + it.x];
}

// ---------------------------------------------------------------- group LayerNorm
// 128 threads reduce one row of H f32 values held as v[j] for c = tid + 128*j.
template <int VPT>
__device__ __forceinline__ void group_ln_row(float (&v)[VPT], int H, const float* g, const float* b,
                                             __half* out, float* red, int bar_id) {
  const int tid = threadIdx.x & 127;
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < VPT; ++j)
    if (tid + 128 * j < H) s = __fadd_rn(s, v[j]);
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  group_bar(bar_id);
  const float mean = __fdiv_rn((red[0] + red[1]) + (red[2] + red[3]), (float)H);
  group_bar(bar_id);
  float ss = 0.0f;
#pragma unroll
  for (int j = 0; j < VPT; ++j)
    if (tid + 128 * j < H) {
      const float d = __fsub_rn(v[j], mean);
      ss = __fadd_rn(ss, __fmul_rn(d, d));
    }
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  group_bar(bar_id);
  const float var = __fdiv_rn((red[0] + red[1]) + (red[2] + red[3]), (float)H);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  group_bar(bar_id);
#pragma unroll
  for (int j = 0; j < VPT; ++j) {
    const int c = tid + 128 * j;
    if (c < H) out[c] = f16_sat(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[j], mean), inv), g[c]), b[c]));
  }
}

constexpr int kVPT = 8;  // H <= 1024 (features per thread of a 128-thread row task)

// ---------------------------------------------------------------- aux tasks
constexpr int kAttWarpFloats = 192;  // + cap: per-warp scratch (q, new k, new v, scores)

// Attention for (layer l, row b, head h) at step s by ONE warp (warp-level sync
// only), so the 4 aux warps of a CTA run 4 independent tasks concurrently.
__device__ void warp_attention(const Params& p, const Ctr& c, int l, int b, int h, int s, float* sm,
                               long long* ts) {
  const int lane = threadIdx.x & 31;
  auto stamp = [&](int k) {
    if (ts && lane == 0) ts[k] = gtimer();
  };
  constexpr int D = 64;
  const int len = *p.len_dev + s;  // slot of the new token
  const int lo = p.pads[b];
  float* qs = sm;        // [64]
  float* kn = sm + 64;   // [64]
  float* vn = sm + 128;  // [64]
  float* sc = sm + 192;  // [cap]
  const size_t head_off = (((size_t)l * p.B + b) * p.NH + h) * (size_t)p.cap * D;
  __half* K = p.kc + head_off;
  __half* V = p.vc + head_off;
  if (lane == 0 && len > lo) {  // cached K/V -> L2 while the QKV GEMMs run
    prefetch_l2(K + (size_t)lo * D, (uint32_t)(len - lo) * D * 2);
    prefetch_l2(V + (size_t)lo * D, (uint32_t)(len - lo) * D * 2);
  }
  const int tq = (h * D) / 128, tk = (p.H + h * D) / 128, tv = (2 * p.H + h * D) / 128;
  if (lane == 0) {
    const int tgt = p.nck * (s + 1);
    wait_ge(c.qkv + l * p.nqkv + tq, tgt);
    wait_ge(c.qkv + l * p.nqkv + tk, tgt);
    wait_ge(c.qkv + l * p.nqkv + tv, tgt);
  }
  __syncwarp();
  stamp(1);
  // q, k, v: lane owns d = lane and lane + 32 of each; chunk-outer batched sums
  {
    const float* src[6];
    int fe[6];
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      const int w = u >> 1, d = lane + 32 * (u & 1);
      const int f = w * p.H + h * D + d;
      fe[u] = f;
      src[u] = part_ptr(p.p_qkv, f >> 7, p.nck, 0, p.bn) + (size_t)b * 128 + (f & 127);
    }
    float acc[6] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    const size_t stride = (size_t)p.bn * 128;
    for (int c0 = 0; c0 < p.nck; c0 += 4) {
      float t[4][6];
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int u = 0; u < 6; ++u) t[cc][u] = (c0 + cc < p.nck) ? __ldcg(src[u] + (size_t)(c0 + cc) * stride) : 0.0f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
#pragma unroll
        for (int u = 0; u < 6; ++u)
          if (c0 + cc < p.nck) acc[u] = __fadd_rn(acc[u], t[cc][u]);
    }
    const float* bq = p.layers[l].bqkv;
#pragma unroll
    for (int u = 0; u < 6; ++u) {
      const int w = u >> 1, d = lane + 32 * (u & 1);
      const __half hv = f16_sat(__fadd_rn(acc[u], bq[fe[u]]));
      if (w == 0) {
        qs[d] = __half2float(hv);
      } else if (w == 1) {
        kn[d] = __half2float(hv);
        K[(size_t)len * D + d] = hv;
      } else {
        vn[d] = __half2float(hv);
        V[(size_t)len * D + d] = hv;
      }
    }
  }
  __syncwarp();
  stamp(3);
  const int n = len - lo + 1;  // window [lo, len], the new slot last
  const int sub = lane >> 3, gl = lane & 7;
  float qv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) qv[e] = qs[gl * 8 + e];
  // scores: 8 lanes per key row (16 B each), 4 keys per load, 8 loads in flight
  for (int base = 0; base < n; base += 32) {
    uint4 raw[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int slot = lo + base + 4 * u + sub;
      raw[u] = (base + 4 * u + sub < n && slot < len)
                   ? __ldcg(reinterpret_cast<const uint4*>(K + (size_t)slot * D + gl * 8))
                   : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      float acc = 0.0f;
      if (lo + j < len) {
        const __half2* kh = reinterpret_cast<const __half2*>(&raw[u]);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const float2 kf = __half22float2(kh[e]);
          acc = __fadd_rn(acc, __fmul_rn(qv[2 * e], kf.x));
          acc = __fadd_rn(acc, __fmul_rn(qv[2 * e + 1], kf.y));
        }
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, __fmul_rn(qv[e], kn[gl * 8 + e]));
      }
      acc += __shfl_xor_sync(0xffffffffu, acc, 4);
      acc += __shfl_xor_sync(0xffffffffu, acc, 2);
      acc += __shfl_xor_sync(0xffffffffu, acc, 1);
      if (gl == 0 && j < n) sc[j] = __fmul_rn(acc, p.scale);
    }
  }
  __syncwarp();
  stamp(4);
  float m = -INFINITY;
  for (int j = lane; j < n; j += 32) m = fmaxf(m, sc[j]);
  m = warp_max(m);
  float z = 0.0f;
  for (int j = lane; j < n; j += 32) {
    const float e = expf(__fsub_rn(sc[j], m));
    sc[j] = e;
    z += e;
  }
  z = warp_sum(z);
  const float inv = __fdiv_rn(1.0f, z);
  __syncwarp();
  stamp(5);
  // P.V: 8 lanes per value row (8 dims each), 4 keys per load, 8 loads in flight
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < n; base += 32) {
    uint4 raw[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int slot = lo + base + 4 * u + sub;
      raw[u] = (base + 4 * u + sub < n && slot < len)
                   ? __ldcg(reinterpret_cast<const uint4*>(V + (size_t)slot * D + gl * 8))
                   : make_uint4(0, 0, 0, 0);
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      if (j < n) {
        const float w = __fmul_rn(sc[j], inv);
        float vf[8];
        if (lo + j < len) {
          unpack8(raw[u], vf);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) vf[e] = vn[gl * 8 + e];
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = __fadd_rn(o[e], __fmul_rn(w, vf[e]));
      }
    }
  }
  stamp(6);
#pragma unroll
  for (int e = 0; e < 8; ++e) {  // combine the 4 key sub-groups (fixed order)
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 8));
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 16));
  }
  if (sub == 0) {
    *reinterpret_cast<uint4*>(p.attn + (size_t)b * p.ldx + h * D + gl * 8) = pack8(o);
    __threadfence();
  }
  __syncwarp();
  if (lane == 0) signal_add(c.att + l * p.NH + h);
  stamp(7);
}

// x += q16(sum of partials + bias); then LN -> out. 128 threads (group barrier 1).
__device__ void aux_resid_ln(const Params& p, const float* part, int nchunks, const float* bias,
                             int b, const float* g, const float* be, __half* out, float* red) {
  const int tid = threadIdx.x & 127;
  float v[kVPT];
  __half* xr = p.x + (size_t)b * p.ldx;
  const int nf = (p.H - tid + 127) / 128;  // features of this thread: tid + 128 j
  const size_t stride = (size_t)p.bn * 128;
#pragma unroll
  for (int j = 0; j < kVPT; ++j) v[j] = 0.0f;
  // feature f = tid + 128 j lives in partial tile j (f >> 7 == j), row r = tid
  const float* src0 = part + (size_t)b * 128 + tid;
  for (int c0 = 0; c0 < nchunks; c0 += 4) {
    float t[4][kVPT];
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int j = 0; j < kVPT; ++j)
        t[cc][j] = (j < nf && c0 + cc < nchunks)
                       ? __ldcg(src0 + ((size_t)j * nchunks + c0 + cc) * stride) : 0.0f;
#pragma unroll
    for (int cc = 0; cc < 4; ++cc)
#pragma unroll
      for (int j = 0; j < kVPT; ++j)
        if (j < nf && c0 + cc < nchunks) v[j] = __fadd_rn(v[j], t[cc][j]);
  }
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int f = tid + 128 * j;
    if (j < nf) {
      const float o = q16(__fadd_rn(v[j], bias[f]));
      const __half xn = f16_sat(__fadd_rn(__half2float(__ldcg(xr + f)), o));
      xr[f] = xn;
      v[j] = __half2float(xn);
    } else {
      v[j] = 0.0f;
    }
  }
  group_ln_row<kVPT>(v, p.H, g, be, out + (size_t)b * p.ldx, red, 1);
}

__device__ void aux_embed(const Params& p, int b, int s, float* red) {
  const int tid = threadIdx.x & 127;
  const int len = *p.len_dev + s;
  const unsigned long long key = __ldcg(p.keys + b);
  const int tok = (int)argmax_id(key);
  group_bar(1);
  if (tid == 0) {
    p.keys[b] = 0ull;
    const int col = *p.step_dev + s - 1;  // previous forward's token
    if (s > 0 && col < p.max_new) p.out_tokens[(size_t)b * p.max_new + col] = tok;
  }
  const int pos = len - p.pads[b];
  float v[kVPT];
  __half* xr = p.x + (size_t)b * p.ldx;
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int f = tid + 128 * j;
    v[j] = 0.0f;
    if (f < p.H) {
      const __half xn = f16_sat(__fadd_rn(__half2float(p.tok_emb[(size_t)tok * p.ldw + f]),
                                          __half2float(p.pos_emb[(size_t)pos * p.ldw + f])));
      xr[f] = xn;
      v[j] = __half2float(xn);
    }
  }
  group_ln_row<kVPT>(v, p.H, p.layers[0].ln1_g, p.layers[0].ln1_b, p.h1 + (size_t)b * p.ldx, red, 1);
}

// ---------------------------------------------------------------- the kernel
__global__ void __launch_bounds__(kThreads, 1) decode_megakernel(const __grid_constant__ Maps maps,
                                                                   const Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int bslot = p.bn * 128;
  uint8_t* wring = smem;
  uint8_t* bring = wring + (size_t)p.ws * kWSlot;
  uint64_t* bars = reinterpret_cast<uint64_t*>(bring + (size_t)p.bs * bslot);
  // barriers: wfull[ws] wempty[ws] bfull[bs] bempty[bs] accfull[2] accempty[2]
  const uint32_t wfull = smem_u32(bars), wempty = wfull + 8 * p.ws;
  const uint32_t bfull = wempty + 8 * p.ws, bempty = bfull + 8 * p.bs;
  const uint32_t accfull = bempty + 8 * p.bs, accempty = accfull + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * p.ws + 2 * p.bs + 4);
  float* aux_sm = reinterpret_cast<float*>(tmem_slot + 4);          // attention / LN scratch
  unsigned long long* lm_red =
      reinterpret_cast<unsigned long long*>(aux_sm + ((448 + 4 * (kAttWarpFloats + p.cap) + 1) & ~1));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Ctr c(p);
  const uint32_t ncols = p.bn * 2 <= 32 ? 32 : (p.bn * 2 <= 64 ? 64 : (p.bn * 2 <= 128 ? 128 : 256));

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4 * p.L + 1; ++i) tma_prefetch_desc(&maps.w[i]);
    for (int i = 0; i < 4; ++i) tma_prefetch_desc(&maps.act[i]);
    for (int i = 0; i < p.ws; ++i) {
      mbar_init(wfull + 8 * i, 1);
      mbar_init(wempty + 8 * i, 1);
    }
    for (int i = 0; i < p.bs; ++i) {
      mbar_init(bfull + 8 * i, 1);
      mbar_init(bempty + 8 * i, 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(accfull + 8 * i, 1);
      mbar_init(accempty + 8 * i, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int i0 = p.item_off[blockIdx.x], i1 = p.item_off[blockIdx.x + 1];
  const int a0 = p.aux_off[blockIdx.x], a1 = p.aux_off[blockIdx.x + 1];
  const int B = p.B;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ weight producer (runs ahead)
      int wk = 0;
      const uint64_t pol = l2_policy_evict_first();
      const bool hint = (p.flags & 1) != 0;
      for (int s = 0; s < p.n_steps; ++s) {
        for (int i = i0; i < i1; ++i) {
          const int4 it = p.items[i];
          const CUtensorMap* map = item_wmap(maps, p, it);
          const int nkb = item_nkb(p, it.x);
          const int kb0 = it.x == G_LM ? 0 : it.w * 2;
          for (int kb = 0; kb < nkb; ++kb, ++wk) {
            const int st = wk % p.ws;
            const uint32_t ph = (uint32_t)(wk / p.ws) & 1u;
            mbar_wait(wempty + 8 * st, ph ^ 1u);
            mbar_expect_tx(wfull + 8 * st, kWSlot);
            if (hint)
              tma_load_2d_hint(smem_u32(wring + (size_t)st * kWSlot), map, (kb0 + kb) * 64, it.z * 128,
                               wfull + 8 * st, pol);
            else
              tma_load_2d(smem_u32(wring + (size_t)st * kWSlot), map, (kb0 + kb) * 64, it.z * 128,
                          wfull + 8 * st);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer (+ activation TMA)
      const uint32_t idesc = idesc_f16_m128((uint32_t)p.bn);
      int wk = 0, bk = 0, n_it = 0;
      for (int s = 0; s < p.n_steps; ++s) {
        for (int i = i0; i < i1; ++i, ++n_it) {
          const int4 it = p.items[i];
          const int acc = n_it & 1;
          const uint32_t aph = (uint32_t)(n_it >> 1) & 1u;
          mbar_wait(accempty + 8 * acc, aph ^ 1u);
          tc_fence_after();
          const int nkb = item_nkb(p, it.x);
          const CUtensorMap* amap = nullptr;
          if (p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 0] = gtimer();
          if (it.x != G_W2) {
            const int tgt = B * (s + 1);
            if (it.x == G_QKV) {
              wait_ge(c.h1 + it.y, tgt);
              amap = &maps.act[0];
            } else if (it.x == G_WO) {
              wait_ge(c.att + it.y * p.NH + 2 * it.w, tgt);
              wait_ge(c.att + it.y * p.NH + 2 * it.w + 1, tgt);
              amap = &maps.act[1];
            } else if (it.x == G_W1) {
              wait_ge(c.h2 + it.y, tgt);
              amap = &maps.act[2];
            } else {
              wait_ge(c.h1 + p.L, tgt);
              amap = &maps.act[3];
            }
            fence_proxy_async_global();
          }
          if (p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 1] = gtimer();
          const int kb0 = it.x == G_LM ? 0 : it.w * 2;
          for (int kb = 0; kb < nkb; ++kb, ++wk, ++bk) {
            const int bs = bk % p.bs;
            const uint32_t bph = (uint32_t)(bk / p.bs) & 1u;
            if (amap) {
              mbar_wait(bempty + 8 * bs, bph ^ 1u);
              mbar_expect_tx(bfull + 8 * bs, (uint32_t)bslot);
              tma_load_2d(smem_u32(bring + (size_t)bs * bslot), amap, (kb0 + kb) * 64, 0, bfull + 8 * bs);
            }
            mbar_wait(bfull + 8 * bs, bph);
            const int st = wk % p.ws;
            mbar_wait(wfull + 8 * st, (uint32_t)(wk / p.ws) & 1u);
            tc_fence_after();
            const uint64_t da = umma_desc_sw128(smem_u32(wring + (size_t)st * kWSlot));
            const uint64_t db = umma_desc_sw128(smem_u32(bring + (size_t)bs * bslot));
#pragma unroll
            for (int k = 0; k < 4; ++k)
              tc_mma_f16(tmem + (uint32_t)(acc * p.bn), da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
            tc_commit(wempty + 8 * st);
            tc_commit(bempty + 8 * bs);
          }
          tc_commit(accfull + 8 * acc);
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ helpers: W2 operands + epilogues
    const int ht = threadIdx.x - 128;  // 0..127 == TMEM lane (warp % 4 quadrant)
    const int row = ht;
    int bk = 0, n_it = 0;
    for (int s = 0; s < p.n_steps; ++s) {
      for (int i = i0; i < i1; ++i, ++n_it) {
        const int4 it = p.items[i];
        const int nkb = item_nkb(p, it.x);
        if (it.x == G_W2) {
          // B operand: f[j][k] = q16(gelu(sum_c' W1 partial[tile=it.w][c'][j][k] + b1)), k < 128
          if (ht == 0) wait_ge(c.w1 + it.y * p.ncf + it.w, p.nck * (s + 1));
          if (ht == 0 && p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 3] = gtimer();
          for (int kb = 0; kb < 2; ++kb) {
            const int bs = (bk + kb) % p.bs;
            const uint32_t bph = (uint32_t)((bk + kb) / p.bs) & 1u;
            if (ht == 0) mbar_wait(bempty + 8 * bs, bph ^ 1u);
          }
          group_bar(2);
          const float* b1 = p.layers[it.y].b1 + it.w * 128;
          for (int u = ht; u < p.bn * 16; u += 128) {
            const int j = u >> 4, q = u & 15;  // row j, 16-byte chunk q of the 128 features
            const int kb = q >> 3, qq = q & 7;
            float acc[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) acc[e] = 0.0f;
            for (int c0 = 0; c0 < p.nck; c0 += 8) {
              float4 lo4[8], hi4[8];
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (c0 + u < p.nck) {
                  const float* src = part_ptr(p.p_w1, it.w, p.nck, c0 + u, p.bn) + (size_t)j * 128 + q * 8;
                  lo4[u] = ldcg4(src);
                  hi4[u] = ldcg4(src + 4);
                }
              }
#pragma unroll
              for (int u = 0; u < 8; ++u) {
                if (c0 + u < p.nck) {
                  acc[0] = __fadd_rn(acc[0], lo4[u].x);
                  acc[1] = __fadd_rn(acc[1], lo4[u].y);
                  acc[2] = __fadd_rn(acc[2], lo4[u].z);
                  acc[3] = __fadd_rn(acc[3], lo4[u].w);
                  acc[4] = __fadd_rn(acc[4], hi4[u].x);
                  acc[5] = __fadd_rn(acc[5], hi4[u].y);
                  acc[6] = __fadd_rn(acc[6], hi4[u].z);
                  acc[7] = __fadd_rn(acc[7], hi4[u].w);
                }
              }
            }
            uint4 packed;
            __half* hp = reinterpret_cast<__half*>(&packed);
#pragma unroll
            for (int e = 0; e < 8; ++e) hp[e] = j < B ? f16_sat(gelu_ref(__fadd_rn(acc[e], b1[q * 8 + e]))) : __float2half_rn(0.0f);
            const int bs = (bk + kb) % p.bs;
            uint8_t* dst = bring + (size_t)bs * bslot + (j >> 3) * 1024 + (j & 7) * 128 + ((qq ^ (j & 7)) * 16);
            *reinterpret_cast<uint4*>(dst) = packed;
          }
          fence_proxy_async_smem();
          group_bar(2);
          if (ht == 0 && p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 4] = gtimer();
          if (ht == 0) {
            mbar_arrive(bfull + 8 * ((bk) % p.bs));
            mbar_arrive(bfull + 8 * ((bk + 1) % p.bs));
          }
        }
        bk += nkb;
        // ---- epilogue
        const int acc = n_it & 1;
        mbar_wait(accfull + 8 * acc, (uint32_t)(n_it >> 1) & 1u);
        tc_fence_after();
        if (ht == 0 && p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 5] = gtimer();
        const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(acc * p.bn);
        float v[16];
        if (it.x != G_LM) {
          float* base = it.x == G_QKV ? p.p_qkv : it.x == G_WO ? p.p_wo : it.x == G_W1 ? p.p_w1 : p.p_w2;
          const int nch = it.x == G_W2 ? p.ncf : p.nck;
          float* dst = part_ptr(base, it.z, nch, it.w, p.bn);
          for (int c0 = 0; c0 < p.bn; c0 += 16) {
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) __stcg(dst + (size_t)(c0 + j) * 128 + row, v[j]);
          }
        } else {
          const int f = it.z * 128 + row;
          for (int c0 = 0; c0 < p.bn; c0 += 16) {
            tmem_ld16(trow + (uint32_t)c0, v);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              unsigned long long k = f < p.V ? argmax_key(q16(v[j]), (uint32_t)f) : 0ull;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) {
                const unsigned long long other = __shfl_xor_sync(0xffffffffu, k, o);
                k = other > k ? other : k;
              }
              if (lane == 0) lm_red[(warp & 3) * 16 + j] = k;
            }
            group_bar(2);
            if (ht < 16 && c0 + ht < B) {
              unsigned long long k = lm_red[ht];
              for (int w = 1; w < 4; ++w) k = lm_red[w * 16 + ht] > k ? lm_red[w * 16 + ht] : k;
              atomicMax(p.keys + c0 + ht, k);
            }
            group_bar(2);
          }
        }
        tc_fence_before();
        __threadfence();
        group_bar(2);
        if (ht == 0) {
          mbar_arrive(accempty + 8 * acc);
          int* ctr = it.x == G_QKV ? c.qkv + it.y * p.nqkv + it.z
                   : it.x == G_WO  ? c.wo + it.y
                   : it.x == G_W1  ? c.w1 + it.y * p.ncf + it.z
                   : it.x == G_W2  ? c.w2 + it.y
                                   : c.lm;
          signal_add(ctr);
          if (p.trace && s == p.trace_step) p.trace[(size_t)i * 8 + 2] = gtimer();
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------ aux group: attention / rows / embed
    const int at = threadIdx.x - 256;
    for (int s = 0; s < p.n_steps; ++s) {
      for (int i = a0; i < a1; ++i) {
        const int4 t = p.aux[i];
        long long* tr = (p.trace && s == p.trace_step && at == 0)
                            ? p.trace + ((size_t)p.item_off[gridDim.x] + i) * 8 : nullptr;
        if (tr) tr[0] = gtimer();
        if (t.x == A_ATT) {
          const int wi = at >> 5;
          if (wi < t.w) {
            const int id = t.z + wi, hh = id / B, bb = id - hh * B;
            long long* ts = (p.trace && s == p.trace_step)
                                ? p.trace + ((size_t)p.item_off[gridDim.x] + i) * 8 : nullptr;
            warp_attention(p, c, t.y, bb, hh, s, aux_sm + 448 + wi * (kAttWarpFloats + p.cap),
                           wi == 0 ? ts : nullptr);
          }
        } else if (t.x == A_R2) {
          if (at == 0) wait_ge(c.wo + t.y, p.nck * p.nck * (s + 1));
          group_bar(1);
          if (tr) tr[1] = gtimer();
          const Layer& ly = p.layers[t.y];
          aux_resid_ln(p, p.p_wo, p.nck, ly.bo, t.z, ly.ln2_g, ly.ln2_b, p.h2, aux_sm + 192);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h2 + t.y);
        } else if (t.x == A_R1) {
          if (at == 0) wait_ge(c.w2 + t.y, p.nck * p.ncf * (s + 1));
          group_bar(1);
          if (tr) tr[1] = gtimer();
          const Layer& ly = p.layers[t.y];
          const bool last = t.y + 1 == p.L;
          aux_resid_ln(p, p.p_w2, p.ncf, ly.b2, t.z, last ? p.fin_g : p.layers[t.y + 1].ln1_g,
                       last ? p.fin_b : p.layers[t.y + 1].ln1_b, last ? p.hf : p.h1, aux_sm + 192);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h1 + t.y + 1);
        } else {  // A_EMB
          if (at == 0) wait_ge(c.lm, p.lm_tiles * s);
          group_bar(1);
          aux_embed(p, t.z, s, aux_sm + 192);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h1);
        }
        if (tr) tr[2] = gtimer();
      }
    }
    // final collect of the last step's argmax (CTA 0) and device state update
    if (blockIdx.x == 0) {
      if (at == 0) wait_ge(c.lm, p.lm_tiles * p.n_steps);
      group_bar(1);
      const int col = *p.step_dev + p.n_steps - 1;
      for (int b = at; b < B; b += 128) {
        const int tok = (int)argmax_id(__ldcg(p.keys + b));
        if (col < p.max_new) p.out_tokens[(size_t)b * p.max_new + col] = tok;
      }
      group_bar(1);
      if (at == 0) {
        *p.step_dev += p.n_steps;
        *p.len_dev += p.n_steps;
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) tmem_dealloc(tmem, ncols);
}

__host__ inline size_t smem_bytes(int ws, int bs, int bn, int cap) {
  return 1024 + (size_t)ws * kWSlot + (size_t)bs * bn * 128 + (2 * ws + 2 * bs + 4) * 8 + 16 +
         (size_t)((448 + 4 * (kAttWarpFloats + cap) + 1) & ~1) * 4 + 64 * 8;
}

}  // namespace mk
}  // namespace tf
