// Persistent decode megakernel (sm_100a): every greedy decode step of a session
// in ONE launch, one CTA per SM, dataflow-synchronised through device counters.
//
// Why: a C2 decode step moves ~420 MB (floor ~65 us at 6.45 TB/s) but is a chain
// of 7 dependent stages per layer x 12 layers; as separate kernels the fixed
// launch/ramp/tail costs dominate. Here weights never wait for data: each CTA's
// weight producer streams its static list of weight tiles through a TMA ring as
// fast as the ring drains, across stage, layer and step boundaries; only the
// small activation operands wait on dependency counters, and attention copies
// its cached K into shared memory before its dependency resolves.
//
// Work items (H % 128 == 0, F % H == 0, head_dim 64, batch <= bn <= 128):
//   GEMM items: 128 output features x H of K (H/64 blocks of 64), swap-AB
//   tcgen05 (weights on MMA-M = 128, batch on MMA-N = bn), f32 accumulator in TMEM.
//     QKV(l, t)     t < 3H/128   B = h1            epilogue: q -> qbuf, k/v -> cache (f16)
//     WO (l, t)     t < H/128    B = attn          epilogue: x = q16(x + q16(acc + bo))
//                                K block kb waits only for head kb's attention
//     W1 (l, t)     t < F/128    B = h2            epilogue: f = q16(gelu(acc + b1))
//     W2 (l, t, c)  c < F/H      B = f[:, cH..]    epilogue: f32 partial [t][b][c][128]
//                                K block waits only for the W1 tile it consumes
//     LM (t)        t < V/128    B = hf            epilogue: fused argmax (atomicMax)
//   aux tasks (4 warps):
//     ATT(l, b, h)  one warp each: K of slots [pad, len) bulk-copied to smem before
//                   the wait; q, new k/v from the QKV epilogue; exact two-pass softmax
//     R2 (l, b)     h2 = LN2(x)
//     R1 (l, b)     x += q16(sum_c W2 partial + b2); h1 = LN1'(x) (next layer / final)
//     EMB(b)        token = argmax key of the previous step; x, h1 = LN1_0(emb)
// Reductions use a fixed order (deterministic). Counters are monotonic within a
// launch (zeroed by the host before it); step s waits for (s + 1) x count.
#pragma once

#include "common.cuh"

namespace tf {
namespace mk {

constexpr int kMaxLayers = 24;
constexpr int kThreads = 384;  // 12 warps: 0 W-TMA, 1 MMA, 2 TMEM, 3 B-TMA, 4-7 epilogue, 8-11 aux
constexpr int kWSlot = 128 * 64 * 2;
constexpr int kAuxFloats = 256;  // per-warp scratch: q, new k, new v (+ pad)

enum GemmType : int { G_QKV = 0, G_WO = 1, G_W1 = 2, G_W2 = 3, G_LM = 4 };
enum AuxType : int { A_ATT = 0, A_R2 = 1, A_R1 = 2, A_EMB = 3 };

struct Layer {
  const float *ln1_g, *ln1_b, *bqkv, *bo, *ln2_g, *ln2_b, *b1, *b2;
};

struct Maps {
  CUtensorMap w[4 * kMaxLayers + 1];  // per layer: qkv, wo, w1, w2; then lm_head
  CUtensorMap act[5];                 // h1, attn, h2, f, hf   (box 64 x bn)
};

struct Params {
  int L, H, F, NH, V, B, bn, cap, n_steps, ws, bs;  // ws/bs: weight / B ring stages
  int nkb, nth, nqkv, nff, nsplit, lm_tiles;        // H/64, H/128, 3H/128, F/128, F/H, V/128
  int att_slots;                                     // K slots per warp held in smem
  const Layer* layers;
  const float *fin_g, *fin_b;
  const __half *tok_emb, *pos_emb;
  int ldw;
  __half *x, *h1, *h2, *attn, *hf, *q, *f;
  int ldx, ldf;
  float* p_w2;
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
  long long* trace;  // optional [items + aux][8] globaltimer stamps of step `trace_step`
  int trace_step;
  int flags;  // bit0: L2 evict_first on weight loads
};

// ---------------------------------------------------------------- counters
struct Ctr {
  int *h1, *qkv, *att, *wo, *h2, *w1, *w2, *lm;
  __device__ Ctr(const Params& p) {
    h1 = p.ctr;
    qkv = h1 + (p.L + 1);
    att = qkv + p.L * p.nqkv;
    wo = att + p.L * p.NH;
    h2 = wo + p.L;
    w1 = h2 + p.L;
    w2 = w1 + p.L * p.nff;
    lm = w2 + p.L;
  }
};
__host__ __device__ inline int ctr_count(int L, int nqkv, int NH, int nff) {
  return (L + 1) + L * nqkv + L * NH + L + L + L * nff + L + 1;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void wait_ge(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  while (ld_acquire(p) < target) __nanosleep(100);
}
__device__ __forceinline__ void signal_add(int* p) {
  __threadfence();
  atomicAdd(p, 1);
}
__device__ __forceinline__ void fence_proxy_async_global() {
  asm volatile("fence.proxy.async.global;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_cta(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void group_bar(int id) {  // named barrier over one 4-warp group
  asm volatile("bar.sync %0, 128;" ::"r"(id) : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* p, uint32_t bytes) {
  if (bytes >= 16)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes & ~15u) : "memory");
}
// contiguous global -> shared bulk copy completing on an mbarrier
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ long long gtimer() {
  long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ const CUtensorMap* item_wmap(const Maps& m, const Params& p, const int4& it) {
  return it.x == G_LM ? &m.w[4 * p.L] : &m.w[4 * it.y + it.x];
}

// ---------------------------------------------------------------- group LayerNorm
// 128 threads; this thread holds v[j] for feature tid + 128 j (j < nf).
constexpr int kVPT = 8;  // H <= 1024
__device__ __forceinline__ void group_ln_row(float (&v)[kVPT], int nf, int H, const float* g, const float* b,
                                             __half* out, float* red) {
  const int tid = threadIdx.x & 127;
  float s = 0.0f;
#pragma unroll
  for (int j = 0; j < kVPT; ++j)
    if (j < nf) s = __fadd_rn(s, v[j]);
  s = warp_sum(s);
  if ((tid & 31) == 0) red[tid >> 5] = s;
  group_bar(1);
  const float mean = __fdiv_rn((red[0] + red[1]) + (red[2] + red[3]), (float)H);
  group_bar(1);
  float ss = 0.0f;
#pragma unroll
  for (int j = 0; j < kVPT; ++j)
    if (j < nf) {
      const float d = __fsub_rn(v[j], mean);
      ss = __fadd_rn(ss, __fmul_rn(d, d));
    }
  ss = warp_sum(ss);
  if ((tid & 31) == 0) red[tid >> 5] = ss;
  group_bar(1);
  const float var = __fdiv_rn((red[0] + red[1]) + (red[2] + red[3]), (float)H);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
  group_bar(1);
#pragma unroll
  for (int j = 0; j < kVPT; ++j) {
    const int c = tid + 128 * j;
    if (j < nf) out[c] = f16_sat(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v[j], mean), inv), g[c]), b[c]));
  }
}

// ---------------------------------------------------------------- attention (one warp)
// sm: [kAuxFloats] scratch + scores [cap] ; kbuf: att_slots x 128 B smem staging.
// Stage 1 (before the dependency): bulk-copy the cached K slots [lo, lo + S)
// into kbuf. Stage 2: wait q/k/v, scores (smem, rest from L2), softmax; then the
// same buffer receives V [lo, lo + S) for P.V.
__device__ void warp_attention(const Params& p, const Ctr& c, int l, int b, int h, int s, float* sm,
                               uint8_t* kbuf, uint32_t bar, uint32_t& phase, long long* ts) {
  const int lane = threadIdx.x & 31;
  auto stamp = [&](int k) {
    if (ts && lane == 0) ts[k] = gtimer();
  };
  constexpr int D = 64;
  const int len = *p.len_dev + s;  // slot of the new token
  const int lo = p.pads[b];
  float* qs = sm;
  float* kn = sm + 64;
  float* vn = sm + 128;
  float* sc = sm + kAuxFloats;
  const size_t head_off = (((size_t)l * p.B + b) * p.NH + h) * (size_t)p.cap * D;
  const __half* K = p.kc + head_off;
  const __half* V = p.vc + head_off;
  const int S = min(len - lo, p.att_slots);  // cached slots staged in smem
  const uint32_t kb_addr = smem_u32(kbuf);
  if (lane == 0) {
    if (S > 0) {
      mbar_expect_tx(bar, (uint32_t)S * D * 2);
      bulk_g2s(kb_addr, K + (size_t)lo * D, (uint32_t)S * D * 2, bar);
    }
    if (len - lo > 0) prefetch_l2(V + (size_t)lo * D, (uint32_t)(len - lo) * D * 2);
    if (len - lo > S) prefetch_l2(K + (size_t)(lo + S) * D, (uint32_t)(len - lo - S) * D * 2);
  }
  const int tq = (h * D) / 128, tk = (p.H + h * D) / 128, tv = (2 * p.H + h * D) / 128;
  if (lane == 0) {
    wait_ge(c.qkv + l * p.nqkv + tq, s + 1);
    wait_ge(c.qkv + l * p.nqkv + tk, s + 1);
    wait_ge(c.qkv + l * p.nqkv + tv, s + 1);
  }
  __syncwarp();
  stamp(1);
  // q from the q buffer; the new k/v from the cache slot the QKV epilogue wrote
  {
    const __half2 q2 = __ldcg(reinterpret_cast<const __half2*>(p.q + (size_t)b * p.ldx + h * D + 2 * lane));
    const __half2 k2 = __ldcg(reinterpret_cast<const __half2*>(K + (size_t)len * D + 2 * lane));
    const __half2 v2 = __ldcg(reinterpret_cast<const __half2*>(V + (size_t)len * D + 2 * lane));
    const float2 qf = __half22float2(q2), kf = __half22float2(k2), vf = __half22float2(v2);
    qs[2 * lane] = qf.x;
    qs[2 * lane + 1] = qf.y;
    kn[2 * lane] = kf.x;
    kn[2 * lane + 1] = kf.y;
    vn[2 * lane] = vf.x;
    vn[2 * lane + 1] = vf.y;
  }
  __syncwarp();
  const int n = len - lo + 1;  // window [lo, len], the new slot last
  const int sub = lane >> 3, gl = lane & 7;
  float qv[8];
#pragma unroll
  for (int e = 0; e < 8; ++e) qv[e] = qs[gl * 8 + e];
  if (S > 0) {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  stamp(3);
  // scores: 8 lanes per key row (16 B each), 4 keys per step
  for (int base = 0; base < n; base += 32) {
    uint4 raw[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      if (j < S) {
        raw[u] = *reinterpret_cast<const uint4*>(kbuf + (size_t)j * 128 + gl * 16);
      } else if (j < n - 1) {
        raw[u] = __ldcg(reinterpret_cast<const uint4*>(K + (size_t)(lo + j) * D + gl * 8));
      } else {
        raw[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      float acc = 0.0f;
      if (j < n - 1) {
        float kf[8];
        unpack8(raw[u], kf);
#pragma unroll
        for (int e = 0; e < 8; ++e) acc = __fadd_rn(acc, __fmul_rn(qv[e], kf[e]));
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
  // V into the same staging buffer (every lane is done with K)
  if (lane == 0 && S > 0) {
    mbar_expect_tx(bar, (uint32_t)S * D * 2);
    bulk_g2s(kb_addr, V + (size_t)lo * D, (uint32_t)S * D * 2, bar);
  }
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
  if (S > 0) {
    mbar_wait(bar, phase);
    phase ^= 1u;
  }
  stamp(5);
  float o[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
  for (int base = 0; base < n; base += 32) {
    uint4 raw[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      if (j < S) {
        raw[u] = *reinterpret_cast<const uint4*>(kbuf + (size_t)j * 128 + gl * 16);
      } else if (j < n - 1) {
        raw[u] = __ldcg(reinterpret_cast<const uint4*>(V + (size_t)(lo + j) * D + gl * 8));
      } else {
        raw[u] = make_uint4(0, 0, 0, 0);
      }
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int j = base + 4 * u + sub;
      if (j < n) {
        const float w = __fmul_rn(sc[j], inv);
        float vf[8];
        if (j < n - 1) {
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
#pragma unroll
  for (int e = 0; e < 8; ++e) {  // combine the 4 key sub-groups (fixed order)
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 8));
    o[e] = __fadd_rn(o[e], __shfl_xor_sync(0xffffffffu, o[e], 16));
  }
  stamp(6);
  if (sub == 0) {
    *reinterpret_cast<uint4*>(p.attn + (size_t)b * p.ldx + h * D + gl * 8) = pack8(o);
    __threadfence();
  }
  __syncwarp();
  if (lane == 0) signal_add(c.att + l * p.NH + h);
  stamp(7);
}

// ---------------------------------------------------------------- row tasks (4 warps)
__device__ void row_ln(const Params& p, int b, const float* g, const float* be, __half* out, float* red,
                       const float* part, const float* bias) {
  const int tid = threadIdx.x & 127;
  const int nf = (p.H - tid + 127) / 128;
  __half* xr = p.x + (size_t)b * p.ldx;
  float v[kVPT];
  __half xo[kVPT];
#pragma unroll
  for (int j = 0; j < kVPT; ++j) xo[j] = j < nf ? __ldcg(xr + tid + 128 * j) : __float2half_rn(0.0f);
  if (part != nullptr) {
    // x += q16(sum_c partial + b2): partial [t][b][c][128], feature tid + 128 j -> tile j
    float pr[kVPT][4];
#pragma unroll
    for (int j = 0; j < kVPT; ++j)
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
        pr[j][cc] = (j < nf && cc < p.nsplit)
                        ? __ldcg(part + (((size_t)j * p.bn + b) * p.nsplit + cc) * 128 + tid) : 0.0f;
#pragma unroll
    for (int j = 0; j < kVPT; ++j) {
      float acc = 0.0f;
#pragma unroll
      for (int cc = 0; cc < 4; ++cc)
        if (cc < p.nsplit) acc = __fadd_rn(acc, pr[j][cc]);
      for (int cc = 4; cc < p.nsplit; ++cc)
        acc = __fadd_rn(acc, __ldcg(part + (((size_t)j * p.bn + b) * p.nsplit + cc) * 128 + tid));
      if (j < nf) {
        const int f = tid + 128 * j;
        const __half xn = f16_sat(__fadd_rn(__half2float(xo[j]), q16(__fadd_rn(acc, bias[f]))));
        xr[f] = xn;
        xo[j] = xn;
      }
    }
  }
#pragma unroll
  for (int j = 0; j < kVPT; ++j) v[j] = __half2float(xo[j]);
  group_ln_row(v, nf, p.H, g, be, out + (size_t)b * p.ldx, red);
}

__device__ void row_embed(const Params& p, int b, int s, float* red) {
  const int tid = threadIdx.x & 127;
  const int nf = (p.H - tid + 127) / 128;
  const int len = *p.len_dev + s;
  const int tok = (int)argmax_id(__ldcg(p.keys + b));
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
    if (j < nf) {
      const __half xn = f16_sat(__fadd_rn(__half2float(p.tok_emb[(size_t)tok * p.ldw + f]),
                                          __half2float(p.pos_emb[(size_t)pos * p.ldw + f])));
      xr[f] = xn;
      v[j] = __half2float(xn);
    }
  }
  group_ln_row(v, nf, p.H, p.layers[0].ln1_g, p.layers[0].ln1_b, p.h1 + (size_t)b * p.ldx, red);
}

// ---------------------------------------------------------------- GEMM epilogue
// this thread: tile row `row` (feature tile*128 + row), columns (tokens) c0 .. c0+15
__device__ __forceinline__ void gemm_epilogue16(const Params& p, const int4& it, int row, int c0,
                                                const float (&v)[16], int s) {
  const int B = p.B;
  const int f = it.z * 128 + row;
  if (it.x == G_QKV) {
    const float bias = p.layers[it.y].bqkv[f];
    const int which = f / p.H, r = f - which * p.H;
    const int head = r >> 6, d = r & 63;
    const int slot = *p.len_dev + s;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tok = c0 + j;
      if (tok >= B) break;
      const __half val = f16_sat(__fadd_rn(v[j], bias));
      if (which == 0) {
        p.q[(size_t)tok * p.ldx + r] = val;
      } else {
        __half* cache = which == 1 ? p.kc : p.vc;
        cache[((((size_t)it.y * B + tok) * p.NH + head) * p.cap + slot) * 64 + d] = val;
      }
    }
  } else if (it.x == G_WO) {
    const float bias = p.layers[it.y].bo[f];
    __half xr[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) xr[j] = (c0 + j < B) ? __ldcg(p.x + (size_t)(c0 + j) * p.ldx + f) : __float2half_rn(0.f);
#pragma unroll
    for (int j = 0; j < 16; ++j)
      if (c0 + j < B)
        p.x[(size_t)(c0 + j) * p.ldx + f] = f16_sat(__fadd_rn(__half2float(xr[j]), q16(__fadd_rn(v[j], bias))));
  } else if (it.x == G_W1) {
    const float bias = p.layers[it.y].b1[f];
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tok = c0 + j;
      if (tok >= B) break;
      p.f[(size_t)tok * p.ldf + f] = f16_sat(gelu_ref(__fadd_rn(v[j], bias)));
    }
  } else {  // G_W2: f32 partial [t][tok][split][128]
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tok = c0 + j;
      if (tok < B) __stcg(p.p_w2 + (((size_t)it.z * p.bn + tok) * p.nsplit + it.w) * 128 + row, v[j]);
    }
  }
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
  uint8_t* kbufs = bring + (size_t)p.bs * bslot;  // 4 x att_slots x 128 B
  uint64_t* bars = reinterpret_cast<uint64_t*>(kbufs + (size_t)4 * p.att_slots * 128);
  // barriers: wfull[ws] wempty[ws] bfull[bs] bempty[bs] accfull[2] accempty[2] att[4]
  const uint32_t wfull = smem_u32(bars), wempty = wfull + 8 * p.ws;
  const uint32_t bfull = wempty + 8 * p.ws, bempty = bfull + 8 * p.bs;
  const uint32_t accfull = bempty + 8 * p.bs, accempty = accfull + 16, attbar = accempty + 16;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * p.ws + 2 * p.bs + 8);
  float* aux_sm = reinterpret_cast<float*>(tmem_slot + 4);  // 4 x (kAuxFloats + cap) + 8
  unsigned long long* lm_red =
      reinterpret_cast<unsigned long long*>(aux_sm + ((4 * (kAuxFloats + p.cap) + 8 + 1) & ~1));

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Ctr c(p);
  const uint32_t ncols = p.bn * 2 <= 32 ? 32 : (p.bn * 2 <= 64 ? 64 : (p.bn * 2 <= 128 ? 128 : 256));
  const bool tracing = p.trace != nullptr;

  if (threadIdx.x == 0) {
    for (int i = 0; i < 4 * p.L + 1; ++i) tma_prefetch_desc(&maps.w[i]);
    for (int i = 0; i < 5; ++i) tma_prefetch_desc(&maps.act[i]);
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
    for (int i = 0; i < 4; ++i) mbar_init(attbar + 8 * i, 1);
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
          const int kb0 = it.x == G_W2 ? it.w * p.nkb : 0;
          for (int kb = 0; kb < p.nkb; ++kb, ++wk) {
            const int st = wk % p.ws;
            const uint32_t ph = (uint32_t)(wk / p.ws) & 1u;
            mbar_wait_sleep(wempty + 8 * st, ph ^ 1u);
            mbar_expect_tx(wfull + 8 * st, kWSlot);
            const uint32_t dst = smem_u32(wring + (size_t)st * kWSlot);
            if (hint)
              tma_load_2d_hint(dst, map, (kb0 + kb) * 64, it.z * 128, wfull + 8 * st, pol);
            else
              tma_load_2d(dst, map, (kb0 + kb) * 64, it.z * 128, wfull + 8 * st);
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ------------------------------------------------ MMA issuer
      const uint32_t idesc = idesc_f16_m128((uint32_t)p.bn);
      int wk = 0, bk = 0, n_it = 0;
      for (int s = 0; s < p.n_steps; ++s) {
        for (int i = i0; i < i1; ++i, ++n_it) {
          const int acc = n_it & 1;
          mbar_wait_sleep(accempty + 8 * acc, ((uint32_t)(n_it >> 1) & 1u) ^ 1u);
          tc_fence_after();
          for (int kb = 0; kb < p.nkb; ++kb, ++wk, ++bk) {
            const int bs = bk % p.bs;
            mbar_wait_sleep(bfull + 8 * bs, (uint32_t)(bk / p.bs) & 1u);
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
  } else if (warp == 3) {
    if (lane == 0) {
      // ------------------------------------------------ activation producer: waits on
      // the dependency counters and streams B k-blocks ahead into the B ring
      int bk = 0;
      for (int s = 0; s < p.n_steps; ++s) {
        for (int i = i0; i < i1; ++i) {
          const int4 it = p.items[i];
          if (tracing && s == p.trace_step) p.trace[(size_t)i * 8 + 0] = gtimer();
          const CUtensorMap* amap;
          int kcol0 = 0;
          if (it.x == G_QKV) {
            wait_ge(c.h1 + it.y, B * (s + 1));
            amap = &maps.act[0];
          } else if (it.x == G_WO) {
            amap = &maps.act[1];
          } else if (it.x == G_W1) {
            wait_ge(c.h2 + it.y, B * (s + 1));
            amap = &maps.act[2];
          } else if (it.x == G_W2) {
            amap = &maps.act[3];
            kcol0 = it.w * p.nkb;
          } else {
            wait_ge(c.h1 + p.L, B * (s + 1));
            amap = &maps.act[4];
          }
          fence_proxy_async_global();
          if (tracing && s == p.trace_step) p.trace[(size_t)i * 8 + 1] = gtimer();
          for (int kb = 0; kb < p.nkb; ++kb, ++bk) {
            // per-K-block dependencies: WO block kb = head kb; W2 block = one W1 tile
            if (it.x == G_WO) {
              wait_ge(c.att + it.y * p.NH + kb, B * (s + 1));
              fence_proxy_async_global();
            } else if (it.x == G_W2 && ((kcol0 + kb) & 1) == 0) {
              wait_ge(c.w1 + it.y * p.nff + ((kcol0 + kb) >> 1), s + 1);
              fence_proxy_async_global();
            }
            const int bs = bk % p.bs;
            mbar_wait_sleep(bempty + 8 * bs, ((uint32_t)(bk / p.bs) & 1u) ^ 1u);
            mbar_expect_tx(bfull + 8 * bs, (uint32_t)bslot);
            tma_load_2d(smem_u32(bring + (size_t)bs * bslot), amap, (kcol0 + kb) * 64, 0, bfull + 8 * bs);
          }
        }
      }
    }
  } else if (warp >= 4 && warp < 8) {
    // ------------------------------------------------ epilogue warps
    const int ht = threadIdx.x - 128;  // == TMEM lane
    int n_it = 0;
    for (int s = 0; s < p.n_steps; ++s) {
      for (int i = i0; i < i1; ++i, ++n_it) {
        const int4 it = p.items[i];
        const int acc = n_it & 1;
        mbar_wait_sleep(accfull + 8 * acc, (uint32_t)(n_it >> 1) & 1u);
        tc_fence_after();
        if (ht == 0 && tracing && s == p.trace_step) p.trace[(size_t)i * 8 + 5] = gtimer();
        const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)(acc * p.bn);
        float v[16];
        if (it.x != G_LM) {
          for (int c0 = 0; c0 < p.bn && c0 < B; c0 += 16) {
            tmem_ld16(trow + (uint32_t)c0, v);
            gemm_epilogue16(p, it, ht, c0, v, s);
          }
        } else {
          const int f = it.z * 128 + ht;
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
          mbar_arrive_cta(accempty + 8 * acc);
          int* ctr = it.x == G_QKV ? c.qkv + it.y * p.nqkv + it.z
                   : it.x == G_WO  ? c.wo + it.y
                   : it.x == G_W1  ? c.w1 + it.y * p.nff + it.z
                   : it.x == G_W2  ? c.w2 + it.y
                                   : c.lm;
          signal_add(ctr);
          if (tracing && s == p.trace_step) p.trace[(size_t)i * 8 + 2] = gtimer();
        }
      }
    }
  } else if (warp >= 8) {
    // ------------------------------------------------ aux group: attention / rows / embed
    const int at = threadIdx.x - 256, aw = at >> 5;
    float* wsm = aux_sm + aw * (kAuxFloats + p.cap);
    float* red = aux_sm + 4 * (kAuxFloats + p.cap);
    uint8_t* kbuf = kbufs + (size_t)aw * p.att_slots * 128;
    uint32_t att_phase = 0;
    for (int s = 0; s < p.n_steps; ++s) {
      for (int i = a0; i < a1; ++i) {
        const int4 t = p.aux[i];
        long long* tr = (tracing && s == p.trace_step) ? p.trace + ((size_t)p.item_off[gridDim.x] + i) * 8 : nullptr;
        if (tr && at == 0) tr[0] = gtimer();
        if (t.x == A_ATT) {
          if (aw < t.w) {
            const int id = t.z + aw, hh = id / B, bb = id - hh * B;
            warp_attention(p, c, t.y, bb, hh, s, wsm, kbuf, attbar + 8 * aw, att_phase,
                           aw == 0 ? tr : nullptr);
          }
        } else if (t.x == A_R2) {
          if (at == 0) wait_ge(c.wo + t.y, p.nth * (s + 1));
          group_bar(1);
          if (tr && at == 0) tr[1] = gtimer();
          const Layer& ly = p.layers[t.y];
          row_ln(p, t.z, ly.ln2_g, ly.ln2_b, p.h2, red, nullptr, nullptr);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h2 + t.y);
        } else if (t.x == A_R1) {
          if (at == 0) wait_ge(c.w2 + t.y, p.nth * p.nsplit * (s + 1));
          group_bar(1);
          if (tr && at == 0) tr[1] = gtimer();
          const Layer& ly = p.layers[t.y];
          const bool last = t.y + 1 == p.L;
          row_ln(p, t.z, last ? p.fin_g : p.layers[t.y + 1].ln1_g, last ? p.fin_b : p.layers[t.y + 1].ln1_b,
                 last ? p.hf : p.h1, red, p.p_w2, ly.b2);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h1 + t.y + 1);
        } else {  // A_EMB
          if (at == 0) wait_ge(c.lm, p.lm_tiles * s);
          group_bar(1);
          row_embed(p, t.z, s, red);
          __threadfence();
          group_bar(1);
          if (at == 0) signal_add(c.h1);
        }
        if (tr && at == 0) tr[2] = gtimer();
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

__host__ inline size_t smem_bytes(int ws, int bs, int bn, int cap, int att_slots) {
  return 1024 + (size_t)ws * kWSlot + (size_t)bs * bn * 128 + (size_t)4 * att_slots * 128 +
         (2 * ws + 2 * bs + 8) * 8 + 16 + (size_t)((4 * (kAuxFloats + cap) + 8 + 1) & ~1) * 4 + 64 * 8;
}

}  // namespace mk
}  // namespace tf
