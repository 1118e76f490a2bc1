// Decode GEMM for small batches (sm_100a): narrow feature tiles, whole-K
// operands resident in shared memory, LayerNorm fused into the operand.
//
// Why a second decode GEMM. A decode step (batch <= 64) is a chain of
// dependent launches whose cost is latency, not bandwidth. The split-K kernel
// (gemm_tc.cuh) spreads each weight matrix over ~100 CTAs so each streams a
// few KB, but pays a cluster reduction (~1.5-2 us) on every GEMM and needs
// separate LayerNorm launches in front of QKV and FFN1. Here:
//   * a CTA owns 64 output features (tcgen05 M = 64) over the FULL reduction
//     (or a K/S slice for long K, S <= 4, reduced over DSMEM in split order);
//   * its whole weight slab (nkb x 8 KB) is requested by TMA before
//     griddepcontrol.wait, so it streams (from L2: the previous layer
//     prefetched it, see l2pf) while the predecessor kernel still runs;
//   * after the wait only the activation rows are loaded (all k-blocks at once);
//   * with ln_g set the operand is x and the CTA normalises its bn rows in
//     shared memory (same per-lane chunking and summation order as
//     layernorm_vec_kernel -> bit-identical to the stand-alone LN,
//     tensor.py:153-160), so no LayerNorm launch precedes QKV / FFN1;
//   * the epilogue stages the f16 tile in smem and writes 16-byte chunks
//     (bias, GELU, residual, Q/K/V->cache routing as in gemm_tc.cuh,
//     model.py:464-494 quantisation points).
// TMEM layout of an M = 64 accumulator (probed, tools/m64_probe.cu): row r lives
// in lane (r / 16) * 32 + r % 16, so warp w owns rows 16w .. 16w + 15 in its
// lanes 0..15.
#pragma once

#include "common.cuh"
#include "gemm_tc.cuh"

namespace tf {

constexpr int kDgRows = 64;                   // MMA M (features per CTA)
constexpr int kDgWBytes = kDgRows * kBK * 2;  // one weight k-block: 64 x 64 f16

struct DgArgs {
  int m_tok, n_feat;
  int bn;      // activation rows per CTA (MMA N, multiple of 16, <= 64)
  int nkb;     // K blocks per CTA
  int splits;  // grid.z == cluster.z
  const float* bias;
  __half* out;
  int ldo;
  const __half* resid;  // EPI_BIAS_RESID (may alias out)
  int ldr;
  __half* q_out;  // EPI_QKV routing
  int ldq;
  __half* kc;
  __half* vc;
  int H, NH, D, cap;
  const int* qbase_dev;
  const float* ln_g;  // fused LayerNorm of the operand rows (K == ln_H), or null
  const float* ln_b;
  int ln_H;
  const void* l2pf;  // HBM -> L2 prefetch range (the next layer's copy of this weight)
  unsigned long long l2pf_bytes;
  int trace;
};

__host__ __device__ inline size_t dg_smem_bytes(int bn, int nkb) {
  return 1024 + (size_t)nkb * kDgWBytes + (size_t)nkb * bn * 128 + (size_t)(nkb + 3) * 8 + 16;
}

__device__ __forceinline__ bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts128(uint32_t a, const uint4& v) {
  asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(a), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// In-place LayerNorm of R operand rows (r0, r0 + rstep, ...) held as swizzled
// K-major tiles at `abase` (tile kb at abase + kb * bn * 128). The rows are
// processed together (independent dependency chains); each row's arithmetic
// is exactly layernorm_vec_kernel<NC>'s (lane owns 16-byte chunks lane + 32 i,
// sequential per-lane sums, xor-butterfly warp sums).
template <int NC, int R>
__device__ __forceinline__ void dg_ln_rows(uint32_t abase, int bn, int r0, int rstep, int n_valid, int H,
                                           const float4 (&gv)[NC * 2], const float4 (&bv)[NC * 2], int lane) {
  float xv[R][NC * 8];
  uint32_t addr[R][NC];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = r0 + j * rstep;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int q = lane + 32 * i;
      addr[j][i] = abase + (uint32_t)((q >> 3) * bn * 128 + r * 128 + (((q & 7) ^ (r & 7)) * 16));
      if (r < bn && q * 8 < H) {
        unpack8(lds128(addr[j][i]), &xv[j][8 * i]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[j][8 * i + e] = 0.0f;
      }
    }
  }
  float s[R], mean[R], ss[R], inv[R];
#pragma unroll
  for (int j = 0; j < R; ++j) {
    s[j] = 0.0f;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if ((lane + 32 * i) * 8 < H)
#pragma unroll
        for (int e = 0; e < 8; ++e) s[j] = __fadd_rn(s[j], xv[j][8 * i + e]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int j = 0; j < R; ++j) s[j] += __shfl_xor_sync(0xffffffffu, s[j], o);
#pragma unroll
  for (int j = 0; j < R; ++j) {
    mean[j] = __fdiv_rn(s[j], (float)H);
    ss[j] = 0.0f;
#pragma unroll
    for (int i = 0; i < NC; ++i)
      if ((lane + 32 * i) * 8 < H)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = __fsub_rn(xv[j][8 * i + e], mean[j]);
          ss[j] = __fadd_rn(ss[j], __fmul_rn(d, d));
        }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1)
#pragma unroll
    for (int j = 0; j < R; ++j) ss[j] += __shfl_xor_sync(0xffffffffu, ss[j], o);
#pragma unroll
  for (int j = 0; j < R; ++j) inv[j] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss[j], (float)H), 1e-5f)));
#pragma unroll
  for (int j = 0; j < R; ++j) {
    const int r = r0 + j * rstep;
    if (r >= bn) continue;
    const bool valid = r < n_valid;
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if ((lane + 32 * i) * 8 < H) {
        const float* gf = reinterpret_cast<const float*>(&gv[2 * i]);
        const float* bf = reinterpret_cast<const float*>(&bv[2 * i]);
        float y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e)
          y[e] = valid ? __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[j][8 * i + e], mean[j]), inv[j]), gf[e]), bf[e])
                       : 0.0f;
        sts128(addr[j][i], pack8(y));
      }
    }
  }
}

constexpr int kDgThreads = 256;

// NC: LayerNorm chunks per lane (ceil(H / 256)); 0 = no fused LayerNorm
template <int MODE, int NC>
__global__ void __launch_bounds__(kDgThreads, 1)
    dgemm_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmA, const DgArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int bn = p.bn, nkb = p.nkb;
  uint8_t* wsm = smem;                            // nkb x [64 rows x 128 B]
  uint8_t* asm_ = wsm + (size_t)nkb * kDgWBytes;  // nkb x [bn rows x 128 B]
  uint64_t* bars = reinterpret_cast<uint64_t*>(asm_ + (size_t)nkb * bn * 128);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + nkb + 3);
  // barriers: wbar (all weights), dbar (accumulator), lnbar (unused), abar[kb]
  const uint32_t wbar = smem_u32(bars), dbar = smem_u32(bars + 1), abar0 = smem_u32(bars + 3);
  const uint32_t a_base = smem_u32(asm_), w_base = smem_u32(wsm);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_f = blockIdx.x, tile_b = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * nkb;
  const uint32_t ncols = bn <= 32 ? 32u : (bn <= 64 ? 64u : 128u);
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(p.trace, 0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmA);
    mbar_init(wbar, 1);
    mbar_init(dbar, 1);
    for (int kb = 0; kb < nkb; ++kb) mbar_init(abar0 + 8 * kb, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  // ---- weights: independent of the previous kernel, requested before the wait
  if (threadIdx.x == 0) {
    mbar_expect_tx(wbar, (uint32_t)(nkb * kDgWBytes));
    for (int kb = 0; kb < nkb; ++kb)
      tma_load_2d(w_base + (uint32_t)(kb * kDgWBytes), &tmW, (kb0 + kb) * kBK, tile_f * kDgRows, wbar);
  }
  if (warp == 3 && lane == 0) l2_prefetch_share(p.l2pf, p.l2pf_bytes);
  constexpr int NCL = NC > 0 ? NC : 1;
  float4 gv[NCL * 2], bv[NCL * 2];
  if constexpr (NC > 0) ln_load_gb<NC>(p.ln_H, p.ln_g, p.ln_b, lane, gv, bv);
  // epilogue thread map: warp w owns TMEM rows 16 (w % 4) .. +15 (lanes 0..15),
  // columns [0, bn/2) for w < 4, [bn/2, bn) for w >= 4
  const int row = (warp & 3) * 16 + (lane & 15);
  const int f = tile_f * kDgRows + row;
  const float bias_r = (p.splits == 1 && lane < 16 && f < p.n_feat) ? p.bias[f] : 0.0f;
  pdl_wait();
  if (threadIdx.x == 0) {
    tr.mark(p.trace, 1);
    for (int kb = 0; kb < nkb; ++kb) {
      mbar_expect_tx(abar0 + 8 * kb, (uint32_t)(bn * 128));
      tma_load_2d(a_base + (uint32_t)(kb * bn * 128), &tmA, (kb0 + kb) * kBK, tile_b * bn, abar0 + 8 * kb);
    }
  }
  const int qslot = (MODE == EPI_QKV) ? *p.qbase_dev : 0;
  if constexpr (NC > 0) {
    // LayerNorm needs whole rows: every k-block, then all 8 warps normalise
    // their rows (warp w: rows w, w + 8, ...) in place
    for (int kb = 0; kb < nkb; ++kb) mbar_wait(abar0 + 8 * kb, 0);
    if (threadIdx.x == 0) tr.mark(p.trace, 3);
    const int n_valid = p.m_tok - tile_b * bn;
    for (int r0 = warp; r0 < bn; r0 += 32) dg_ln_rows<NC, 4>(a_base, bn, r0, 8, n_valid, p.ln_H, gv, bv, lane);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) tr.mark(p.trace, 4);
  }
  if (warp == 1) {
    // ---- MMA issue: the whole warp walks the k-blocks (warp-uniform control
    // flow keeps the descriptors in uniform registers), one elected lane issues
    mbar_wait(wbar, 0);
    if (lane == 0) tr.mark(p.trace, 5);
    tc_fence_after();
    const uint32_t idesc = (1u << 4) | (((uint32_t)bn >> 3) << 17) | ((uint32_t)(kDgRows >> 4) << 24);
    const uint64_t da0 = umma_desc_sw128(w_base), db0 = umma_desc_sw128(a_base);
    const uint32_t bstep = (uint32_t)(bn * 128) >> 4;
    for (int kb = 0; kb < nkb; ++kb) {
      if constexpr (NC == 0) {
        mbar_wait(abar0 + 8 * kb, 0);
        tc_fence_after();
      }
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k)
          tc_mma_f16(tmem, da0 + (uint64_t)(kb * (kDgWBytes >> 4) + 2 * k), db0 + (uint64_t)(kb * bstep + 2 * k),
                     idesc, (kb | k) != 0 ? 1u : 0u);
      }
      __syncwarp();
    }
    if (elect_one()) tc_commit(dbar);
    __syncwarp();
  }
  mbar_wait(dbar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) tr.mark(p.trace, 2);
  const uint32_t trow = tmem + ((uint32_t)((warp & 3) * 32) << 16);
  const int half = bn / 2;  // multiple of 8
  const int c_lo = warp < 4 ? 0 : half, c_hi = warp < 4 ? half : bn;

  if (p.splits == 1) {
    // ---- stage q16(epilogue) as f16 [tok][64 features] in the drained operand region
    __half* stile = reinterpret_cast<__half*>(asm_);
    float v[16];
    for (int c = c_lo; c < c_hi; c += 16) {
      tmem_ld16(trow + (uint32_t)c, v);
      if (lane < 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          if (c + j >= c_hi) break;
          float y;
          if constexpr (MODE == EPI_BIAS_GELU) {
            y = gelu_ref(__fadd_rn(v[j], bias_r));
          } else {  // BIAS / QKV / BIAS_RESID (residual added per chunk below)
            y = __fadd_rn(v[j], bias_r);
          }
          stile[(c + j) * kDgRows + row] = f16_sat(y);
        }
      }
    }
    __syncthreads();
    // ---- 16-byte chunks: 8 features of one token
    for (int idx = threadIdx.x; idx < bn * (kDgRows / 8); idx += kDgThreads) {
      const int t = idx >> 3, ch = idx & 7;
      const int tok = tile_b * bn + t;
      const int f0 = tile_f * kDgRows + ch * 8;
      if (tok >= p.m_tok || f0 >= p.n_feat) continue;
      uint4 val = *reinterpret_cast<const uint4*>(stile + t * kDgRows + ch * 8);
      if constexpr (MODE == EPI_BIAS_RESID) {
        float a8[8], r8[8];
        unpack8(val, a8);
        unpack8(*reinterpret_cast<const uint4*>(p.resid + (size_t)tok * p.ldr + f0), r8);
#pragma unroll
        for (int e = 0; e < 8; ++e) a8[e] = __fadd_rn(r8[e], a8[e]);
        val = pack8(a8);
      }
      __half* dst;
      if constexpr (MODE == EPI_QKV) {
        const int which = f0 / p.H, rr = f0 - which * p.H;
        if (which == 0) {
          dst = p.q_out + (size_t)tok * p.ldq + rr;
        } else {
          const int head = rr / p.D, d = rr - head * p.D;
          dst = (which == 1 ? p.kc : p.vc) + (((size_t)tok * p.NH + head) * p.cap + qslot) * p.D + d;
        }
      } else {
        dst = p.out + (size_t)tok * p.ldo + f0;
      }
      *reinterpret_cast<uint4*>(dst) = val;
    }
  } else {
    // ---- split-K over the cluster: park the f32 partial [tok][64] in the
    // drained weight region, then CTA `rank` reduces tokens [rank*tpr, +tpr)
    // from every peer in split order 0..S-1 (deterministic) and stores them.
    float* part = reinterpret_cast<float*>(wsm);
    float v[16];
    for (int c = c_lo; c < c_hi; c += 16) {
      tmem_ld16(trow + (uint32_t)c, v);
      if (lane < 16) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c + j < c_hi) part[(c + j) * kDgRows + row] = v[j];
      }
    }
    const int S = p.splits;
    const uint32_t rank = cluster_ctarank();
    const int tpr = (bn + S - 1) / S;
    const int u_lo = (int)rank * tpr * (kDgRows / 4), u_hi = min(bn, ((int)rank + 1) * tpr) * (kDgRows / 4);
    cluster_arrive();
    // bias / residual of this thread's first unit while the peers finish
    int u = u_lo + (int)threadIdx.x;
    float b4[4] = {0.f, 0.f, 0.f, 0.f}, x4[4] = {0.f, 0.f, 0.f, 0.f};
    auto pre = [&](int uu) {
      const int t = uu >> 4, fq = tile_f * kDgRows + (uu & 15) * 4, tok = tile_b * bn + t;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const bool ok = fq + e < p.n_feat && tok < p.m_tok;
        b4[e] = ok ? p.bias[fq + e] : 0.0f;
        if constexpr (MODE == EPI_BIAS_RESID) x4[e] = ok ? __half2float(p.resid[(size_t)tok * p.ldr + fq + e]) : 0.0f;
      }
    };
    if (u < u_hi) pre(u);
    cluster_wait();
    const uint32_t local = smem_u32(part);
    for (bool first = true; u < u_hi; u += kDgThreads, first = false) {
      if (!first) pre(u);
      float4 pv[4];
#pragma unroll
      for (int sp = 0; sp < 4; ++sp)
        if (sp < S) pv[sp] = ld_dsmem_f32x4(dsmem_addr(local + 16u * (uint32_t)u, (uint32_t)sp));
      float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
      for (int sp = 0; sp < 4; ++sp)
        if (sp < S) {
          acc[0] = __fadd_rn(acc[0], pv[sp].x);
          acc[1] = __fadd_rn(acc[1], pv[sp].y);
          acc[2] = __fadd_rn(acc[2], pv[sp].z);
          acc[3] = __fadd_rn(acc[3], pv[sp].w);
        }
      const int t = u >> 4, fq = tile_f * kDgRows + (u & 15) * 4, tok = tile_b * bn + t;
      if (tok < p.m_tok && fq + 3 < p.n_feat) {
        float y[4];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          if constexpr (MODE == EPI_BIAS_RESID) {
            y[e] = __fadd_rn(x4[e], q16(__fadd_rn(acc[e], b4[e])));
          } else if constexpr (MODE == EPI_BIAS_GELU) {
            y[e] = gelu_ref(__fadd_rn(acc[e], b4[e]));
          } else {
            y[e] = __fadd_rn(acc[e], b4[e]);
          }
        }
        __half2 lo = __halves2half2(f16_sat(y[0]), f16_sat(y[1])), hi = __halves2half2(f16_sat(y[2]), f16_sat(y[3]));
        uint2 w;
        w.x = *reinterpret_cast<uint32_t*>(&lo);
        w.y = *reinterpret_cast<uint32_t*>(&hi);
        *reinterpret_cast<uint2*>(p.out + (size_t)tok * p.ldo + fq) = w;
      }
    }
    cluster_arrive();  // peers may still read this CTA's partial
    cluster_wait();
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tr.mark(p.trace, 7);
    tr.flush(p.trace);
  }
  if (warp == 2) tmem_dealloc(tmem, ncols);
}

}  // namespace tf
