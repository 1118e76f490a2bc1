// tcgen05 GEMM with fused generation-path epilogues (sm_100a).
//
// Computes C[i][j] = sum_k P[i][k] * Q[j][k] for two K-major f16 operands:
//   prefill (SWAP=false): P = activations [tokens, K], Q = W^T [features, K]
//   decode  (SWAP=true) : P = W^T [features, K],     Q = activations [tokens, K]
// Swap-AB puts the (large) output-feature dimension on MMA-M = 128 and the
// (small) decode batch on MMA-N = 16..256, so one CTA streams a 128-row weight
// slab while the batch rides along in the N dimension.
//
// Structure (one output tile per CTA, 128 threads):
//   warp 0 / lane 0 : TMA producer over a `stages`-deep smem ring (128B swizzle)
//   warp 1 / lane 0 : tcgen05.mma issuer, f32 accumulator in TMEM
//   warp 2          : TMEM allocation owner
//   warps 0-3       : epilogue, tcgen05.ld 32 lanes x 16 columns at a time
// Split-K (grid.z) runs as one thread-block cluster per output tile: the S
// K-slices reduce their f32 partial tiles through distributed shared memory in
// split order 0..S-1 (deterministic, no global round trip). The split count
// depends only on (features, K), never on the batch, so a row's result is
// batch-invariant.
//
// Epilogues implement the reference's f16 quantisation points exactly
// (model.py:465-504): bias is added to the f32
// accumulator, GELU (tanh form) in f32, then saturating RNE to f16; the residual
// add is f32(x) + f32(o) rounded again.
#pragma once

#include "common.cuh"
#include "norm_embed.cuh"

namespace tf {

enum EpiMode : int {
  EPI_F32 = 0,         // raw f32 accumulator store (operator API / tests)
  EPI_BIAS = 1,        // out = q16(acc + b)
  EPI_BIAS_GELU = 2,   // out = q16(gelu(acc + b))
  EPI_BIAS_RESID = 3,  // out = q16(x + q16(acc + b))
  EPI_QKV = 4,         // q16(acc + b) routed to q buffer / K cache / V cache
  EPI_LOGITS = 5,      // q16(acc) stored and/or folded into a per-token argmax key
};

struct GemmArgs {
  int rows_a, rows_b;  // rows of operand P and Q
  int k_blocks;        // number of 64-wide K blocks
  int kb_per_split;    // K blocks per split (grid.z = splits)
  int splits;
  int bn;              // Q rows per tile == MMA N (multiple of 16, <= 256)
  int stages;
  int m_tok, n_feat;   // logical output shape tokens x features
  const float* bias;   // [n_feat] f32 (f16-representable values)
  __half* out;         // [m_tok, ldo] f16
  int ldo;
  float* out_f32;      // EPI_F32 target [m_tok, ldo]
  const __half* resid; // EPI_BIAS_RESID residual [m_tok, ldr] (may alias out)
  int ldr;
  // EPI_QKV routing: features [0,H) -> q_out, [H,2H) -> K cache, [2H,3H) -> V cache
  __half* q_out;
  int ldq;
  __half* kc;  // layer base of [B, NH, cap, D]
  __half* vc;
  int H, NH, D, cap, T;
  const int* qbase_dev;  // cache slot of token t = 0 (device scalar; graph-replayable)
  // EPI_LOGITS
  unsigned long long* keys;  // [m_tok] packed (value, ~id) argmax keys, or null
  // SWAP only: B operand = LayerNorm of x rows computed in-kernel (ln_x != null);
  // token t reads x row t * ln_src_stride + ln_src_off (full ln_H-wide row for the
  // statistics, this CTA's K-slice written into shared memory)
  const __half* ln_x;
  int ln_ldx, ln_src_stride, ln_src_off, ln_H;
  const float* ln_g;
  const float* ln_b;
  int trace;  // diagnostics slot (0 = off)
  int late_trigger;  // release the next kernel only after this kernel's PDL wait
  // decode: activation-independent bytes of a later kernel (the next layer's
  // copy of this weight matrix) streamed HBM -> L2 by this launch's CTAs
  const void* l2pf;
  unsigned long long l2pf_bytes;
  // ln_x set + ln_coop: the LayerNorm of the operand rows is computed
  // cooperatively by the split-K cluster (each CTA loads and normalises only its
  // own K slice; row statistics are exchanged over DSMEM), see ln_coop_build
  int ln_coop;
  // decode EPI_BIAS_RESID with the whole output row in one cluster (grid =
  // cluster = tiles_a x 1 x 2): split-K pair reduction plus the LayerNorm of
  // the new residual rows over DSMEM (gemm_rowln_epilogue); writes out (x) and
  // lnf_h = q16(LN(x)) with lnf_g / lnf_b
  int row_ln;
  // RED_PUSHLN: lnf_cnt[token] counts the features of a row stored so far; the
  // CTA that completes a row normalises it (gemm_ln_tail), writes lnf_h and
  // resets the counter
  int* lnf_cnt;
  const float* lnf_g;
  const float* lnf_b;
  __half* lnf_h;
  int lnf_ldh;
};

constexpr int kTileA = 128;          // MMA M
constexpr int kBK = 64;              // K elements per stage (one 128-B swizzle row)
constexpr int kABytes = kTileA * kBK * 2;

__host__ __device__ inline int gemm_tmem_cols(int bn) {
  return bn <= 32 ? 32 : (bn <= 64 ? 64 : (bn <= 128 ? 128 : 256));
}
__host__ __device__ inline int gemm_stage_bytes(int bn) { return kABytes + bn * kBK * 2; }
// ring bytes: the pipeline stages, or the f32 partial tile of the cluster
// split-K reduction if that is larger (it reuses the drained ring)
// (non-swap tiles also stage the output tile through it: 128 rows x (bn*4 + 16) B)
__host__ __device__ inline size_t gemm_ring_bytes(int bn, int stages, int splits, bool swap) {
  size_t ring = (size_t)stages * gemm_stage_bytes(bn);
  size_t part = splits > 1 ? (size_t)kTileA * bn * 4 : 0;
  size_t out = swap ? 0 : (size_t)kTileA * (bn * 4 + 16);
  ring = ring > part ? ring : part;
  return ring > out ? ring : out;
}
// LN-fused B operand: the normalised K-slice (kb_per_split tiles) plus the TMA
// staging of the full source rows (k_blocks tiles of 64 columns)
__host__ __device__ inline size_t gemm_ln_bytes(int bn, int kb_per_split, int k_blocks) {
  // + gamma / beta of the CTA's K slice (f32)
  return (size_t)(kb_per_split + k_blocks) * bn * kBK * 2 + (size_t)2 * kb_per_split * kBK * 4;
}
// cooperative LN operand: the CTA's K slice of the rows (kb_per_split tiles),
// then f32 scratch: 2 exchange rounds [splits][bn], segment partials
// [bn][ceil(kb_per_split*8/4)], mean / inv [bn] each, gamma / beta of the
// slice [kb_per_split * 64] each
__host__ __device__ inline int gemm_ln_coop_seg(int bn, int kb_per_split) { return bn * ((kb_per_split * 8 + 3) / 4); }
__host__ __device__ inline size_t gemm_ln_coop_bytes(int bn, int kb_per_split, int splits) {
  return (size_t)kb_per_split * bn * kBK * 2 +
         (size_t)(2 * splits * bn + gemm_ln_coop_seg(bn, kb_per_split) + 2 * bn + 2 * kb_per_split * kBK) * 4;
}
// push-based split-K reduction (SWAP, splits > 1, bn <= 128): every CTA owns a
// receive buffer for the S-1 peer slices of its 1/S share of the tile
__host__ __device__ inline bool gemm_push_reduce(int bn, int splits, bool swap) {
  return swap && splits > 1 && bn <= 128;
}
__host__ __device__ inline size_t gemm_recv_bytes(int bn, int splits, bool swap) {
  if (!gemm_push_reduce(bn, splits, swap)) return 0;
  const int U = (kTileA / 4) * bn, per = (U + splits - 1) / splits;
  return (size_t)splits * per * 16;
}
__host__ inline size_t gemm_smem_bytes(int bn, int stages, int splits, bool swap, size_t ln_bytes = 0) {
  return 1024 + gemm_ring_bytes(bn, stages, splits, swap) + ln_bytes + gemm_recv_bytes(bn, splits, swap) +
         (2 * stages + 3) * 8 + 16;
}

// LN-fused B operand: the CTA's bn source rows were staged in smem by TMA
// (k_blocks swizzled 64-column tiles at `stg`). kLnTpr = 8 consecutive threads
// own one row (NT / 8 rows per pass): each sums its 16-byte chunks q = sub,
// sub + 8, ... in order, the 8 partials combine by an xor butterfly (fixed
// order, independent of the batch), two passes (mean; squared deviations,
// tensor.py:153-160); then the CTA's K slice [kb0*64, (kb0+nkb)*64) is
// normalised with gamma / beta staged in smem (gsl / bsl) and written into
// `bln` as nkb swizzled K-major tiles of bn rows.
constexpr int kLnTpr = 8;
template <int NT>
__device__ __forceinline__ void ln_build_b(const GemmArgs& p, int tile_b, int kb0, int nkb, uint8_t* bln,
                                           const uint8_t* stg, const float* gsl, const float* bsl) {
  const int bn = p.bn, H = p.ln_H, C = H / 8;
  const int tid = threadIdx.x, sub = tid % kLnTpr;
  const float Hf = (float)H;
  for (int r0 = 0; r0 < bn; r0 += NT / kLnTpr) {
    const int r = r0 + tid / kLnTpr;
    const bool rv = r < bn;
    const int rr = rv ? r : 0;
    auto chunk = [&](int q) {
      return *reinterpret_cast<const uint4*>(stg + (size_t)(q >> 3) * bn * 128 + rr * 128 + (((q & 7) ^ (rr & 7)) * 16));
    };
    float s = 0.0f;
    if (rv)
      for (int q = sub; q < C; q += kLnTpr) {
        float xv[8];
        unpack8(chunk(q), xv);
#pragma unroll
        for (int e = 0; e < 8; ++e) s = __fadd_rn(s, xv[e]);
      }
#pragma unroll
    for (int o = kLnTpr / 2; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
    const float mean = __fdiv_rn(s, Hf);
    float ss = 0.0f;
    if (rv)
      for (int q = sub; q < C; q += kLnTpr) {
        float xv[8];
        unpack8(chunk(q), xv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float d = __fsub_rn(xv[e], mean);
          ss = __fadd_rn(ss, __fmul_rn(d, d));
        }
      }
#pragma unroll
    for (int o = kLnTpr / 2; o > 0; o >>= 1) ss = __fadd_rn(ss, __shfl_xor_sync(0xffffffffu, ss, o));
    const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, Hf), 1e-5f)));
    if (rv) {
      const bool valid = tile_b * bn + r < p.m_tok;
      for (int q = kb0 * 8 + sub; q < (kb0 + nkb) * 8; q += kLnTpr) {
        float xv[8], y[8];
        unpack8(chunk(q), xv);
        const int f0 = (q - kb0 * 8) * 8;
#pragma unroll
        for (int e = 0; e < 8; ++e)
          y[e] = (valid && q * 8 + e < H) ? __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[e], mean), inv), gsl[f0 + e]), bsl[f0 + e])
                                          : 0.0f;
        uint8_t* dst = bln + (size_t)(q / 8 - kb0) * bn * kBK * 2 + r * 128 + (((q & 7) ^ (r & 7)) * 16);
        *reinterpret_cast<uint4*>(dst) = pack8(y);
      }
    }
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// elect.sync over the full warp (lane 0 when every lane is active)
__device__ __forceinline__ bool elect_lane0() {
  uint32_t pred = 0;
  asm volatile(
      "{\n\t.reg .pred p;\n\t.reg .b32 r;\n\telect.sync r|p, 0xffffffff;\n\tselp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(pred));
  return pred != 0;
}

template <int MODE, bool SWAP>
__device__ __forceinline__ void epi_store(const GemmArgs& p, int tok, int f, float acc) {
  if constexpr (MODE == EPI_F32) {
    p.out_f32[(size_t)tok * p.ldo + f] = acc;
  } else if constexpr (MODE == EPI_BIAS) {
    p.out[(size_t)tok * p.ldo + f] = f16_sat(__fadd_rn(acc, p.bias[f]));
  } else if constexpr (MODE == EPI_BIAS_GELU) {
    p.out[(size_t)tok * p.ldo + f] = f16_sat(gelu_ref(__fadd_rn(acc, p.bias[f])));
  } else if constexpr (MODE == EPI_BIAS_RESID) {
    float o = q16(__fadd_rn(acc, p.bias[f]));
    float x = __half2float(p.resid[(size_t)tok * p.ldr + f]);
    p.out[(size_t)tok * p.ldo + f] = f16_sat(__fadd_rn(x, o));
  } else if constexpr (MODE == EPI_QKV) {
    __half val = f16_sat(__fadd_rn(acc, p.bias[f]));
    int which = f / p.H;
    int r = f - which * p.H;
    if (which == 0) {
      p.q_out[(size_t)tok * p.ldq + r] = val;
    } else {
      int b = tok / p.T, t = tok - b * p.T;
      int head = r / p.D, d = r - head * p.D;
      int slot = *p.qbase_dev + t;
      size_t idx = (((size_t)b * p.NH + head) * p.cap + slot) * p.D + d;
      (which == 1 ? p.kc : p.vc)[idx] = val;
    }
  } else if constexpr (MODE == EPI_LOGITS) {
    if (p.out) p.out[(size_t)tok * p.ldo + f] = f16_sat(acc);
  }
}

// Epilogue for one 16-column chunk held by this thread (A-tile row `ra`,
// Q rows qb .. qb+15). For EPI_LOGITS with SWAP the argmax over the CTA's 128
// features is reduced warp -> CTA -> one atomicMax per token.
template <int MODE, bool SWAP>
__device__ __forceinline__ void epi_chunk(const GemmArgs& p, int ra, int qb, const float (&v)[16],
                                          unsigned long long* red) {
  if constexpr (!SWAP) {
    const int tok = ra;
    if (tok < p.m_tok) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int f = qb + j;
        if (f < p.n_feat) epi_store<MODE, SWAP>(p, tok, f, v[j]);
      }
    }
    if constexpr (MODE == EPI_LOGITS) {
      if (p.keys != nullptr && tok < p.m_tok) {
        unsigned long long best = 0;
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int f = qb + j;
          if (f < p.n_feat) {
            unsigned long long k = argmax_key(q16(v[j]), (uint32_t)f);
            best = k > best ? k : best;
          }
        }
        atomicMax(&p.keys[tok], best);
      }
    }
  } else {
    const int f = ra;
    const bool fok = f < p.n_feat;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tok = qb + j;
      if (fok && tok < p.m_tok) epi_store<MODE, SWAP>(p, tok, f, v[j]);
    }
    if constexpr (MODE == EPI_LOGITS) {
      if (p.keys != nullptr) {
        // keys of this 16-token chunk staged in smem (the drained ring) as
        // [16][129] u64; each token column is then reduced by 8 threads over
        // 16 rows each + 3 shuffle rounds, and one atomicMax per token
        unsigned long long* kred = reinterpret_cast<unsigned long long*>(red);
        const int row = threadIdx.x;
#pragma unroll
        for (int j = 0; j < 16; ++j)
          kred[j * 129 + row] = fok ? argmax_key(q16(v[j]), (uint32_t)f) : 0ull;
        __syncthreads();
        const int j = threadIdx.x >> 3, part = threadIdx.x & 7;
        unsigned long long best = 0ull;
#pragma unroll
        for (int r = 0; r < 16; ++r) {
          const unsigned long long k = kred[j * 129 + part * 16 + r];
          best = k > best ? k : best;
        }
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
          const unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
          best = other > best ? other : best;
        }
        const int tok = qb + j;
        if (part == 0 && tok < p.m_tok) atomicMax(&p.keys[tok], best);
        __syncthreads();
      }
    }
  }
}

// Full-K swap tile (RED_ONE, thread = output feature f, TMEM columns = tokens):
// the per-feature terms (bias, Q/K/V routing, cache slot) are loaded once per
// thread instead of once per element -- per-element loads cannot be hoisted
// past the stores (possible aliasing), so epi_store's form serialises a global
// load round trip per element (C4 QKV epilogue 17 us -> ~1 us). Same math.
template <int MODE>
// 16-column chunks c0, c0 + cstep, ... (two warps per TMEM lane quadrant split them)
__device__ __forceinline__ void epi_swap_one(const GemmArgs& p, int f, int tok0, int bn, uint32_t trow, int c0,
                                             int cstep) {
  const bool fok = f < p.n_feat;
  const float bf = fok ? p.bias[f] : 0.0f;
  __half* dst = nullptr;
  size_t stride = 0, tstride = 0;
  int T = 1;
  if constexpr (MODE == EPI_QKV) {
    const int which = fok ? f / p.H : 0, r = f - which * p.H;
    if (which == 0) {
      dst = p.q_out + r;
      stride = p.ldq;
    } else {
      const int head = r / p.D, d = r - head * p.D;
      dst = (which == 1 ? p.kc : p.vc) + ((size_t)head * p.cap + *p.qbase_dev) * p.D + d;
      stride = (size_t)p.NH * p.cap * p.D;
      tstride = p.D;
      T = p.T;
    }
  } else {
    dst = p.out + f;
    stride = p.ldo;
  }
  for (int c = c0; c < bn; c += cstep) {
    float v[16];
    tmem_ld16(trow + (uint32_t)c, v);
    float x[16];
    if constexpr (MODE == EPI_BIAS_RESID) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int tok = tok0 + c + j;
        x[j] = fok && tok < p.m_tok ? __half2float(p.resid[(size_t)tok * p.ldr + f]) : 0.0f;
      }
    }
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int tok = tok0 + c + j;
      if (fok && tok < p.m_tok) {
        const float a = __fadd_rn(v[j], bf);
        __half o;
        if constexpr (MODE == EPI_BIAS_GELU) {
          o = f16_sat(gelu_ref(a));
        } else if constexpr (MODE == EPI_BIAS_RESID) {
          o = f16_sat(__fadd_rn(x[j], q16(a)));
        } else {
          o = f16_sat(a);
        }
        const int b = T == 1 ? tok : tok / T;
        dst[(size_t)b * stride + (size_t)(tok - b * T) * tstride] = o;
      }
    }
  }
}

// ---------------------------------------------------------------- non-swap (prefill) epilogue
// Thread = output row, so direct stores would hit 32 rows per warp instruction.
// Instead the tile is staged through the drained ring (row pitch padded by 16 B)
// after the per-element math, then written out cooperatively: each thread moves
// 16-byte chunks of one row (8 f16 / 4 f32), consecutive threads consecutive
// chunks, with the residual read and the Q/K/V routing done per chunk.
// NAMED: run by the 4 epilogue warps of the persistent prefill kernel (named
// barrier 1 instead of __syncthreads); `row` = this thread's TMEM lane / tile
// row (a bijection over 0..127); `tmem_free` (mbarrier, or 0) is arrived once
// every TMEM read of the tile is done, so the MMA warp can refill the buffer
// while the stores drain.
// NT = 256: eight warps; warps w and w + 4 share TMEM lane quadrant w % 4 and
// split the tile's columns in halves (the phase-1 TMEM reads and math are
// latency-bound with one warp per scheduler).
template <int MODE, bool NAMED = false, int NT = 128>
__device__ __forceinline__ void epi_tile_nonswap(const GemmArgs& p, int tile_a, int tile_b, uint32_t trow,
                                                 uint8_t* stage, int row_ = -1, uint32_t tmem_free = 0) {
  auto esync = [] {
    if constexpr (NAMED)
      asm volatile("bar.sync 1, 128;" ::: "memory");
    else
      __syncthreads();
  };
  constexpr bool F32OUT = MODE == EPI_F32;
  constexpr int ESZ = F32OUT ? 4 : 2;
  const int bn = p.bn;
  const int pitch = bn * ESZ + 16;
  const int et = row_ >= 0 ? row_ : (int)threadIdx.x;  // linear epilogue thread id, 0 .. NT-1
  const int row = NT == 256 ? (int)(((threadIdx.x >> 5) & 3) * 32 + (threadIdx.x & 31)) : et;
  const int c_begin = NT == 256 ? (int)(threadIdx.x >> 7) * (p.bn / 2) : 0;
  const int c_end = NT == 256 ? c_begin + p.bn / 2 : p.bn;
  const int tok = tile_a * kTileA + row;
  // the tile's bias columns, loaded once (not one dependent load per element)
  __shared__ float s_bias[256];
  if constexpr (MODE != EPI_F32 && MODE != EPI_LOGITS) {
    for (int c = et; c < bn; c += NT) s_bias[c] = p.bias[min(tile_b * bn + c, p.n_feat - 1)];
    esync();
  } else if constexpr (NAMED) {
    esync();  // persistent loop: the previous tile's stores have drained the staging buffer
  }
  float v[16];
  for (int c = c_begin; c < c_end; c += 16) {
    tmem_ld16(trow + (uint32_t)c, v);
    uint8_t* dst = stage + (size_t)row * pitch + (size_t)c * ESZ;
    if constexpr (F32OUT) {
#pragma unroll
      for (int q = 0; q < 4; ++q)
        *reinterpret_cast<float4*>(dst + 16 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    } else {
      float y[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        if constexpr (MODE == EPI_BIAS || MODE == EPI_QKV) {
          y[j] = __fadd_rn(v[j], s_bias[c + j]);
        } else if constexpr (MODE == EPI_BIAS_GELU) {
          y[j] = gelu_ref(__fadd_rn(v[j], s_bias[c + j]));
        } else if constexpr (MODE == EPI_BIAS_RESID) {
          y[j] = __fadd_rn(v[j], s_bias[c + j]);  // rounded to f16 here, residual added below
        } else {  // EPI_LOGITS
          y[j] = v[j];
        }
      }
      *reinterpret_cast<uint4*>(dst) = pack8(y);
      *reinterpret_cast<uint4*>(dst + 16) = pack8(y + 8);
    }
  }
  if (tmem_free) tc_fence_before();
  esync();
  if (tmem_free && row == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(tmem_free) : "memory");
  const int cpr = bn * ESZ / 16;  // 16-byte chunks per row
  const int epc = 16 / ESZ;       // elements per chunk
  if constexpr (MODE == EPI_BIAS_RESID) {
    // residual chunks are loaded 8 at a time before use (one exposed global
    // latency per 8 chunks instead of per chunk)
    constexpr int BATCH = 8;
    for (int base = et; base < kTileA * cpr; base += NT * BATCH) {
      uint4 rv[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int idx = base + u * NT;
        const int r = idx / cpr, ch = idx - r * cpr;
        const int t = tile_a * kTileA + r, f0 = tile_b * bn + ch * 8;
        const bool fast = idx < kTileA * cpr && t < p.m_tok && f0 + 8 <= p.n_feat && (p.ldr % 8) == 0;
        rv[u] = fast ? *reinterpret_cast<const uint4*>(p.resid + (size_t)t * p.ldr + f0) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int idx = base + u * NT;
        if (idx >= kTileA * cpr) break;
        const int r = idx / cpr, ch = idx - r * cpr;
        const int t = tile_a * kTileA + r, f0 = tile_b * bn + ch * 8;
        if (t >= p.m_tok || f0 >= p.n_feat) continue;
        const uint4 val = *reinterpret_cast<const uint4*>(stage + (size_t)r * pitch + ch * 16);
        const bool full = f0 + 8 <= p.n_feat;
        float a8[8], r8[8];
        unpack8(val, a8);
        if (full && (p.ldr % 8) == 0) {
          unpack8(rv[u], r8);
        } else {
          const __half* rp = p.resid + (size_t)t * p.ldr + f0;
#pragma unroll
          for (int e = 0; e < 8; ++e) r8[e] = f0 + e < p.n_feat ? __half2float(rp[e]) : 0.0f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) a8[e] = __fadd_rn(r8[e], a8[e]);
        const uint4 res = pack8(a8);
        __half* o = p.out + (size_t)t * p.ldo + f0;
        if (full && (p.ldo % 8) == 0) {
          *reinterpret_cast<uint4*>(o) = res;
        } else {
          const __half* hv = reinterpret_cast<const __half*>(&res);
          for (int e = 0; e < 8 && f0 + e < p.n_feat; ++e) o[e] = hv[e];
        }
      }
    }
    return;
  }
  if constexpr (MODE == EPI_QKV) {
    // the thread's chunk column is fixed (NT is a multiple of the chunks per
    // row), so the q/k/v routing of its 8 features is computed once
    if (NT % cpr == 0 && (p.D % 8) == 0 && (p.ldq % 8) == 0) {
      const int ch = et % cpr, f0 = tile_b * bn + ch * 8;
      if (f0 + 8 > p.n_feat) return;
      const int which = f0 / p.H, rr = f0 - which * p.H;
      const int head = rr / p.D, d = rr - head * p.D;
      const int qb = *p.qbase_dev;
      __half* const cache = which == 1 ? p.kc : p.vc;
      for (int r = et / cpr; r < kTileA; r += NT / cpr) {
        const int t = tile_a * kTileA + r;
        if (t >= p.m_tok) break;
        const uint4 val = *reinterpret_cast<const uint4*>(stage + (size_t)r * pitch + ch * 16);
        __half* dst;
        if (which == 0) {
          dst = p.q_out + (size_t)t * p.ldq + rr;
        } else {
          const int b = t / p.T, tt = t - b * p.T;
          dst = cache + (((size_t)b * p.NH + head) * p.cap + qb + tt) * p.D + d;
        }
        *reinterpret_cast<uint4*>(dst) = val;
      }
      return;
    }
  }
  for (int idx = et; idx < kTileA * cpr; idx += NT) {
    const int r = idx / cpr, ch = idx - r * cpr;
    const int t = tile_a * kTileA + r;
    const int f0 = tile_b * bn + ch * epc;
    if (t >= p.m_tok || f0 >= p.n_feat) continue;
    const uint4 val = *reinterpret_cast<const uint4*>(stage + (size_t)r * pitch + ch * 16);
    const bool full = f0 + epc <= p.n_feat;
    if constexpr (F32OUT) {
      float* o = p.out_f32 + (size_t)t * p.ldo + f0;
      const float* fv = reinterpret_cast<const float*>(&val);
      if (full && (p.ldo % 4) == 0) {
        *reinterpret_cast<uint4*>(o) = val;
      } else {
        for (int e = 0; e < epc && f0 + e < p.n_feat; ++e) o[e] = fv[e];
      }
    } else if constexpr (MODE == EPI_QKV) {
      // 8 features never straddle a head (head_dim % 8 == 0) or a q/k/v boundary
      const int which = f0 / p.H, rr = f0 - which * p.H;
      __half* dst;
      if (which == 0) {
        dst = p.q_out + (size_t)t * p.ldq + rr;
      } else {
        const int b = t / p.T, tt = t - b * p.T;
        const int head = rr / p.D, d = rr - head * p.D;
        const int slot = *p.qbase_dev + tt;
        dst = (which == 1 ? p.kc : p.vc) + (((size_t)b * p.NH + head) * p.cap + slot) * p.D + d;
      }
      if (full && (p.D % 8) == 0 && (p.ldq % 8) == 0) {
        *reinterpret_cast<uint4*>(dst) = val;
      } else {
        const __half* hv = reinterpret_cast<const __half*>(&val);
        for (int e = 0; e < epc && f0 + e < p.n_feat; ++e) {
          const int fe = f0 + e, w2 = fe / p.H, r2 = fe - w2 * p.H;
          if (w2 == 0) {
            p.q_out[(size_t)t * p.ldq + r2] = hv[e];
          } else {
            const int b = t / p.T, tt = t - b * p.T;
            const int head = r2 / p.D, d = r2 - head * p.D;
            (w2 == 1 ? p.kc : p.vc)[(((size_t)b * p.NH + head) * p.cap + *p.qbase_dev + tt) * p.D + d] = hv[e];
          }
        }
      }
    } else {
      __half* o = p.out + (size_t)t * p.ldo + f0;
      uint4 res = val;
      if constexpr (MODE == EPI_BIAS_RESID) {
        const __half* rp = p.resid + (size_t)t * p.ldr + f0;
        float a8[8], r8[8];
        unpack8(val, a8);
        if (full && (p.ldr % 8) == 0) {
          unpack8(*reinterpret_cast<const uint4*>(rp), r8);
        } else {
#pragma unroll
          for (int e = 0; e < 8; ++e) r8[e] = f0 + e < p.n_feat ? __half2float(rp[e]) : 0.0f;
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) a8[e] = __fadd_rn(r8[e], a8[e]);
        res = pack8(a8);
      }
      if (full && (p.ldo % 8) == 0) {
        *reinterpret_cast<uint4*>(o) = res;
      } else {
        const __half* hv = reinterpret_cast<const __half*>(&res);
        for (int e = 0; e < epc && f0 + e < p.n_feat; ++e) o[e] = hv[e];
      }
    }
  }
}

// ---- split-K reduction epilogue, 4 rows of one tile column per unit.
// Unit u of tile (tile_a, tile_b): column u / 32, rows 4 * (u % 32) .. +3.
// SWAP: rows are features, the column is a token; otherwise the reverse.
struct EpiPre4 {
  float b[4];  // bias
  float x[4];  // residual
};

template <bool SWAP>
__device__ __forceinline__ void unit_coords(int tile_a, int tile_b, int bn, int u, int& tok, int& f, int& step) {
  const int col = tile_b * bn + u / 32, r = tile_a * kTileA + (u % 32) * 4;
  tok = SWAP ? col : r;
  f = SWAP ? r : col;
  step = SWAP ? 1 : 0;  // the 4 rows advance the feature (SWAP) or the token
}

template <int MODE, bool SWAP>
__device__ __forceinline__ void epi_pre4(const GemmArgs& p, int tile_a, int tile_b, int u, EpiPre4& q) {
  int tok, f, st;
  unit_coords<SWAP>(tile_a, tile_b, p.bn, u, tok, f, st);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int tj = tok + (st ? 0 : j), fj = f + (st ? j : 0);
    const bool ok = tj < p.m_tok && fj < p.n_feat;
    if constexpr (MODE == EPI_BIAS || MODE == EPI_BIAS_GELU || MODE == EPI_BIAS_RESID || MODE == EPI_QKV)
      q.b[j] = ok ? p.bias[fj] : 0.0f;
    if constexpr (MODE == EPI_BIAS_RESID)
      q.x[j] = ok ? __half2float(p.resid[(size_t)tj * p.ldr + fj]) : 0.0f;
  }
}

template <int MODE, bool SWAP>
__device__ __forceinline__ void epi_fin4(const GemmArgs& p, int tile_a, int tile_b, int u, const float (&acc)[4],
                                         const EpiPre4& q, int qslot) {
  int tok, f, st;
  unit_coords<SWAP>(tile_a, tile_b, p.bn, u, tok, f, st);
  if constexpr (MODE == EPI_F32) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tj = tok + (st ? 0 : j), fj = f + (st ? j : 0);
      if (tj < p.m_tok && fj < p.n_feat) p.out_f32[(size_t)tj * p.ldo + fj] = acc[j];
    }
    return;
  }
  __half val[4];
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    if constexpr (MODE == EPI_BIAS || MODE == EPI_QKV) {
      val[j] = f16_sat(__fadd_rn(acc[j], q.b[j]));
    } else if constexpr (MODE == EPI_BIAS_GELU) {
      val[j] = f16_sat(gelu_ref(__fadd_rn(acc[j], q.b[j])));
    } else if constexpr (MODE == EPI_BIAS_RESID) {
      val[j] = f16_sat(__fadd_rn(q.x[j], q16(__fadd_rn(acc[j], q.b[j]))));
    } else {
      val[j] = f16_sat(acc[j]);
    }
  }
  // destination of the 4 values: contiguous when they run along features
  __half* dst = nullptr;
  if constexpr (MODE == EPI_QKV) {
    if (st && tok < p.m_tok && f + 3 < p.n_feat && p.H % 4 == 0 && p.D % 4 == 0) {
      const int which = f / p.H, r = f - which * p.H;
      if (which == 0) {
        dst = p.q_out + (size_t)tok * p.ldq + r;
      } else {
        const int b = tok / p.T, t = tok - b * p.T;
        const int head = r / p.D, d = r - head * p.D;
        const int slot = qslot + t;
        dst = (which == 1 ? p.kc : p.vc) + (((size_t)b * p.NH + head) * p.cap + slot) * p.D + d;
      }
    }
  } else {
    if (st && tok < p.m_tok && f + 3 < p.n_feat && p.out) dst = p.out + (size_t)tok * p.ldo + f;
  }
  if (dst != nullptr && (reinterpret_cast<uintptr_t>(dst) & 7u) == 0) {
    __half2 lo = __halves2half2(val[0], val[1]), hi = __halves2half2(val[2], val[3]);
    uint2 w;
    w.x = *reinterpret_cast<uint32_t*>(&lo);
    w.y = *reinterpret_cast<uint32_t*>(&hi);
    *reinterpret_cast<uint2*>(dst) = w;
    return;
  }
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int tj = tok + (st ? 0 : j), fj = f + (st ? j : 0);
    if (tj >= p.m_tok || fj >= p.n_feat) continue;
    if constexpr (MODE == EPI_QKV) {
      const int which = fj / p.H, r = fj - which * p.H;
      if (which == 0) {
        p.q_out[(size_t)tj * p.ldq + r] = val[j];
      } else {
        const int b = tj / p.T, t = tj - b * p.T;
        const int head = r / p.D, d = r - head * p.D;
        const int slot = qslot + t;
        (which == 1 ? p.kc : p.vc)[(((size_t)b * p.NH + head) * p.cap + slot) * p.D + d] = val[j];
      }
    } else if (p.out) {
      p.out[(size_t)tj * p.ldo + fj] = val[j];
    }
  }
}

__device__ __forceinline__ void st_dsmem_f32(uint32_t addr, float v) {
  asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// Cooperative LayerNorm of the B operand across the split-K cluster. The CTA
// holds its K slice [kb0*64, (kb0+nkb)*64) of bn rows as swizzled tiles at
// `bln`; the S CTAs of the cluster together hold the whole rows. Two exchange
// rounds (row sums, then sums of squared deviations from the mean), each a
// per-CTA partial written into every peer's `red` slot [rank][row] over DSMEM
// and summed in rank order after a cluster barrier (deterministic), give the
// reference's two-pass statistics (tensor.py:153-160: mean; c = x - mean;
// var = mean(c*c); c * (1/sqrt(var + 1e-5)) * g + b); the CTA then normalises
// its slice in place (f16, rows past m_tok zero). Cluster-barrier protocol on
// entry: with `pending_arrive` the caller has already arrived once (push
// reduction); on exit with `rearm` one arrive is left pending for the caller.
__device__ __forceinline__ void ln_coop_build(const GemmArgs& p, int tile_b, int nkb, uint8_t* bln, float* sc,
                                              bool pending_arrive, bool rearm) {
  const int bn = p.bn, S = p.splits, tid = threadIdx.x;
  const float H = (float)p.ln_H;
  float* red0 = sc;                   // [S][bn]
  float* red1 = red0 + S * bn;        // [S][bn]
  float* seg = red1 + S * bn;         // [bn][nsr]
  float* mean_s = seg + bn * ((nkb * 8 + 3) / 4);  // [bn]
  float* inv_s = mean_s + bn;         // [bn]
  const float* g_s = inv_s + bn;      // [nkb*64] gamma of the slice (staged by the caller)
  const float* b_s = g_s + nkb * kBK;  // [nkb*64]
  const uint32_t rank = S > 1 ? cluster_ctarank() : 0u;
  const int C = nkb * 8;  // 16-byte chunks of one row in this slice
  auto chunk_addr = [&](int r, int c) {
    return bln + (size_t)(c >> 3) * bn * 128 + r * 128 + ((((c & 7) ^ (r & 7))) * 16);
  };
  // per-(row, segment) partials over fixed 4-chunk (32-feature) segments, then
  // the per-row total in segment order (independent of bn: batch-invariant),
  // then one write per peer
  const int nsr = (C + 3) / 4;
  auto round = [&](float* red, bool second) {
    for (int idx = tid; idx < bn * nsr; idx += 128) {
      const int r = idx / nsr, sg = idx - r * nsr;
      const float m = second ? mean_s[r] : 0.0f;
      float acc = 0.0f;
      for (int c = 4 * sg; c < min(C, 4 * sg + 4); ++c) {
        float xv[8];
        unpack8(*reinterpret_cast<const uint4*>(chunk_addr(r, c)), xv);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (second) {
            const float d = __fsub_rn(xv[e], m);
            acc = __fadd_rn(acc, __fmul_rn(d, d));
          } else {
            acc = __fadd_rn(acc, xv[e]);
          }
        }
      }
      seg[idx] = acc;
    }
    __syncthreads();
    for (int r = tid; r < bn; r += 128) {
      float tot = 0.0f;
      for (int sg = 0; sg < nsr; ++sg) tot = __fadd_rn(tot, seg[r * nsr + sg]);
      if (S > 1) {
        const uint32_t a = smem_u32(red + (int)rank * bn + r);
        for (int pr = 0; pr < S; ++pr) st_dsmem_f32(dsmem_addr(a, (uint32_t)pr), tot);
      } else {
        red[r] = tot;
      }
    }
    __syncthreads();
  };
  if (S > 1) {
    if (!pending_arrive) cluster_arrive_relaxed();
    cluster_wait();  // every peer is running before its smem is written
  }
  round(red0, false);
  if (S > 1) {
    cluster_arrive();
    cluster_wait();
  }
  for (int r = tid; r < bn; r += 128) {
    float s = 0.0f;
    for (int pr = 0; pr < S; ++pr) s = __fadd_rn(s, red0[pr * bn + r]);
    mean_s[r] = __fdiv_rn(s, H);
  }
  __syncthreads();
  round(red1, true);
  if (S > 1) {
    cluster_arrive();
    cluster_wait();
  }
  for (int r = tid; r < bn; r += 128) {
    float s = 0.0f;
    for (int pr = 0; pr < S; ++pr) s = __fadd_rn(s, red1[pr * bn + r]);
    inv_s[r] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s, H), 1e-5f)));
  }
  __syncthreads();
  for (int idx = tid; idx < bn * C; idx += 128) {
    const int r = idx / C, c = idx - r * C;
    uint8_t* a = chunk_addr(r, c);
    float xv[8], y[8];
    unpack8(*reinterpret_cast<const uint4*>(a), xv);
    const bool valid = tile_b * bn + r < p.m_tok;
    const float m = mean_s[r], iv = inv_s[r];
#pragma unroll
    for (int e = 0; e < 8; ++e)
      y[e] = valid ? __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[e], m), iv), g_s[c * 8 + e]), b_s[c * 8 + e]) : 0.0f;
    *reinterpret_cast<uint4*>(a) = pack8(y);
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (S > 1 && rearm) cluster_arrive_relaxed();
  __syncthreads();
}

// Scratch the row-LN epilogue needs in the drained ring: the parked partial
// tile [bn][128] f32, the finished values [bn/2][128] f32, exchange slots
// [2][TA][bn/2], warp partials [2][4][bn/2], mean / inv [bn/2].
__host__ __device__ inline size_t gemm_rowln_scratch_bytes(int bn, int tiles_a) {
  const int bh = bn / 2;
  return (size_t)kTileA * bn * 4 + (size_t)kTileA * bh * 4 + (size_t)(2 * tiles_a * bh + 10 * bh) * 4;
}

// Row-LN epilogue (see GemmArgs::row_ln). The cluster is the whole grid: CTA
// (x, z) holds the f32 partial of features [128x, 128x+128) over K half z.
// CTA (x, z) finalises tokens [z*bn/2, (z+1)*bn/2): acc = p0 + p1 (split
// order), v = q16(x + q16(acc + b)) (model.py:478-482 / 491-494, bit-identical
// to the other epilogues), then the LayerNorm of each token row over the TA
// CTAs that share z (tensor.py:153-160 two-pass form: per-CTA column sums ->
// every peer over DSMEM -> summed in CTA order after a cluster barrier; then the
// same for the squared deviations). Deterministic; per-token, so batch-invariant.
// Loops are kept rolled: the executed path stays short for the i-cache.
__device__ __noinline__ void gemm_rowln_epilogue(const GemmArgs& p, uint32_t trow, uint8_t* smem) {
  const int TA = gridDim.x, x = blockIdx.x, z = blockIdx.z;
  const int bn = p.bn, bh = bn / 2, t0 = z * bh;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int f = x * kTileA + tid;
  const bool fok = f < p.n_feat;
  const float H = (float)p.n_feat;
  float* part = reinterpret_cast<float*>(smem);  // [bn][128]
  float* vals = part + kTileA * bn;              // [bh][128]
  float* red = vals + kTileA * bh;               // [2][TA][bh]
  float* wsum = red + 2 * TA * bh;               // [2][4][bh]
  float* mean = wsum + 8 * bh;                   // [bh]
  float* inv = mean + bh;                        // [bh]
  for (int c = 0; c < bn; c += 16) {
    float v[16];
    tmem_ld16(trow + (uint32_t)c, v);
#pragma unroll
    for (int j = 0; j < 16; ++j) part[(c + j) * kTileA + tid] = v[j];
  }
  const float bias = fok ? p.bias[f] : 0.0f;
  cluster_arrive();
  cluster_wait();  // every partial tile parked
  const uint32_t loc = smem_u32(part) + (uint32_t)((t0 * kTileA + tid) * 4);
  const uint32_t a0 = dsmem_addr(loc, (uint32_t)x), a1 = dsmem_addr(loc, (uint32_t)(x + TA));
#pragma unroll 4
  for (int t = 0; t < bh; ++t) {
    const int tok = t0 + t;
    const float p0 = ld_dsmem_f32(a0 + (uint32_t)(t * kTileA * 4));
    const float p1 = ld_dsmem_f32(a1 + (uint32_t)(t * kTileA * 4));
    const float xo = (fok && tok < p.m_tok) ? __half2float(p.resid[(size_t)tok * p.ldr + f]) : 0.0f;
    const float acc = __fadd_rn(__fadd_rn(0.0f, p0), p1);
    vals[t * kTileA + tid] = (fok && tok < p.m_tok) ? q16(__fadd_rn(xo, q16(__fadd_rn(acc, bias)))) : 0.0f;
  }
  for (int rnd = 0; rnd < 2; ++rnd) {
    float* w = wsum + rnd * 4 * bh;
    float* rr = red + rnd * TA * bh;
    for (int t = 0; t < bh; ++t) {
      const float v = vals[t * kTileA + tid];
      float q = v;
      if (rnd == 1) {
        const float d = fok ? __fsub_rn(v, mean[t]) : 0.0f;
        q = __fmul_rn(d, d);
      }
      q = warp_sum(q);
      if (lane == 0) w[warp * bh + t] = q;
    }
    __syncthreads();
    if (tid < bh) {
      const float tot = __fadd_rn(__fadd_rn(__fadd_rn(w[tid], w[bh + tid]), w[2 * bh + tid]), w[3 * bh + tid]);
      const uint32_t ad = smem_u32(rr + x * bh + tid);
      for (int xx = 0; xx < TA; ++xx) st_dsmem_f32(dsmem_addr(ad, (uint32_t)(xx + TA * z)), tot);
    }
    cluster_arrive();
    cluster_wait();
    if (tid < bh) {
      float s = 0.0f;
      for (int xx = 0; xx < TA; ++xx) s = __fadd_rn(s, rr[xx * bh + tid]);
      if (rnd == 0)
        mean[tid] = __fdiv_rn(s, H);
      else
        inv[tid] = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(s, H), 1e-5f)));
    }
    __syncthreads();
  }
  if (fok) {
    const float gam = p.lnf_g[f], bet = p.lnf_b[f];
    for (int t = 0; t < bh; ++t) {
      const int tok = t0 + t;
      if (tok >= p.m_tok) break;
      const float v = vals[t * kTileA + tid];
      p.out[(size_t)tok * p.ldo + f] = __float2half_rn(v);
      p.lnf_h[(size_t)tok * p.lnf_ldh + f] =
          f16_sat(__fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(v, mean[t]), inv[t]), gam), bet));
    }
  }
}

// LayerNorm of the rows this CTA completes (RED_PUSHLN). [u_lo, u_hi): the
// CTA's reduction units (unit u = token column u / 32, features 4 * (u % 32)
// .. +3 of the tile). Release: every thread's x stores, a CTA barrier, then one
// acq_rel fence; each touched token gets one atomicAdd (its own thread) of the
// features this CTA stored; the add that completes n_feat makes this CTA the
// row's normaliser (acquire fence, L2 reads of the row). Arithmetic: the
// stand-alone LN kernel's (ln_row_apply), so h is bit-identical to it.
template <int NT>
__device__ __forceinline__ void gemm_ln_tail(const GemmArgs& p, int tile_a, int tile_b, int u_lo, int u_hi) {
  __shared__ int s_rows[64];
  __shared__ int s_nrows;
  if (threadIdx.x == 0) s_nrows = 0;
  __syncthreads();  // every thread's x stores happen-before the fences below
  const int c_lo = u_lo / 32, c_hi = u_hi > u_lo ? (u_hi - 1) / 32 : c_lo - 1;
  for (int c = c_lo + (int)threadIdx.x; c <= c_hi; c += NT) {
    const int tok = tile_b * p.bn + c;
    if (tok >= p.m_tok) continue;
    int n = 0;
    for (int u = max(u_lo, c * 32); u < min(u_hi, c * 32 + 32); ++u)
      n += max(0, min(4, p.n_feat - (tile_a * kTileA + (u % 32) * 4)));
    if (n == 0) continue;
    asm volatile("fence.acq_rel.gpu;" ::: "memory");  // release (cumulative over the barrier)
    const int prev = atomicAdd(p.lnf_cnt + tok, n);
    if (prev + n == p.n_feat) s_rows[atomicAdd(&s_nrows, 1)] = tok;
  }
  __syncthreads();
  const int nl = s_nrows;
  if (nl == 0) return;
  asm volatile("fence.acq_rel.gpu;" ::: "memory");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int NC = 4;  // H <= 1024; chunks past H are skipped (same sums as NC = ceil(H/256))
  float4 gv[NC * 2], bv[NC * 2];
  ln_load_gb<NC>(p.n_feat, p.lnf_g, p.lnf_b, lane, gv, bv);
  for (int i = warp; i < nl; i += NT / 32) {
    const int tok = s_rows[i];
    const __half* xr = p.out + (size_t)tok * p.ldo;
    uint4 raw[NC];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      const int c = (lane + 32 * j) * 8;
      if (c < p.n_feat) raw[j] = __ldcg(reinterpret_cast<const uint4*>(xr + c));
    }
    float xv[NC * 8];
#pragma unroll
    for (int j = 0; j < NC; ++j) {
      if ((lane + 32 * j) * 8 < p.n_feat) {
        unpack8(raw[j], &xv[8 * j]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[8 * j + e] = 0.0f;
      }
    }
    ln_row_apply<NC>(xv, p.n_feat, gv, bv, p.lnf_h + (size_t)tok * p.lnf_ldh, lane);
    if (lane == 0) p.lnf_cnt[tok] = 0;
  }
}

// Reduction / epilogue path of a launch (template parameter, so every
// instantiation carries only the code it executes: decode kernels are
// i-cache-bound when they carry all paths)
enum GemmRed : int {
  RED_ONE = 0,    // splits == 1 (full-K tile; non-swap staged epilogue or per-chunk stores)
  RED_PUSH = 1,   // split-K cluster, push form (swap, bn <= 128)
  RED_PULL = 2,   // split-K cluster, pull form
  RED_ROWLN = 3,  // whole-row cluster + fused LayerNorm (EPI_BIAS_RESID, swap)
  RED_PUSHLN = 4,  // push split-K + LayerNorm of completed rows by their last CTA (EPI_BIAS_RESID)
};
// LayerNorm of the B operand built in-kernel: 0 none, 1 full-row staging
// (ln_build_b), 2 cluster-cooperative (ln_coop_build)
// threads per CTA: the prefill (non-swap, full-K) tiles run their staged
// epilogue with eight warps; so does the decode push reduction (one pass over
// the CTA's units instead of two at batch 32 with 6 or fewer splits)
__host__ __device__ constexpr int gemm_threads(int mode, bool swap, int red, int lnv = 0) {
  return ((!swap && red == RED_ONE && mode != EPI_LOGITS) || (swap && (red == RED_PUSH || red == RED_PUSHLN) && lnv <= 1) ||
          (swap && red == RED_ONE && lnv == 0 &&
           (mode == EPI_QKV || mode == EPI_BIAS || mode == EPI_BIAS_GELU || mode == EPI_BIAS_RESID)))
             ? 256
             : 128;
}

template <int MODE, bool SWAP, int RED, int LNV>
__global__ void __launch_bounds__(gemm_threads(MODE, SWAP, RED, LNV), 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  const int bn = p.bn, stages = p.stages;
  const int stage_bytes = gemm_stage_bytes(bn);
  constexpr bool ln_mode = SWAP && LNV != 0;
  uint8_t* bln = smem + gemm_ring_bytes(bn, stages, p.splits, SWAP);
  constexpr bool coop = ln_mode && LNV == 2;
  uint8_t* recv = bln + (ln_mode ? (coop ? gemm_ln_coop_bytes(bn, p.kb_per_split, p.splits)
                                         : gemm_ln_bytes(bn, p.kb_per_split, p.k_blocks))
                                 : 0);
  float* ln_sc = reinterpret_cast<float*>(bln + (size_t)p.kb_per_split * bn * kBK * 2);  // coop scratch
  uint8_t* stg = bln + (size_t)p.kb_per_split * bn * kBK * 2;  // LN source rows (ln_mode)
  constexpr bool push = RED == RED_PUSH || RED == RED_PUSHLN;
  uint64_t* bars = reinterpret_cast<uint64_t*>(recv + gemm_recv_bytes(bn, p.splits, SWAP));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 3);
  __shared__ unsigned long long red[64];

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tile_a = blockIdx.x, tile_b = blockIdx.y, split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int nkb = min(p.kb_per_split, p.k_blocks - kb0);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + stages),
                 done_bar = smem_u32(bars + 2 * stages), recv_bar = smem_u32(bars + 2 * stages + 1),
                 ln_bar = smem_u32(bars + 2 * stages + 2);
  const uint32_t ncols = (uint32_t)gemm_tmem_cols(bn);
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(p.trace, 0);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done_bar, 1);
    mbar_init(recv_bar, 1);
    mbar_init(ln_bar, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  // push reduction: peers may signal this CTA's recv_bar only after it is
  // initialised; the matching wait sits right before the first push
  if constexpr (push) cluster_arrive_relaxed();
  const uint32_t tmem = *tmem_slot;
  // let the next kernel in the stream launch now: its prologue (barrier init,
  // TMEM alloc, weight TMA prefetch) overlaps this kernel; it still waits on
  // griddepcontrol.wait before touching anything this kernel writes. With
  // late_trigger the release waits for this kernel's own dependency instead
  // (so a heavy prefetching successor does not compete with this kernel's
  // weight prefetch).
  if (!p.late_trigger) pdl_trigger();

  // ---------------- TMA producer. Weights do not depend on the previous
  // kernel, so in decode (SWAP) mode the first ring's worth of weight tiles is
  // requested before waiting on the programmatic launch dependency.
  const uint32_t tx = ln_mode ? (uint32_t)kABytes : (uint32_t)stage_bytes;
  const int pre = SWAP ? min(stages, nkb) : 0;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < pre; ++i) {
      const uint32_t sa = smem_u32(smem + (size_t)i * stage_bytes);
      mbar_expect_tx(full0 + 8 * i, tx);
      tma_load_2d(sa, &tmA, (kb0 + i) * kBK, tile_a * kTileA, full0 + 8 * i);
    }
  }
  if (warp == 3 && lane == 0) l2_prefetch_share(p.l2pf, p.l2pf_bytes);
  if constexpr (coop) {
    // gamma / beta of this CTA's K slice are weights: staged before the wait
    float* g_s = ln_sc + 2 * p.splits * bn + gemm_ln_coop_seg(bn, p.kb_per_split) + 2 * bn;
    for (int i = threadIdx.x; i < nkb * kBK; i += 128) {
      const int f = kb0 * kBK + i;
      g_s[i] = f < p.ln_H ? p.ln_g[f] : 0.0f;
      g_s[nkb * kBK + i] = f < p.ln_H ? p.ln_b[f] : 0.0f;
    }
    pdl_wait();
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(ln_bar, (uint32_t)(nkb * bn * kBK * 2));
      for (int kb = 0; kb < nkb; ++kb)
        tma_load_2d(smem_u32(bln + (size_t)kb * bn * kBK * 2), &tmB, (kb0 + kb) * kBK, tile_b * bn, ln_bar);
    }
    mbar_wait(ln_bar, 0);
    __syncthreads();  // g_s / b_s visible
    ln_coop_build(p, tile_b, nkb, bln, ln_sc, push, push);
  } else if constexpr (ln_mode) {  // stage the source rows by TMA, then every thread builds the normalised B tiles
    // gamma / beta of this CTA's K slice are weights: staged before the wait
    float* gsl = reinterpret_cast<float*>(stg + (size_t)p.k_blocks * bn * kBK * 2);
    float* bsl = gsl + p.kb_per_split * kBK;
    for (int i = threadIdx.x; i < nkb * kBK; i += gemm_threads(MODE, SWAP, RED, LNV)) {
      const int f = kb0 * kBK + i;
      gsl[i] = f < p.ln_H ? p.ln_g[f] : 0.0f;
      bsl[i] = f < p.ln_H ? p.ln_b[f] : 0.0f;
    }
    pdl_wait();
    if (warp == 0 && lane == 0) {
      mbar_expect_tx(ln_bar, (uint32_t)(p.k_blocks * bn * kBK * 2));
      for (int kb = 0; kb < p.k_blocks; ++kb)
        tma_load_2d(smem_u32(stg + (size_t)kb * bn * kBK * 2), &tmB, kb * kBK, tile_b * bn, ln_bar);
    }
    mbar_wait(ln_bar, 0);
    __syncthreads();  // gsl / bsl visible
    ln_build_b<gemm_threads(MODE, SWAP, RED, LNV)>(p, tile_b, kb0, nkb, bln, stg, gsl, bsl);
    __syncthreads();
  }
  if (warp == 0 && lane == 0) {
    if (!ln_mode) pdl_wait();
    tr.mark(p.trace, 1);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (uint32_t)(i / stages) & 1u;
      const uint32_t sa = smem_u32(smem + (size_t)s * stage_bytes);
      const uint32_t sb = sa + kABytes;
      if (i >= pre) {
        mbar_wait(empty0 + 8 * s, ph ^ 1u);
        mbar_expect_tx(full0 + 8 * s, tx);
        tma_load_2d(sa, &tmA, (kb0 + i) * kBK, tile_a * kTileA, full0 + 8 * s);
      }
      if (!ln_mode) tma_load_2d(sb, &tmB, (kb0 + i) * kBK, tile_b * bn, full0 + 8 * s);
    }
  } else if (warp == 1) {
    // ---------------- MMA issue: the whole warp walks the k-blocks (warp-
    // uniform control flow keeps descriptors in uniform registers: ~35-40
    // instead of ~60 cycles per tcgen05.mma, tools/mma_rate.cu); the elected
    // lane (always lane 0 with the full warp active) issues the MMAs and the
    // commits, which track that thread's MMAs
    const uint32_t idesc = idesc_f16_m128((uint32_t)bn);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % stages;
      const uint32_t ph = (uint32_t)(i / stages) & 1u;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + (size_t)s * stage_bytes);
      const uint64_t da = umma_desc_sw128(sa);
      const uint64_t db = umma_desc_sw128(ln_mode ? smem_u32(bln + (size_t)i * bn * kBK * 2) : sa + kABytes);
      if (elect_lane0()) {
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          // advance 16 f16 = 32 B along K inside the swizzle atom (+2 in 16-B units)
          tc_mma_f16(tmem, da + 2 * k, db + 2 * k, idesc, (i | k) != 0 ? 1u : 0u);
        }
        tc_commit(empty0 + 8 * s);
      }
      __syncwarp();
    }
    if (elect_lane0()) tc_commit(done_bar);
  }
  __syncwarp();

  // ---------------- epilogue (all 4 warps)
  pdl_wait();
  if (p.late_trigger) pdl_trigger();
  // cache slot of token t = 0 (EPI_QKV): one load per thread, overlapping the MMA
  const int qslot = (MODE == EPI_QKV && p.qbase_dev != nullptr) ? *p.qbase_dev : 0;
  mbar_wait(done_bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) tr.mark(p.trace, 2);
  const int row = warp * 32 + lane;  // TMEM lane == row of the A tile
  const int ra = tile_a * kTileA + row;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  float v[16];
  if constexpr (RED == RED_ROWLN) {
    if constexpr (MODE == EPI_BIAS_RESID && SWAP) gemm_rowln_epilogue(p, trow, smem);
  } else if constexpr (RED == RED_ONE && !SWAP) {
    if (MODE != EPI_LOGITS || p.keys == nullptr) {
      epi_tile_nonswap<MODE, false, gemm_threads(MODE, SWAP, RED)>(p, tile_a, tile_b,
                                                                   tmem + (uint32_t)((warp & 3) * 32 << 16), smem);
    } else {
      for (int c = 0; c < bn; c += 16) {
        tmem_ld16(trow + (uint32_t)c, v);
        epi_chunk<MODE, SWAP>(p, ra, tile_b * bn + c, v, reinterpret_cast<unsigned long long*>(smem));
      }
    }
  } else if constexpr (RED == RED_ONE) {
    if constexpr (MODE == EPI_QKV || MODE == EPI_BIAS || MODE == EPI_BIAS_GELU || MODE == EPI_BIAS_RESID) {
      constexpr int NT = gemm_threads(MODE, SWAP, RED, LNV);
      const uint32_t tq = tmem + ((uint32_t)((warp & 3) * 32) << 16);
      epi_swap_one<MODE>(p, tile_a * kTileA + (warp & 3) * 32 + lane, tile_b * bn, bn, tq, NT == 256 ? (warp >> 2) * 16 : 0,
                         NT == 256 ? 32 : 16);
    } else {
      for (int c = 0; c < bn; c += 16) {
        tmem_ld16(trow + (uint32_t)c, v);
        epi_chunk<MODE, SWAP>(p, ra, tile_b * bn + c, v, reinterpret_cast<unsigned long long*>(smem));
      }
    }
  } else if constexpr (RED == RED_PUSH || RED == RED_PUSHLN) {
    // Split-K across the CTAs of one cluster, push form. Each CTA parks its f32
    // partial tile ([column][128 rows], in the drained ring), then one thread
    // bulk-copies the slice owned by every peer r (units [r*per, r*per+per),
    // 16 B per unit) into r's receive buffer at row `rank`, completing bytes
    // on r's recv_bar. Each CTA waits only for its own S-1 incoming slices and
    // reduces them from local smem in split order 0..S-1 (deterministic; the
    // same sums as the pull form). No cluster barrier on the data path; the
    // CTA only waits for its outgoing copies to finish reading before exit.
    constexpr int NT = gemm_threads(MODE, SWAP, RED, LNV);
    float* part = reinterpret_cast<float*>(smem);
    {
      // warps w and w + 4 share TMEM lane quadrant w % 4 and park column halves
      const int prow = (warp & 3) * 32 + lane;
      const int pc0 = NT == 256 ? (warp >> 2) * (bn / 2) : 0, pc1 = NT == 256 ? pc0 + bn / 2 : bn;
      const uint32_t prow_t = tmem + ((uint32_t)((warp & 3) * 32) << 16);
      for (int c = pc0; c < pc1; c += 16) {
        tmem_ld16(prow_t + (uint32_t)c, v);
#pragma unroll
        for (int j = 0; j < 16; ++j)
          if (c + j < pc1) part[(c + j) * kTileA + prow] = v[j];
      }
    }
    fence_proxy_async_smem();  // generic smem writes -> visible to the bulk-copy engine
    const uint32_t rank = cluster_ctarank();
    const int S = p.splits;
    const int U = (kTileA / 4) * bn;
    const int per = (U + S - 1) / S;
    const int u_lo = (int)rank * per, u_hi = min(U, u_lo + per);
    cluster_wait();  // every peer's recv_bar is initialised
    __syncthreads();
    if (threadIdx.x == 0) {
      tr.mark(p.trace, 3);
      const int mine = max(0, u_hi - u_lo);
      mbar_expect_tx(recv_bar, (uint32_t)((S - 1) * mine * 16));
      const uint32_t src0 = smem_u32(part), rcv0 = smem_u32(recv);
      for (int r = 0; r < S; ++r) {
        if (r == (int)rank) continue;
        const int r_lo = r * per, r_n = min(U, r_lo + per) - r_lo;
        if (r_n <= 0) continue;
        bulk_copy_to_peer(dsmem_addr(rcv0 + (uint32_t)(rank * per * 16), (uint32_t)r),
                          src0 + (uint32_t)(r_lo * 16), (uint32_t)(r_n * 16), dsmem_addr(recv_bar, (uint32_t)r));
      }
      bulk_commit();
    }
    // epilogue operands of this thread's first two units, loaded while the
    // peer slices are in flight
    EpiPre4 pre, pre2;
    int u = u_lo + (int)threadIdx.x;
    if (u < u_hi) epi_pre4<MODE, SWAP>(p, tile_a, tile_b, u, pre);
    if (u + NT < u_hi) epi_pre4<MODE, SWAP>(p, tile_a, tile_b, u + NT, pre2);
    mbar_wait(recv_bar, 0);
    if (threadIdx.x == 0) tr.mark(p.trace, 4);
    const float4* own = reinterpret_cast<const float4*>(part);
    const float4* rin = reinterpret_cast<const float4*>(recv);
    for (int it = 0; u < u_hi; u += NT, ++it) {
      const bool first = it == 0;
      if (it == 1) pre = pre2;
      if (it >= 2) epi_pre4<MODE, SWAP>(p, tile_a, tile_b, u, pre);
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int sp = 0; sp < 16; ++sp)
        if (sp < S) {
          const float4 pv = sp == (int)rank ? own[u] : rin[sp * per + (u - u_lo)];
          acc[0] = __fadd_rn(acc[0], pv.x);
          acc[1] = __fadd_rn(acc[1], pv.y);
          acc[2] = __fadd_rn(acc[2], pv.z);
          acc[3] = __fadd_rn(acc[3], pv.w);
        }
      if (threadIdx.x == 0 && first) tr.mark(p.trace, 5);
      epi_fin4<MODE, SWAP>(p, tile_a, tile_b, u, acc, pre, qslot);
    }
    if (threadIdx.x == 0) {
      tr.mark(p.trace, 6);
      bulk_wait_read_all();  // outgoing slices read before this smem is released
    }
    if constexpr (RED == RED_PUSHLN && MODE == EPI_BIAS_RESID) gemm_ln_tail<NT>(p, tile_a, tile_b, u_lo, u_hi);
  } else {
    static_assert(RED == RED_PULL, "reduction path");
    // Split-K across the CTAs of one thread-block cluster (grid.z == cluster.z
    // == splits). Each CTA parks its f32 partial tile in its own (drained)
    // pipeline smem as [column][128 rows]; after a cluster barrier every CTA
    // reduces a contiguous 1/S slice of the tile by reading the S partials over
    // DSMEM in split order 0..S-1 (deterministic), then runs the epilogue on it.
    float* part = reinterpret_cast<float*>(smem);
    for (int c = 0; c < bn; c += 16) {
      tmem_ld16(trow + (uint32_t)c, v);
#pragma unroll
      for (int j = 0; j < 16; ++j) part[(c + j) * kTileA + row] = v[j];
    }
    // Work unit = 4 adjacent rows of one column of the tile (16 B of every
    // partial); CTA `rank` reduces a contiguous 1/S of the units. The epilogue
    // operands of the first unit (bias, residual) are loaded before the
    // cluster barrier so their latency overlaps the wait for the slowest split.
    const uint32_t rank = cluster_ctarank();
    const int S = p.splits;
    const int U = (kTileA / 4) * bn;
    const int per = (U + S - 1) / S;
    const int u_lo = (int)rank * per, u_hi = min(U, u_lo + per);
    EpiPre4 pre;
    int u = u_lo + (int)threadIdx.x;
    if (threadIdx.x == 0) tr.mark(p.trace, 3);
    cluster_arrive();  // release: this CTA's partial tile is complete
    if (u < u_hi) epi_pre4<MODE, SWAP>(p, tile_a, tile_b, u, pre);
    cluster_wait();
    if (threadIdx.x == 0) tr.mark(p.trace, 4);
    const uint32_t local = smem_u32(part);
    // the last DSMEM read of this thread is followed by the arrive that lets the
    // other CTAs exit; the epilogue stores of the last unit overlap that barrier
    const int n_units = u < u_hi ? (u_hi - 1 - u) / 128 + 1 : 0;
    int it = 0;
    if (n_units == 0) cluster_arrive_any();
    for (bool first = true; u < u_hi; u += 128, first = false, ++it) {
      if (!first) epi_pre4<MODE, SWAP>(p, tile_a, tile_b, u, pre);
      // all S loads in flight, then the sum in split order (deterministic)
      float4 pv[16];
#pragma unroll
      for (int sp = 0; sp < 16; ++sp)
        if (sp < S) pv[sp] = ld_dsmem_f32x4(dsmem_addr(local + 16u * (uint32_t)u, (uint32_t)sp));
      float acc[4] = {0.0f, 0.0f, 0.0f, 0.0f};
#pragma unroll
      for (int sp = 0; sp < 16; ++sp)
        if (sp < S) {
          acc[0] = __fadd_rn(acc[0], pv[sp].x);
          acc[1] = __fadd_rn(acc[1], pv[sp].y);
          acc[2] = __fadd_rn(acc[2], pv[sp].z);
          acc[3] = __fadd_rn(acc[3], pv[sp].w);
        }
      if (threadIdx.x == 0 && first) tr.mark(p.trace, 5);
      if (it == n_units - 1) cluster_arrive_any();
      epi_fin4<MODE, SWAP>(p, tile_a, tile_b, u, acc, pre, qslot);
    }
    if (threadIdx.x == 0) tr.mark(p.trace, 6);
    cluster_wait_any();  // partial tiles stay alive until every CTA has read them
  }
  tc_fence_before();
  __syncthreads();
  if (threadIdx.x == 0) {
    tr.mark(p.trace, 7);
    tr.flush(p.trace);
  }
  if (warp == 2) tmem_dealloc(tmem, ncols);
}

// ---------------------------------------------------------------- persistent prefill GEMM
// Non-swap (token-major) GEMM for prefill-sized M: one CTA per SM loops over
// output tiles; warp 0 streams A/B k-blocks through a `stages`-deep TMA ring
// across tile boundaries, warp 1 issues tcgen05.mma into one of TWO TMEM
// accumulators, warps 2-5 run the staged epilogue of the previous tile from the
// other accumulator (released to the MMA warp as soon as its TMEM reads are
// done). Tiles are visited token-tile-fastest so the CTAs running at the same
// time share the weight tile (L2 reuse).
constexpr int kPfThreadsGemm = 192;
__host__ __device__ inline size_t gemm_pf_smem_bytes(int bn, int stages, bool f32out) {
  return 1024 + (size_t)stages * gemm_stage_bytes(bn) + (size_t)kTileA * (bn * (f32out ? 4 : 2) + 16) +
         (size_t)(2 * stages + 4) * 8 + 16;
}

template <int MODE>
__global__ void __launch_bounds__(kPfThreadsGemm, 1)
    gemm_pf_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  constexpr bool F32OUT = MODE == EPI_F32;
  const int bn = p.bn, stages = p.stages;
  const int stage_bytes = gemm_stage_bytes(bn);
  uint8_t* out_stage = smem + (size_t)stages * stage_bytes;
  uint64_t* bars = reinterpret_cast<uint64_t*>(out_stage + (size_t)kTileA * (bn * (F32OUT ? 4 : 2) + 16));
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * stages + 4);
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + stages);
  const uint32_t accf0 = smem_u32(bars + 2 * stages), acce0 = smem_u32(bars + 2 * stages + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int tiles_a = (p.m_tok + kTileA - 1) / kTileA, tiles_b = (p.n_feat + bn - 1) / bn;
  const int n_tiles = tiles_a * tiles_b, nkb = p.k_blocks;
  const uint32_t ncols = 2 * bn <= 32 ? 32u : (2 * bn <= 64 ? 64u : (2 * bn <= 128 ? 128u : (2 * bn <= 256 ? 256u : 512u)));
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(p.trace, 0);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < stages; ++s) {
      mbar_init(full0 + 8 * s, 1);
      mbar_init(empty0 + 8 * s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(accf0 + 8 * b, 1);
      mbar_init(acce0 + 8 * b, 1);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(smem_u32(tmem_slot), ncols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();
  pdl_wait();
  if (threadIdx.x == 0) tr.mark(p.trace, 1);
  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer, continuous over tiles
      int it = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x) {
        const int ta = t % tiles_a, tb = t / tiles_a;
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (uint32_t)(it / stages) & 1u;
          mbar_wait(empty0 + 8 * s, ph ^ 1u);
          const uint32_t sa = smem_u32(smem + (size_t)s * stage_bytes);
          mbar_expect_tx(full0 + 8 * s, (uint32_t)stage_bytes);
          tma_load_2d(sa, &tmA, kb * kBK, ta * kTileA, full0 + 8 * s);
          tma_load_2d(sa + kABytes, &tmB, kb * kBK, tb * bn, full0 + 8 * s);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer, two TMEM accumulators
      const uint32_t idesc = idesc_f16_m128((uint32_t)bn);
      int it = 0, tc = 0;
      for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tc) {
        const int b = tc & 1, use = tc >> 1;
        mbar_wait(acce0 + 8 * b, ((uint32_t)use & 1u) ^ 1u);
        tc_fence_after();
        const uint32_t acc = tmem + (uint32_t)(b * bn);
        for (int kb = 0; kb < nkb; ++kb, ++it) {
          const int s = it % stages;
          const uint32_t ph = (uint32_t)(it / stages) & 1u;
          mbar_wait(full0 + 8 * s, ph);
          tc_fence_after();
          const uint32_t sa = smem_u32(smem + (size_t)s * stage_bytes);
          const uint64_t da = umma_desc_sw128(sa), db = umma_desc_sw128(sa + kABytes);
#pragma unroll
          for (int k = 0; k < kBK / 16; ++k) tc_mma_f16(acc, da + 2 * k, db + 2 * k, idesc, (kb | k) != 0 ? 1u : 0u);
          tc_commit(empty0 + 8 * s);
        }
        tc_commit(accf0 + 8 * b);
      }
    }
  } else {  // ---- epilogue warps 2..5 (TMEM lane quadrant = warp % 4)
    const int q = warp & 3, row = q * 32 + lane;
    int tc = 0;
    for (int t = blockIdx.x; t < n_tiles; t += gridDim.x, ++tc) {
      const int ta = t % tiles_a, tb = t / tiles_a;
      const int b = tc & 1, use = tc >> 1;
      mbar_wait(accf0 + 8 * b, (uint32_t)use & 1u);
      tc_fence_after();
      const uint32_t trow = tmem + (uint32_t)(b * bn) + ((uint32_t)(q * 32) << 16);
      epi_tile_nonswap<MODE, true>(p, ta, tb, trow, out_stage, row, acce0 + 8 * b);
    }
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
