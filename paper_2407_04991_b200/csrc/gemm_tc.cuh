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
  // SWAP consumer (LNV = 1), LayerNorm folded into the GEMM: the B operand
  // rows are the raw residual stream x and the weights W' = q16(W * gamma)
  // (gamma folded over K), so LN(x) . W = inv_t * (x . W' - mean_t * c) + d
  // with c = sum_k W'[:, k], d = sum_k beta_k W[:, k] (per output feature,
  // ln_c / ln_d). Row t's (mean, inv) come from per-128-feature-tile partials
  // ln_stats[tile * ln_stats_ld + t] = (mean_i, M2_i) written by the residual
  // GEMM that produced x (stats_out below), merged in the epilogue.
  const float2* ln_stats;
  int ln_H, ln_tiles, ln_stats_ld;
  const float* ln_c;
  const float* ln_d;
  // EPI_BIAS_RESID producer (push split-K): per-token (mean, M2) of the tile's
  // new residual values, stats_out[tile_a * stats_ld + tok]
  float2* stats_out;
  int stats_ld;
  int trace;  // diagnostics slot (0 = off)
  int late_trigger;  // release the next kernel only after this kernel's PDL wait
  // decode: activation-independent bytes of a later kernel (the next layer's
  // copy of this weight matrix) streamed HBM -> L2 by this launch's CTAs
  const void* l2pf;
  unsigned long long l2pf_bytes;
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
// LN-folded epilogue (LNV = 1): (mean, inv) of the tile's bn rows, f32
__host__ __device__ inline size_t gemm_ln_bytes(int bn) { return (size_t)2 * bn * 4 + 16; }
// push-based split-K reduction (SWAP, splits > 1, bn <= 128): every CTA owns a
// receive buffer for the S-1 peer slices of its share of the tile
__host__ __device__ inline bool gemm_push_reduce(int bn, int splits, bool swap) {
  return swap && splits > 1 && bn <= 128;
}
// units (4 features x 1 token) per CTA of the push reduction: whole token
// columns (32 units each), so one warp holds all 128 features of a token
__host__ __device__ inline int gemm_push_per(int bn, int splits) { return 32 * ((bn + splits - 1) / splits); }
__host__ __device__ inline size_t gemm_recv_bytes(int bn, int splits, bool swap) {
  if (!gemm_push_reduce(bn, splits, swap)) return 0;
  return (size_t)splits * gemm_push_per(bn, splits) * 16;
}
__host__ inline size_t gemm_smem_bytes(int bn, int stages, int splits, bool swap, size_t ln_bytes = 0) {
  return 1024 + gemm_ring_bytes(bn, stages, splits, swap) + ln_bytes + gemm_recv_bytes(bn, splits, swap) +
         (2 * stages + 3) * 8 + 16;
}

// Row statistics for the folded LayerNorm (LNV = 1): the reference's two-pass
// LayerNorm (tensor.py:153-160: mean; c = x - mean; var = mean(c*c);
// c * (1/sqrt(var + 1e-5))) restated as a merge of per-tile partials
// (mean_i, M2_i over n_i features, written by the residual GEMM that produced
// x): mean = sum n_i mean_i / H, M2 = sum M2_i + sum n_i (mean_i - mean)^2,
// merged in tile order (deterministic, per row, so batch-invariant). Threads
// [t0, t0 + nthr) fill s_mi[r] = mean, s_mi[bn + r] = inv for the tile's rows.
__device__ __forceinline__ void ln_stats_rows(const GemmArgs& p, int tile_b, float* s_mi, int t0, int nthr) {
  const int bn = p.bn;
  for (int r = (int)threadIdx.x - t0; r >= 0 && r < bn; r += nthr) {
    const int t = tile_b * bn + r;
    float mean = 0.0f, inv = 0.0f;
    if (t < p.m_tok) {
      float2 st[16];
      const int nt = p.ln_tiles;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nt) st[i] = p.ln_stats[(size_t)i * p.ln_stats_ld + t];
      float s = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nt) s = __fadd_rn(s, __fmul_rn((float)min(kTileA, p.ln_H - i * kTileA), st[i].x));
      mean = __fdiv_rn(s, (float)p.ln_H);
      float m2 = 0.0f;
#pragma unroll
      for (int i = 0; i < 16; ++i)
        if (i < nt) {
          const float d = __fsub_rn(st[i].x, mean);
          m2 = __fadd_rn(m2, __fadd_rn(st[i].y, __fmul_rn((float)min(kTileA, p.ln_H - i * kTileA), __fmul_rn(d, d))));
        }
      inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(m2, (float)p.ln_H), 1e-5f)));
    }
    s_mi[r] = mean;
    s_mi[bn + r] = inv;
  }
}
// folded LayerNorm of one accumulator: inv * (acc - mean * c) + d
__device__ __forceinline__ float ln_fold(float acc, float mean, float inv, float c, float d) {
  return __fadd_rn(__fmul_rn(__fsub_rn(acc, __fmul_rn(mean, c)), inv), d);
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
                                             int cstep, const float* s_mi) {
  const bool fok = f < p.n_feat;
  const float bf = fok ? p.bias[f] : 0.0f;
  const float lc = (s_mi && fok) ? p.ln_c[f] : 0.0f, ld = (s_mi && fok) ? p.ln_d[f] : 0.0f;
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
    if (s_mi) {
#pragma unroll
      for (int j = 0; j < 16; ++j) v[j] = ln_fold(v[j], s_mi[c + j], s_mi[bn + c + j], lc, ld);
    }
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
  // row / chunk of a linear chunk index: a shift when cpr is a power of two (every
  // 128-wide tile); an integer division per 16-B chunk was ~15% of the kernel's
  // stall samples (ncu source view, 4096x3072x768)
  const bool cpr_pow2 = (cpr & (cpr - 1)) == 0;
  const int cpr_sh = 31 - __clz(cpr);
  auto split_idx = [&](int idx, int& r, int& ch) {
    r = cpr_pow2 ? (idx >> cpr_sh) : idx / cpr;
    ch = idx - r * cpr;
  };
  if constexpr (MODE == EPI_BIAS_RESID) {
    // residual chunks are loaded 8 at a time before use (one exposed global
    // latency per 8 chunks instead of per chunk)
    constexpr int BATCH = 8;
    for (int base = et; base < kTileA * cpr; base += NT * BATCH) {
      uint4 rv[BATCH];
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int idx = base + u * NT;
        int r, ch;
        split_idx(idx, r, ch);
        const int t = tile_a * kTileA + r, f0 = tile_b * bn + ch * 8;
        const bool fast = idx < kTileA * cpr && t < p.m_tok && f0 + 8 <= p.n_feat && (p.ldr % 8) == 0;
        rv[u] = fast ? *reinterpret_cast<const uint4*>(p.resid + (size_t)t * p.ldr + f0) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < BATCH; ++u) {
        const int idx = base + u * NT;
        if (idx >= kTileA * cpr) break;
        int r, ch;
        split_idx(idx, r, ch);
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
    int r, ch;
    split_idx(idx, r, ch);
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
  float c[4], d[4];  // folded LayerNorm terms (LNV = 1)
};

template <bool SWAP>
__device__ __forceinline__ void unit_coords(int tile_a, int tile_b, int bn, int u, int& tok, int& f, int& step) {
  const int col = tile_b * bn + u / 32, r = tile_a * kTileA + (u % 32) * 4;
  tok = SWAP ? col : r;
  f = SWAP ? r : col;
  step = SWAP ? 1 : 0;  // the 4 rows advance the feature (SWAP) or the token
}

template <int MODE, bool SWAP, bool LNF = false>
__device__ __forceinline__ void epi_pre4(const GemmArgs& p, int tile_a, int tile_b, int u, EpiPre4& q) {
  int tok, f, st;
  unit_coords<SWAP>(tile_a, tile_b, p.bn, u, tok, f, st);
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const int tj = tok + (st ? 0 : j), fj = f + (st ? j : 0);
    const bool ok = tj < p.m_tok && fj < p.n_feat;
    if constexpr (LNF) {
      q.c[j] = ok ? p.ln_c[fj] : 0.0f;
      q.d[j] = ok ? p.ln_d[fj] : 0.0f;
    }
    if constexpr (MODE == EPI_BIAS || MODE == EPI_BIAS_GELU || MODE == EPI_BIAS_RESID || MODE == EPI_QKV)
      q.b[j] = ok ? p.bias[fj] : 0.0f;
    if constexpr (MODE == EPI_BIAS_RESID)
      q.x[j] = ok ? __half2float(p.resid[(size_t)tj * p.ldr + fj]) : 0.0f;
  }
}

template <int MODE, bool SWAP>
__device__ __forceinline__ void epi_fin4(const GemmArgs& p, int tile_a, int tile_b, int u, const float (&acc)[4],
                                         const EpiPre4& q, int qslot, float (&yv)[4]) {
  int tok, f, st;
  unit_coords<SWAP>(tile_a, tile_b, p.bn, u, tok, f, st);
  if constexpr (MODE == EPI_F32) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int tj = tok + (st ? 0 : j), fj = f + (st ? j : 0);
      if (tj < p.m_tok && fj < p.n_feat) p.out_f32[(size_t)tj * p.ldo + fj] = acc[j];
      yv[j] = acc[j];
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
    yv[j] = __half2float(val[j]);
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

// Reduction / epilogue path of a launch (template parameter, so every
// instantiation carries only the code it executes: decode kernels are
// i-cache-bound when they carry all paths)
enum GemmRed : int {
  RED_ONE = 0,    // splits == 1 (full-K tile; non-swap staged epilogue or per-chunk stores)
  RED_PUSH = 1,   // split-K cluster, push form (swap, bn <= 128)
  RED_PULL = 2,   // split-K cluster, pull form
};
// LNV (operand LayerNorm): 0 none, 1 the B operand is q16(LN(x)) built in smem
// from the raw rows and the producer's row-statistics partials (ln_stats_*).
// threads per CTA: the prefill (non-swap, full-K) tiles run their staged
// epilogue with eight warps; so do the decode push reduction (one pass over
// the CTA's units at batch 32) and the decode full-K swap epilogues
__host__ __device__ constexpr int gemm_threads(int mode, bool swap, int red, int lnv = 0) {
  return ((!swap && red == RED_ONE && mode != EPI_LOGITS) || (swap && red == RED_PUSH) ||
          (swap && red == RED_ONE &&
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
  constexpr int NTH = gemm_threads(MODE, SWAP, RED, LNV);
  float* s_mi = reinterpret_cast<float*>(smem + gemm_ring_bytes(bn, stages, p.splits, SWAP));  // ln_mode
  uint8_t* recv = reinterpret_cast<uint8_t*>(s_mi) + (ln_mode ? gemm_ln_bytes(bn) : 0);
  constexpr bool push = RED == RED_PUSH;
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
  const uint32_t tx = (uint32_t)stage_bytes;
  const int pre = SWAP ? min(stages, nkb) : 0;
  if (warp == 0 && lane == 0) {
    for (int i = 0; i < pre; ++i) {
      const uint32_t sa = smem_u32(smem + (size_t)i * stage_bytes);
      mbar_expect_tx(full0 + 8 * i, tx);
      tma_load_2d(sa, &tmA, (kb0 + i) * kBK, tile_a * kTileA, full0 + 8 * i);
    }
  }
  if (warp == 3 && lane == 0) l2_prefetch_share(p.l2pf, p.l2pf_bytes);
  if (warp == 0 && lane == 0) {
    pdl_wait();
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
      tma_load_2d(sb, &tmB, (kb0 + i) * kBK, tile_b * bn, full0 + 8 * s);
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
      const uint64_t db = umma_desc_sw128(sa + kABytes);
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
  // folded LayerNorm: the rows' (mean, inv), merged by the warps that neither
  // load nor issue (they overlap the operand TMA and the MMAs)
  if constexpr (ln_mode) ln_stats_rows(p, tile_b, s_mi, 64, NTH - 64);
  mbar_wait(done_bar, 0);
  tc_fence_after();
  if constexpr (ln_mode) __syncthreads();
  if (threadIdx.x == 0) tr.mark(p.trace, 2);
  const int row = warp * 32 + lane;  // TMEM lane == row of the A tile
  const int ra = tile_a * kTileA + row;
  const uint32_t trow = tmem + ((uint32_t)(warp * 32) << 16);
  float v[16];
  if constexpr (RED == RED_ONE && !SWAP) {
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
                         NT == 256 ? 32 : 16, ln_mode ? s_mi : nullptr);
    } else {
      const float lc = (ln_mode && ra < p.n_feat) ? p.ln_c[ra] : 0.0f;
      const float ld = (ln_mode && ra < p.n_feat) ? p.ln_d[ra] : 0.0f;
      for (int c = 0; c < bn; c += 16) {
        tmem_ld16(trow + (uint32_t)c, v);
        if constexpr (ln_mode) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = ln_fold(v[j], s_mi[c + j], s_mi[bn + c + j], lc, ld);
        }
        epi_chunk<MODE, SWAP>(p, ra, tile_b * bn + c, v, reinterpret_cast<unsigned long long*>(smem));
      }
    }
  } else if constexpr (RED == RED_PUSH) {
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
    const int per = gemm_push_per(bn, S);  // whole token columns per CTA
    const int u_lo = min(U, (int)rank * per), u_hi = min(U, u_lo + per);
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
    if (u < u_hi) epi_pre4<MODE, SWAP, ln_mode>(p, tile_a, tile_b, u, pre);
    if (u + NT < u_hi) epi_pre4<MODE, SWAP, ln_mode>(p, tile_a, tile_b, u + NT, pre2);
    mbar_wait(recv_bar, 0);
    if (threadIdx.x == 0) tr.mark(p.trace, 4);
    const float4* own = reinterpret_cast<const float4*>(part);
    const float4* rin = reinterpret_cast<const float4*>(recv);
    for (int it = 0; u < u_hi; u += NT, ++it) {
      const bool first = it == 0;
      if (it == 1) pre = pre2;
      if (it >= 2) epi_pre4<MODE, SWAP, ln_mode>(p, tile_a, tile_b, u, pre);
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
      if constexpr (ln_mode) {  // SWAP: the unit's 4 values share one token
        const int tl = u / 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = ln_fold(acc[j], s_mi[tl], s_mi[bn + tl], pre.c[j], pre.d[j]);
      }
      if (threadIdx.x == 0 && first) tr.mark(p.trace, 5);
      float yv[4];
      epi_fin4<MODE, SWAP>(p, tile_a, tile_b, u, acc, pre, qslot, yv);
      if constexpr (MODE == EPI_BIAS_RESID && SWAP) {
        // row statistics of the new residual values over this tile's features
        // for the LayerNorm fused into the next GEMM (ln_stats_rows): the 32
        // lanes of this warp hold the tile's 128 features of one token
        // (u_lo is a multiple of 32); fixed xor tree, then the two-pass M2
        if (p.stats_out != nullptr) {
          int tok, f, st;
          unit_coords<SWAP>(tile_a, tile_b, bn, u, tok, f, st);
          const int nf = min(kTileA, p.n_feat - tile_a * kTileA);
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < 4; ++j) s = __fadd_rn(s, f + j < p.n_feat ? yv[j] : 0.0f);
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s = __fadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
          const float mean = __fdiv_rn(s, (float)nf);
          float m2 = 0.0f;
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const float d = f + j < p.n_feat ? __fsub_rn(yv[j], mean) : 0.0f;
            m2 = __fadd_rn(m2, __fmul_rn(d, d));
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) m2 = __fadd_rn(m2, __shfl_xor_sync(0xffffffffu, m2, o));
          if (lane == 0 && tok < p.m_tok) p.stats_out[(size_t)tile_a * p.stats_ld + tok] = make_float2(mean, m2);
        }
      }
    }
    if (threadIdx.x == 0) {
      tr.mark(p.trace, 6);
      bulk_wait_read_all();  // outgoing slices read before this smem is released
    }
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
    if (u < u_hi) epi_pre4<MODE, SWAP, ln_mode>(p, tile_a, tile_b, u, pre);
    cluster_wait();
    if (threadIdx.x == 0) tr.mark(p.trace, 4);
    const uint32_t local = smem_u32(part);
    // the last DSMEM read of this thread is followed by the arrive that lets the
    // other CTAs exit; the epilogue stores of the last unit overlap that barrier
    const int n_units = u < u_hi ? (u_hi - 1 - u) / 128 + 1 : 0;
    int it = 0;
    if (n_units == 0) cluster_arrive_any();
    for (bool first = true; u < u_hi; u += 128, first = false, ++it) {
      if (!first) epi_pre4<MODE, SWAP, ln_mode>(p, tile_a, tile_b, u, pre);
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
      if constexpr (ln_mode) {
        const int tl = u / 32;
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = ln_fold(acc[j], s_mi[tl], s_mi[bn + tl], pre.c[j], pre.d[j]);
      }
      if (threadIdx.x == 0 && first) tr.mark(p.trace, 5);
      if (it == n_units - 1) cluster_arrive_any();
      float yv[4];
      epi_fin4<MODE, SWAP>(p, tile_a, tile_b, u, acc, pre, qslot, yv);
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

}  // namespace tf

namespace tf {

// ---------------------------------------------------------------- prefill, 2-CTA (cta_group::2)
// Non-swap GEMM on CTA pairs: a 2-CTA cluster computes a 256-token x 256-feature
// tile with tcgen05.mma.cta_group::2 (M = 256, N = 256). Each CTA stages its own
// 128 token rows of A and HALF of the feature rows of B (128) per 64-wide K
// block — 32 KB per CTA per k-block for 128x256x64 MACs, twice the MACs per
// staged byte of the 128x128 single-CTA tiles, whose main loop is bound by the
// per-SM TMA ingest. The leader CTA (rank 0) waits on its full barrier (both
// CTAs' TMA bytes complete on it: the peer's loads carry the leader's barrier
// address, the peer's producer arrives remotely) and issues the MMAs reading
// both CTAs' shared memory at the same offsets; its commits are multicast to
// both CTAs' empty / done barriers. Every CTA then drains its own TMEM rows
// (128 tokens x 256 features) with the staged 8-warp epilogue of the
// single-CTA kernel. Two such CTAs (of different pairs) share an SM: one's
// epilogue overlaps the other's main loop.
constexpr int kPf2BN = 256, kPf2Stages = 3;
constexpr int kPf2StageBytes = 128 * kBK * 2 + 128 * kBK * 2;  // A 16 KB + B half 16 KB
__host__ __device__ constexpr size_t gemm_pf2_smem_bytes() {
  return 1024 + (size_t)kPf2Stages * kPf2StageBytes + (2 * kPf2Stages + 1) * 8 + 16;
}

__device__ __forceinline__ uint32_t peer0_addr(uint32_t smem_addr) {  // the leader CTA's copy of a barrier
  return smem_addr & 0xFEFFFFFFu;
}

template <int MODE>
__global__ void __launch_bounds__(256, 1)
    gemm_pf2_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const GemmArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)kPf2Stages * kPf2StageBytes);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 2 * kPf2Stages + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;
  const int tile_a = blockIdx.x;  // this CTA's 128-token block
  const int tile_b = blockIdx.y;  // 256-feature block
  const int nkb = p.k_blocks;
  const uint32_t full0 = smem_u32(bars), empty0 = smem_u32(bars + kPf2Stages),
                 done_bar = smem_u32(bars + 2 * kPf2Stages);
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(p.trace, 0);
  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < kPf2Stages; ++s) {
      mbar_init(full0 + 8 * s, 2);  // leader: both producers arrive (leader with the expected bytes)
      mbar_init(empty0 + 8 * s, 1);
    }
    mbar_init(done_bar, 1);
    fence_mbar_init();
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "r"(256)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  cluster_sync();  // both CTAs' barriers initialised and TMEM allocated
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  pdl_trigger();

  if (warp == 0 && lane == 0) {
    // ---------------- producer (both CTAs): own A rows, own half of the B rows
    pdl_wait();
    if (threadIdx.x == 0) tr.mark(p.trace, 1);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kPf2Stages;
      const uint32_t ph = (uint32_t)(i / kPf2Stages) & 1u;
      mbar_wait(empty0 + 8 * s, ph ^ 1u);
      const uint32_t sa = smem_u32(smem + (size_t)s * kPf2StageBytes);
      const uint32_t sb = sa + 128 * kBK * 2;
      const uint32_t fb = full0 + 8 * s;
      if (leader) {
        mbar_expect_tx(fb, (uint32_t)(2 * kPf2StageBytes));
      } else {
        asm volatile("{\n\t.reg .b32 ra;\n\tmapa.shared::cluster.u32 ra, %0, 0;\n\t"
                     "mbarrier.arrive.shared::cluster.b64 _, [ra];\n\t}" ::"r"(fb)
                     : "memory");
      }
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(sa),
          "l"(reinterpret_cast<uint64_t>(&tmA)), "r"(i * kBK), "r"(tile_a * 128), "r"(peer0_addr(fb))
          : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3}], [%4];" ::"r"(sb),
          "l"(reinterpret_cast<uint64_t>(&tmB)), "r"(i * kBK), "r"(tile_b * kPf2BN + (int)rank * 128),
          "r"(peer0_addr(fb))
          : "memory");
    }
  } else if (warp == 1 && leader) {
    // ---------------- MMA issue (leader only), M = 256 over both CTAs' rows
    const uint32_t idesc = idesc_f16(256u, (uint32_t)kPf2BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % kPf2Stages;
      const uint32_t ph = (uint32_t)(i / kPf2Stages) & 1u;
      mbar_wait(full0 + 8 * s, ph);
      tc_fence_after();
      const uint32_t sa = smem_u32(smem + (size_t)s * kPf2StageBytes);
      const uint64_t da = umma_desc_sw128(sa);
      const uint64_t db = umma_desc_sw128(sa + 128 * kBK * 2);
      if (elect_lane0()) {
#pragma unroll
        for (int k = 0; k < kBK / 16; ++k) {
          asm volatile(
              "{\n\t.reg .pred pp;\n\tsetp.ne.b32 pp, %4, 0;\n\t"
              "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, pp;\n\t}" ::"r"(tmem),
              "l"(da + 2 * k), "l"(db + 2 * k), "r"(idesc), "r"((i | k) != 0 ? 1u : 0u)
              : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                empty0 + 8 * s),
            "h"((unsigned short)3)
            : "memory");
      }
      __syncwarp();
    }
    if (elect_lane0())
      asm volatile(
          "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
              done_bar),
          "h"((unsigned short)3)
          : "memory");
  }
  __syncwarp();

  // ---------------- epilogue (all 8 warps, each CTA its own 128 token rows)
  pdl_wait();
  mbar_wait(done_bar, 0);
  tc_fence_after();
  if (threadIdx.x == 0) tr.mark(p.trace, 2);
  GemmArgs q = p;
  q.bn = kPf2BN;
  epi_tile_nonswap<MODE, false, 256>(q, tile_a, tile_b, tmem + (uint32_t)((warp & 3) * 32 << 16), smem);
  tc_fence_before();
  cluster_sync();  // neither CTA frees TMEM / smem while the pair may still touch it
  if (threadIdx.x == 0) {
    tr.mark(p.trace, 7);
    tr.flush(p.trace);
  }
  if (warp == 2) asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256) : "memory");
}

}  // namespace tf
