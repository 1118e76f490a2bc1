// Embedding gather-sum (+ optional pruned-vocab remap and type row) fused with
// the first LayerNorm, the stand-alone LayerNorm, and step bookkeeping.
//
// Numerics follow the reference exactly where it is integer/elementwise:
//   x = q16(tok[id] + pos[p] (+ type[t]))      (model.py:453-455, bit-exact)
//   LN: mean = sum/H; c = x - mean; var = sum(c*c)/H;
//       y = q16(((c * (1/sqrt(var + 1e-5))) * g) + b)   (tensor.py:153-160)
// Only the two reductions differ in summation order from numpy's pairwise sum.
#pragma once

#include "common.cuh"

namespace tf {

struct EmbedArgs {
  int n_tok, H, V, P;
  const int* ids;            // [n_tok] token ids (model vocab), or null -> keys
  unsigned long long* keys;  // decode: argmax keys of the previous step (consumed + reset)
  const int* remap;          // optional [remap_n] old->new id table (-1 = dropped)
  int remap_n, unk_id;       // ids >= remap_n or unmapped -> unk_id
  const int* pos;            // [n_tok] positions, or null -> (*len_dev - pads[row])
  const int* len_dev;
  const int* pads;
  const int* type_ids;       // optional [n_tok] (null: every row uses type_const)
  int type_const;            // type row of rows without type_ids (generated tokens)
  const __half* tok_emb;     // [V, ldw]
  const __half* pos_emb;     // [P, ldw]
  const __half* type_emb;    // optional [n_types, ldw]
  int ldw;
  const float* ln_g;         // [H]
  const float* ln_b;
  __half* x;                 // [n_tok, ldx]
  __half* h;                 // [n_tok, ldx] (may be null: no LN)
  int ldx;
  int* tok_out;              // optional: ids actually embedded
};

template <int VPL>
__device__ __forceinline__ void ln_row_store(const float (&xv)[VPL], int H, const float* g,
                                             const float* b, __half* hrow, int lane) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c < H) s = __fadd_rn(s, xv[i]);
  }
  s = warp_sum(s);
  const float mean = __fdiv_rn(s, (float)H);
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c < H) {
      const float d = __fsub_rn(xv[i], mean);
      ss = __fadd_rn(ss, __fmul_rn(d, d));
    }
  }
  ss = warp_sum(ss);
  const float var = __fdiv_rn(ss, (float)H);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(var, 1e-5f)));
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    if (c < H) {
      const float d = __fsub_rn(xv[i], mean);
      hrow[c] = f16_sat(__fadd_rn(__fmul_rn(__fmul_rn(d, inv), g[c]), b[c]));
    }
  }
}

// ---- 16-byte vectorised variants (H % 8 == 0): lane owns 8-element chunks
// c8 = lane + 32*i; every load of the row (x, gamma, beta) is issued before the
// first use so one row costs ~one memory round trip.
template <int NC>
__device__ __forceinline__ void ln_load_gb(int H, const float* g, const float* b, int lane, float4 (&gv)[NC * 2],
                                           float4 (&bv)[NC * 2]) {
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < H) {
      gv[2 * i] = *reinterpret_cast<const float4*>(g + c);
      gv[2 * i + 1] = *reinterpret_cast<const float4*>(g + c + 4);
      bv[2 * i] = *reinterpret_cast<const float4*>(b + c);
      bv[2 * i + 1] = *reinterpret_cast<const float4*>(b + c + 4);
    }
  }
}

template <int NC>
__device__ __forceinline__ void ln_row_apply(float (&xv)[NC * 8], int H, const float4 (&gv)[NC * 2],
                                             const float4 (&bv)[NC * 2], __half* hrow, int lane) {
  float s = 0.0f;
#pragma unroll
  for (int i = 0; i < NC; ++i)
    if ((lane + 32 * i) * 8 < H)
#pragma unroll
      for (int e = 0; e < 8; ++e) s = __fadd_rn(s, xv[8 * i + e]);
  s = warp_sum(s);
  const float mean = __fdiv_rn(s, (float)H);
  float ss = 0.0f;
#pragma unroll
  for (int i = 0; i < NC; ++i)
    if ((lane + 32 * i) * 8 < H)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float d = __fsub_rn(xv[8 * i + e], mean);
        ss = __fadd_rn(ss, __fmul_rn(d, d));
      }
  ss = warp_sum(ss);
  const float inv = __fdiv_rn(1.0f, __fsqrt_rn(__fadd_rn(__fdiv_rn(ss, (float)H), 1e-5f)));
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < H) {
      const float* gf = reinterpret_cast<const float*>(&gv[2 * i]);
      const float* bf = reinterpret_cast<const float*>(&bv[2 * i]);
      float y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e)
        y[e] = __fadd_rn(__fmul_rn(__fmul_rn(__fsub_rn(xv[8 * i + e], mean), inv), gf[e]), bf[e]);
      *reinterpret_cast<uint4*>(hrow + c) = pack8(y);
    }
  }
}

template <int NC>
__device__ __forceinline__ void ln_row_vec(float (&xv)[NC * 8], int H, const float* g, const float* b, __half* hrow,
                                           int lane) {
  float4 gv[NC * 2], bv[NC * 2];
  ln_load_gb<NC>(H, g, b, lane, gv, bv);
  ln_row_apply<NC>(xv, H, gv, bv, hrow, lane);
}

template <int NC>
__global__ void __launch_bounds__(256) embed_ln_vec_kernel(const EmbedArgs a) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= a.n_tok) return;
  int id = (a.ids != nullptr) ? a.ids[row] : (int)argmax_id(a.keys[row]);
  if (a.remap != nullptr) {
    id = (id >= 0 && id < a.remap_n) ? a.remap[id] : -1;
    if (id < 0) id = a.unk_id;
  }
  const int p = (a.pos != nullptr) ? a.pos[row] : (*a.len_dev - a.pads[row]);
  const __half* tr = a.tok_emb + (size_t)id * a.ldw;
  const __half* pr = a.pos_emb + (size_t)p * a.ldw;
  const __half* yr = a.type_emb ? a.type_emb + (size_t)(a.type_ids ? a.type_ids[row] : a.type_const) * a.ldw : nullptr;
  uint4 tv[NC], pv[NC], yv[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < a.H) {
      tv[i] = *reinterpret_cast<const uint4*>(tr + c);
      pv[i] = *reinterpret_cast<const uint4*>(pr + c);
      if (yr) yv[i] = *reinterpret_cast<const uint4*>(yr + c);
    }
  }
  __half* xr = a.x + (size_t)row * a.ldx;
  float xv[NC * 8];
#pragma unroll
  for (int i = 0; i < NC; ++i) {
    const int c = (lane + 32 * i) * 8;
    if (c < a.H) {
      float t[8], q[8];
      unpack8(tv[i], t);
      unpack8(pv[i], q);
      float w[8];
      if (yr) unpack8(yv[i], w);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float v = __fadd_rn(t[e], q[e]);
        if (yr) v = __fadd_rn(v, w[e]);
        xv[8 * i + e] = q16(v);
      }
      *reinterpret_cast<uint4*>(xr + c) = pack8(&xv[8 * i]);
    } else {
#pragma unroll
      for (int e = 0; e < 8; ++e) xv[8 * i + e] = 0.0f;
    }
  }
  if (a.h != nullptr) ln_row_vec<NC>(xv, a.H, a.ln_g, a.ln_b, a.h + (size_t)row * a.ldx, lane);
  if (lane == 0 && a.tok_out) a.tok_out[row] = id;
  if (a.ids == nullptr && lane == 0) a.keys[row] = 0ull;
}

template <int VPL>
__global__ void __launch_bounds__(256) embed_ln_kernel(const EmbedArgs a) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= a.n_tok) return;
  int id;
  if (a.ids != nullptr) {
    id = a.ids[row];
  } else {
    id = (int)argmax_id(a.keys[row]);
  }
  if (a.remap != nullptr) {
    id = (id >= 0 && id < a.remap_n) ? a.remap[id] : -1;
    if (id < 0) id = a.unk_id;
  }
  const int p = (a.pos != nullptr) ? a.pos[row] : (*a.len_dev - a.pads[row]);
  const __half* tr = a.tok_emb + (size_t)id * a.ldw;
  const __half* pr = a.pos_emb + (size_t)p * a.ldw;
  const __half* yr = a.type_emb ? a.type_emb + (size_t)(a.type_ids ? a.type_ids[row] : a.type_const) * a.ldw : nullptr;
  __half* xr = a.x + (size_t)row * a.ldx;
  float xv[VPL];
#pragma unroll
  for (int i = 0; i < VPL; ++i) {
    const int c = lane + 32 * i;
    float v = 0.0f;
    if (c < a.H) {
      v = __fadd_rn(__half2float(tr[c]), __half2float(pr[c]));
      if (yr) v = __fadd_rn(v, __half2float(yr[c]));
      const __half hv = f16_sat(v);
      xr[c] = hv;
      v = __half2float(hv);
    }
    xv[i] = v;
  }
  if (a.h != nullptr) ln_row_store<VPL>(xv, a.H, a.ln_g, a.ln_b, a.h + (size_t)row * a.ldx, lane);
  if (lane == 0 && a.tok_out) a.tok_out[row] = id;
  if (a.ids == nullptr && lane == 0) a.keys[row] = 0ull;  // consumed: reset for the next argmax
}

struct LnArgs {
  int n_rows, H;
  const __half* x;  // source rows: x + (row * src_stride + src_off) * ldx
  int ldx, src_stride, src_off;
  const float* g;
  const float* b;
  __half* h;  // [n_rows, ldh]
  int ldh;
  int trace;  // diagnostics slot (0 = off)
  int early_trigger;  // release the next kernel before this kernel's dependency wait
};

template <int VPL>
__global__ void __launch_bounds__(256) layernorm_kernel(const LnArgs a) {
  pdl_wait();
  pdl_trigger();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row < a.n_rows) {
    const __half* xr = a.x + ((size_t)row * a.src_stride + a.src_off) * a.ldx;
    float xv[VPL];
#pragma unroll
    for (int i = 0; i < VPL; ++i) {
      const int c = lane + 32 * i;
      xv[i] = (c < a.H) ? __half2float(xr[c]) : 0.0f;
    }
    ln_row_store<VPL>(xv, a.H, a.g, a.b, a.h + (size_t)row * a.ldh, lane);
  }
}

template <int NC>
__global__ void __launch_bounds__(256) layernorm_vec_kernel(const LnArgs a) {
  TF_TRACE_INIT(tr);
  if (threadIdx.x == 0) tr.mark(a.trace, 0);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // gamma / beta are weights: loaded before the dependency wait
  float4 gv[NC * 2], bv[NC * 2];
  ln_load_gb<NC>(a.H, a.g, a.b, lane, gv, bv);
  if (a.early_trigger) pdl_trigger();  // the next GEMM may launch and prefetch its weights now
  pdl_wait();
  if (threadIdx.x == 0) tr.mark(a.trace, 1);
  if (!a.early_trigger) pdl_trigger();
  const int row = blockIdx.x * (blockDim.x >> 5) + warp;
  if (row < a.n_rows) {
    const __half* xr = a.x + ((size_t)row * a.src_stride + a.src_off) * a.ldx;
    uint4 raw[NC];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      const int c = (lane + 32 * i) * 8;
      if (c < a.H) raw[i] = *reinterpret_cast<const uint4*>(xr + c);
    }
    float xv[NC * 8];
#pragma unroll
    for (int i = 0; i < NC; ++i) {
      if ((lane + 32 * i) * 8 < a.H) {
        unpack8(raw[i], &xv[8 * i]);
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) xv[8 * i + e] = 0.0f;
      }
    }
    ln_row_apply<NC>(xv, a.H, gv, bv, a.h + (size_t)row * a.ldh, lane);
  }
  if (a.trace) {
    __syncthreads();
    if (threadIdx.x == 0) {
      tr.mark(a.trace, 7);
      tr.flush(a.trace);
    }
  }
}

// Step bookkeeping after the logits argmax: feed ids, append the generated
// token, advance the device-side cache length (model.py:651-666).
struct CollectArgs {
  int B;
  unsigned long long* keys;  // [B] consumed here only when consume != 0
  int* out_tokens;           // [B, max_new]
  int max_new;
  int* step_dev;             // generated-token counter
  int* len_dev;              // cache length
  int advance;               // tokens appended to the cache by this forward
};

__global__ void collect_kernel(const CollectArgs a) {
  pdl_wait();
  pdl_trigger();
  const int step = *a.step_dev;
  for (int b = threadIdx.x; b < a.B; b += blockDim.x) {
    const int tok = (int)argmax_id(a.keys[b]);
    if (step < a.max_new) a.out_tokens[(size_t)b * a.max_new + step] = tok;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.step_dev = step + 1;
    *a.len_dev += a.advance;
  }
}

}  // namespace tf
