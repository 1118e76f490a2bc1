// Beam-search step on the device (north star (3): "fused with a per-row argmax
// or top-k for greedy and beam search"). The reference has no beam search
// (SPEC.md:14, 183); semantics follow oracle/tinfer_oracle.py::beam_search_decode:
//
//   lp      = (x - max) - log(sum exp(x - max))        over f16-rounded logits, f32
//   cand    = score[beam] + lp[token]                  (f32)
//   frozen  : a finished beam proposes only (eos, score)
//   select  : top-K over the flat (beam, token) index, larger first, ties to the
//             lower flat index
//
// One CTA per request. The KV cache is never reordered: each row keeps an
// indirection table indir[b][slot] = which beam of the request wrote that slot
// (FasterTransformer-style cache indirection); the decode attention reads K/V
// through it. The selecting CTA rewrites its request's K rows of the table in
// place (parents are always in the same request) via a shared-memory stage.
#pragma once

#include "common.cuh"

namespace tf {

constexpr int kMaxBeam = 8;

struct BeamArgs {
  int R, K, V, cap, max_new;
  int eos;
  const __half* logits;  // [R*K, ldl]
  int ldl;
  float* scores;         // [R*K]
  unsigned char* finished;  // [R*K]
  int* tokens;           // [R*K] next token fed to each beam row
  int* tok_hist;         // [max_new, R*K]
  int* par_hist;         // [max_new, R*K] parent beam (within request)
  int* indir;            // [R*K, cap]
  const int* len_dev;    // cache length = slot the fed token will occupy
  int prompt_len;        // step index = *len_dev - prompt_len
  const int* pads;       // [R*K] left pads (the attention window of request r starts at pads[r*K])
  uint8_t* plan;         // [R][kBeamPlanBytes] next step's attention plans (cluster select), or null
};

struct Cand {
  float v;
  int i;  // flat index beam*V + token
};
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  return a.v > b.v || (a.v == b.v && a.i < b.i);
}

// insert into a descending top-K list (K <= kMaxBeam)
__device__ __forceinline__ void topk_insert(Cand (&t)[kMaxBeam], int K, Cand c) {
  if (!cand_better(c, t[K - 1])) return;
  int j = K - 1;
  while (j > 0 && cand_better(c, t[j - 1])) {
    t[j] = t[j - 1];
    --j;
  }
  t[j] = c;
}

// register form: a compare-and-swap pass over the (statically indexed) list;
// `worst` tracks top[K - 1] for the cheap rejection test
__device__ __forceinline__ void topk_insert_reg(Cand (&t)[kMaxBeam], int K, Cand c, Cand& worst) {
  if (!cand_better(c, worst)) return;
#pragma unroll
  for (int j = 0; j < kMaxBeam; ++j) {
    if (j < K && cand_better(c, t[j])) {
      const Cand x = t[j];
      t[j] = c;
      c = x;
    }
  }
#pragma unroll
  for (int j = 0; j < kMaxBeam; ++j)
    if (j == K - 1) worst = t[j];
}

__device__ __forceinline__ Cand cand_shfl_best(Cand c) {  // warp arg-best (total order: any tree)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const Cand x{__shfl_xor_sync(0xffffffffu, c.v, o), __shfl_xor_sync(0xffffffffu, c.i, o)};
    if (cand_better(x, c)) c = x;
  }
  return c;
}

// blockDim = kSelThreads; dynamic smem = K * cap ints (indirection staging)
constexpr int kSelThreads = 1024, kSelWarps = kSelThreads / 32;
// KB = beam width (compile time: the top-K list stays in registers)
template <int KB>
__global__ void __launch_bounds__(kSelThreads) beam_select_kernel(const BeamArgs a) {
  pdl_wait();
  __shared__ float s_max[kMaxBeam], s_lz[kMaxBeam], s_red2[kMaxBeam][kSelWarps];
  __shared__ Cand s_cand[kSelWarps];
  __shared__ int s_parent[kMaxBeam], s_tok[kMaxBeam];
  __shared__ float s_best[kMaxBeam];
  __shared__ unsigned char s_pfin[kMaxBeam];
  extern __shared__ int s_indir[];  // [K][cap]
  constexpr int K = KB;
  const int r = blockIdx.x, V = a.V;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int step = *a.len_dev - a.prompt_len;
  const int len = *a.len_dev;

  // ---- per-beam max and log(sum exp(x - max)) over the f16 logits, all K
  // rows per pass (per-row arithmetic and summation order unchanged)
  {
    const __half* rows = a.logits + (size_t)(r * K) * a.ldl;
    float m[kMaxBeam], z[kMaxBeam];
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k) m[k] = -INFINITY, z[k] = 0.0f;
    for (int v = tid; v < V; v += kSelThreads) {
#pragma unroll
      for (int k = 0; k < kMaxBeam; ++k)
        if (k < K) m[k] = fmaxf(m[k], __half2float(rows[(size_t)k * a.ldl + v]));
    }
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k) {
      m[k] = warp_max(m[k]);
      if (k < K && lane == 0) s_red2[k][warp] = m[k];
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k) {
      if (k < K) {
        float mm = s_red2[k][0];
        for (int w = 1; w < kSelWarps; ++w) mm = fmaxf(mm, s_red2[k][w]);
        m[k] = mm;
      }
    }
    for (int v = tid; v < V; v += kSelThreads) {
#pragma unroll
      for (int k = 0; k < kMaxBeam; ++k)
        if (k < K) z[k] += expf(__fsub_rn(__half2float(rows[(size_t)k * a.ldl + v]), m[k]));
    }
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k) z[k] = warp_sum(z[k]);
    __syncthreads();  // every thread has read s_red2 (max)
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k)
      if (k < K && lane == 0) s_red2[k][warp] = z[k];
    __syncthreads();
    if (tid < K) {
      float t = 0.0f;
      for (int w = 0; w < kSelWarps; ++w) t += s_red2[tid][w];
      s_lz[tid] = logf(t);
    }
#pragma unroll
    for (int k = 0; k < kMaxBeam; ++k)
      if (k < K && tid == 0) s_max[k] = m[k];
    __syncthreads();
  }
  // ---- per-thread top-K over this request's K*V candidates
  Cand top[kMaxBeam];
#pragma unroll
  for (int j = 0; j < kMaxBeam; ++j) top[j] = Cand{-INFINITY, 0x7fffffff};
  Cand worst = top[0];  // == top[K - 1]
  for (int k = 0; k < K; ++k) {
    const int b = r * K + k;
    const float sc = a.scores[b];
    if (a.finished[b]) {  // frozen: proposes only itself, with eos
      if (tid == 0) topk_insert_reg(top, K, Cand{sc, k * V + a.eos}, worst);
      continue;
    }
    if (sc == -INFINITY) continue;
    const float m = s_max[k], lz = s_lz[k];
    const __half* row = a.logits + (size_t)b * a.ldl;
    // 8 independent loads in flight per batch: the insert's dependency chain
    // through `worst` otherwise serialises one L2 round trip per element
    for (int v0 = tid; v0 < V; v0 += 8 * kSelThreads) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelThreads;
        x[u] = v < V ? __half2float(row[v]) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelThreads;
        if (v >= V) break;
        const float lp = __fsub_rn(__fsub_rn(x[u], m), lz);
        const Cand c{__fadd_rn(sc, lp), k * V + v};
        if (cand_better(c, worst)) topk_insert_reg(top, K, c, worst);
      }
    }
  }
  // ---- block merge: K rounds of arg-best over the per-thread list heads
  // (warp shuffles, then the warp winners; candidates are unique by index)
  int head = 0;
  for (int round = 0; round < K; ++round) {
    const Cand mine = head < K ? top[0] : Cand{-INFINITY, 0x7fffffff};
    const Cand wb = cand_shfl_best(mine);
    if (lane == 0) s_cand[warp] = wb;
    __syncthreads();
    if (warp == 0) {
      const Cand c = cand_shfl_best(lane < kSelWarps ? s_cand[lane] : Cand{-INFINITY, 0x7fffffff});
      if (lane == 0) s_cand[0] = c;
    }
    __syncthreads();
    const Cand best = s_cand[0];
    if (head < K && mine.i == best.i && mine.v == best.v) {  // owner pops its head (static shift)
      ++head;
#pragma unroll
      for (int j = 0; j + 1 < kMaxBeam; ++j) top[j] = top[j + 1];
      top[kMaxBeam - 1] = Cand{-INFINITY, 0x7fffffff};
    }
    if (tid == 0) {
      const int pb = best.i / V;
      s_parent[round] = pb;
      s_tok[round] = best.i - pb * V;
      s_best[round] = best.v;
    }
    __syncthreads();  // s_cand[0] read by all before the next round's writes
  }
  // ---- read everything the children inherit before any row is rewritten
  if (tid < K) s_pfin[tid] = a.finished[r * K + s_parent[tid]];
  for (int i = tid; i < K * len; i += kSelThreads) {
    const int k = i / len, s = i - k * len;
    s_indir[k * a.cap + s] = a.indir[(size_t)(r * K + k) * a.cap + s];
  }
  __syncthreads();
  const int span = min(len + 1, a.cap);
  for (int i = tid; i < K * span; i += kSelThreads) {
    const int k = i / span, s = i - k * span;
    a.indir[(size_t)(r * K + k) * a.cap + s] = (s < len) ? s_indir[s_parent[k] * a.cap + s] : k;
  }
  if (tid < K) {
    const int b = r * K + tid, tok = s_tok[tid];
    a.scores[b] = s_best[tid];
    a.finished[b] = (s_pfin[tid] || tok == a.eos) ? 1 : 0;
    a.tokens[b] = tok;
    if (step < a.max_new) {
      a.tok_hist[(size_t)step * (a.R * K) + b] = tok;
      a.par_hist[(size_t)step * (a.R * K) + b] = s_parent[tid];
    }
  }
  pdl_trigger();
}

// Cluster form: one 2..8-CTA cluster per request, CTA k owns beam row k (the
// K rows are scanned in parallel instead of by one CTA): per row the max, the
// log-sum-exp and the row's own top-K candidates (8 logits in flight per
// thread), then the leader CTA reads the K lists over DSMEM, picks the top K of
// the K*K candidates (same total order: larger score, then lower flat index)
// and rewrites the request's indirection rows, scores and histories.
constexpr int kSelCThreads = 512, kSelCWarps = kSelCThreads / 32;

__device__ __forceinline__ float sel_block_reduce(float v, bool is_max, float* s_red) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  v = is_max ? warp_max(v) : warp_sum(v);
  __syncthreads();  // s_red free
  if (lane == 0) s_red[warp] = v;
  __syncthreads();
  float t = s_red[0];
  for (int w = 1; w < kSelCWarps; ++w) t = is_max ? fmaxf(t, s_red[w]) : __fadd_rn(t, s_red[w]);
  return t;
}

template <int KB>
__global__ void __launch_bounds__(kSelCThreads) beam_select_cluster_kernel(const BeamArgs a) {
  pdl_wait();
  constexpr int K = KB;
  __shared__ float s_red[kSelCWarps];
  __shared__ Cand s_cand[kSelCWarps];
  __shared__ Cand s_list[kMaxBeam];
  __shared__ int s_parent[kMaxBeam], s_tok[kMaxBeam];
  __shared__ float s_best[kMaxBeam];
  __shared__ unsigned char s_pfin[kMaxBeam];
  extern __shared__ int s_indir[];  // [K][cap] (leader)
  const int k = (int)cluster_ctarank(), r = blockIdx.y, V = a.V;
  const int b = r * K + k;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int len = *a.len_dev;
  const int step = len - a.prompt_len;
  const float sc = a.scores[b];
  const bool fin = a.finished[b] != 0;
  Cand top[kMaxBeam];
#pragma unroll
  for (int j = 0; j < kMaxBeam; ++j) top[j] = Cand{-INFINITY, 0x7fffffff};
  Cand worst = top[0];
  if (fin) {  // frozen: proposes only itself, with eos
    if (tid == 0) topk_insert_reg(top, K, Cand{sc, k * V + a.eos}, worst);
  } else if (sc != -INFINITY) {
    const __half* row = a.logits + (size_t)b * a.ldl;
    float m = -INFINITY;
    for (int v0 = tid; v0 < V; v0 += 8 * kSelCThreads) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelCThreads;
        if (v < V) m = fmaxf(m, __half2float(row[v]));
      }
    }
    m = sel_block_reduce(m, true, s_red);
    float z = 0.0f;
    for (int v0 = tid; v0 < V; v0 += 8 * kSelCThreads) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelCThreads;
        if (v < V) z = __fadd_rn(z, expf(__fsub_rn(__half2float(row[v]), m)));
      }
    }
    const float lz = logf(sel_block_reduce(z, false, s_red));
    for (int v0 = tid; v0 < V; v0 += 8 * kSelCThreads) {
      float x[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelCThreads;
        x[u] = v < V ? __half2float(row[v]) : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = v0 + u * kSelCThreads;
        if (v >= V) break;
        const Cand c{__fadd_rn(sc, __fsub_rn(__fsub_rn(x[u], m), lz)), k * V + v};
        if (cand_better(c, worst)) topk_insert_reg(top, K, c, worst);
      }
    }
  }
  // ---- this row's top K: K rounds of arg-best over the per-thread list heads
  int head = 0;
  for (int round = 0; round < K; ++round) {
    const Cand mine = head < K ? top[0] : Cand{-INFINITY, 0x7fffffff};
    const Cand wb = cand_shfl_best(mine);
    if (lane == 0) s_cand[warp] = wb;
    __syncthreads();
    if (warp == 0) {
      const Cand c = cand_shfl_best(lane < kSelCWarps ? s_cand[lane] : Cand{-INFINITY, 0x7fffffff});
      if (lane == 0) s_cand[0] = c;
    }
    __syncthreads();
    const Cand best = s_cand[0];
    if (head < K && mine.i == best.i && mine.v == best.v) {
      ++head;
#pragma unroll
      for (int j = 0; j + 1 < kMaxBeam; ++j) top[j] = top[j + 1];
      top[kMaxBeam - 1] = Cand{-INFINITY, 0x7fffffff};
    }
    if (tid == 0) s_list[round] = best;
    __syncthreads();
  }
  cluster_sync();  // every row's list is in its CTA's shared memory
  if (k == 0) {
    if (tid == 0) {  // top K of the K x K candidates (unique flat indices)
      Cand t[kMaxBeam];
#pragma unroll
      for (int j = 0; j < kMaxBeam; ++j) t[j] = Cand{-INFINITY, 0x7fffffff};
      for (int q = 0; q < K; ++q) {
        const uint32_t base = dsmem_addr(smem_u32(s_list), (uint32_t)q);
        for (int j = 0; j < K; ++j) {
          Cand c;
          c.v = ld_dsmem_f32(base + 8u * j);
          uint32_t ci;
          asm volatile("ld.shared::cluster.u32 %0, [%1];" : "=r"(ci) : "r"(base + 8u * j + 4u));
          c.i = (int)ci;
          topk_insert(t, K, c);
        }
      }
      for (int j = 0; j < K; ++j) {
        const int pb = t[j].i / V;
        s_parent[j] = pb;
        s_tok[j] = t[j].i - pb * V;
        s_best[j] = t[j].v;
      }
    }
    __syncthreads();
    // ---- read everything the children inherit before any row is rewritten
    if (tid < K) s_pfin[tid] = a.finished[r * K + s_parent[tid]];
    for (int i = tid; i < K * len; i += kSelCThreads) {
      const int kk = i / len, sl = i - kk * len;
      s_indir[kk * a.cap + sl] = a.indir[(size_t)(r * K + kk) * a.cap + sl];
    }
    __syncthreads();
    const int span = min(len + 1, a.cap);
    for (int i = tid; i < K * span; i += kSelCThreads) {
      const int kk = i / span, sl = i - kk * span;
      a.indir[(size_t)(r * K + kk) * a.cap + sl] = (sl < len) ? s_indir[s_parent[kk] * a.cap + sl] : kk;
    }
    if (tid < K) {
      const int bb = r * K + tid, tok = s_tok[tid];
      a.scores[bb] = s_best[tid];
      a.finished[bb] = (s_pfin[tid] || tok == a.eos) ? 1 : 0;
      a.tokens[bb] = tok;
      if (step < a.max_new) {
        a.tok_hist[(size_t)step * (a.R * K) + bb] = tok;
        a.par_hist[(size_t)step * (a.R * K) + bb] = s_parent[tid];
      }
    }
    if (a.plan != nullptr) {
      // the next step's attention plan for this request (attention.cuh
      // kBeamPlanBytes): window [lo, hi = len], the new rows' source per slot,
      // per 64-slot chunk whether every beam reads the same rows (never the
      // chunk holding the newest slot, which is each beam's own), and the units
      uint8_t* P = a.plan + (size_t)r * kBeamPlanBytes;
      __shared__ int s_shc[64];
      const int lo = a.pads[r * K], hi = len, istr = 4096 / K;
      const int n = hi - lo + 1, nch = n > 0 ? (n + 63) / 64 : 0;
      auto nrow = [&](int kk, int sl) { return sl < len ? s_indir[s_parent[kk] * a.cap + sl] : kk; };
      for (int i = tid; i < K * n; i += kSelCThreads) {
        const int kk = i / n, k = i - kk * n;
        P[kk * istr + k] = (uint8_t)nrow(kk, lo + k);
      }
      for (int c = warp; c < nch; c += kSelCWarps) {
        bool same = true;
        for (int kq = c * 64 + lane; kq < c * 64 + 64; kq += 32) {
          const int sl = lo + kq;
          if (sl == hi) same = false;
          if (sl < hi) {
            const int s0 = nrow(0, sl);
            for (int q = 1; q < K; ++q) same = same && nrow(q, sl) == s0;
          }
        }
        same = __all_sync(0xffffffffu, same);
        if (lane == 0) s_shc[c] = same;
      }
      __syncthreads();
      if (warp == 0) {  // units in (half-chunk, beam) order, placed by a warp prefix sum
        int* U = reinterpret_cast<int*>(P + 4112);
        int base = 0;
        for (int h0 = 0; h0 < 2 * nch; h0 += 32) {
          const int hh = h0 + lane;
          const bool live = hh < 2 * nch && hh * 32 < n;
          const bool sh = live && s_shc[hh >> 1];
          const int cnt = live ? (sh ? 1 : K) : 0;
          int incl = cnt;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= o) incl += y;
          }
          const int u0 = base + incl - cnt;
          if (live) {
            if (sh) {
              U[u0] = hh << 8;
            } else {
              for (int q = 0; q < K; ++q) U[u0 + q] = (hh << 8) | (q + 1);
            }
          }
          base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (lane == 0) *reinterpret_cast<int*>(P + 4096) = base;
      }
    }
  }
  cluster_sync();  // the peers' lists stay alive until the leader has read them
  pdl_trigger();
}

}  // namespace tf
