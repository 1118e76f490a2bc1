/*
 * tinfer_sm100.h — C ABI of the B200 (sm_100a) Ernie generation path.
 *
 * The reference (`tinfer`, pure Python + numba) has no FFI layer; its hot path
 * sits behind two Python APIs:
 *   - the operator API `tinfer.kernels` (kernels.py:96-109 gemm_f32,
 *     kernels.py:216-233 attend_f32, kernels.py:112-126 bias_add/gelu), called
 *     only from model._gemm/_attend (model.py:407-437), and
 *   - the model API `tinfer.model` (_forward_tokens model.py:440-504, and the
 *     generate loop model.py:613-667) that the north star keeps.
 * This header is the C boundary that replaces both: the tf_gemm / tf_attention /
 * tf_embed_ln / tf_layernorm operators replace the numba kernels, and the
 * model/session runtime replaces _forward_tokens plus the decode loop. The
 * Python package `paper_2407_04991_b200` binds it with ctypes.
 *
 * Conventions
 *   - Every entry point returns an int status (tf_status); it never throws.
 *     tf_last_error() returns a thread-local message for the last failure.
 *   - All tensor arguments are DEVICE pointers owned by the caller. Streams are
 *     cudaStream_t passed as void*. One device per process.
 *   - Activations and weights are f16 (IEEE binary16) with f32 accumulation;
 *     every f32->f16 conversion is the reference's saturating RNE
 *     (tensor.py:95-100).
 *   - GEMM operands are K-major: activations [rows, ld] row-major, weights packed
 *     as W^T [out_features, ld] (the reference stores W as [in, out],
 *     model.py:190-207). K is zero-padded to a multiple of 64 (ld >= pad64(K)).
 *   - The ctypes call releases the GIL, preserving the reference kernels'
 *     nogil=True threading contract (kernels.py:42-233).
 */
#ifndef TINFER_SM100_H
#define TINFER_SM100_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TF_ABI_VERSION 2

enum tf_status {
  TF_OK = 0,
  TF_ERR_ARG = 1,         /* -> ParameterError */
  TF_ERR_SHAPE = 2,       /* -> DimensionError */
  TF_ERR_CUDA = 3,        /* -> DeviceError    */
  TF_ERR_UNSUPPORTED = 4, /* -> DeviceError    */
  TF_ERR_CAPACITY = 5     /* -> CapacityError  */
};

/* GEMM epilogues (fused; replaces the fused/unfused bias + GELU launches of
 * model._gemm, model.py:407-426, and the residual adds model.py:481/493). */
enum tf_epilogue {
  TF_EPI_F32 = 0,        /* out_f32 = acc                                   */
  TF_EPI_BIAS = 1,       /* out = q16(acc + bias)                           */
  TF_EPI_BIAS_GELU = 2,  /* out = q16(gelu_tanh(acc + bias))                */
  TF_EPI_BIAS_RESID = 3, /* out = q16(resid + q16(acc + bias))              */
  TF_EPI_QKV = 4,        /* q16(acc + bias) -> q buffer / K cache / V cache */
  TF_EPI_LOGITS = 5      /* q16(acc) -> logits and/or argmax keys           */
};

int tf_abi_version(void);
const char* tf_last_error(void);
/* SM count and compute capability of the current device. */
int tf_device_info(int* sm_count, int* cc_major, int* cc_minor);

/* ------------------------------------------------------------------ operators */

/* out[m_tok, n_feat] = epilogue(act[m_tok, k] . wt[n_feat, k]^T).
 * Replaces kernels.gemm_f32 (kernels.py:96-109) + bias_add/gelu (112-126). */
typedef struct tf_gemm_desc {
  int m_tok, n_feat, k;
  const void* act; int lda;      /* f16 [m_tok, lda]                              */
  const void* wt; int ldw;       /* f16 [n_feat, ldw]                             */
  int epilogue;                  /* tf_epilogue                                   */
  const float* bias;             /* [n_feat] or NULL (EPI_F32 / EPI_LOGITS)       */
  void* out; int ldo;            /* f16 (or f32 for TF_EPI_F32) [m_tok, ldo]      */
  const void* resid; int ldr;    /* TF_EPI_BIAS_RESID: f16 [m_tok, ldr]           */
  /* TF_EPI_QKV: features [0,H) -> q_out[tok, ldq]; [H,2H) / [2H,3H) -> cache
   * [B, heads, cap, head_dim] at slot (*qbase_dev + tok % seq_len), B = tok / seq_len */
  void* q_out; int ldq;
  void* k_cache; void* v_cache;
  int hidden, heads, head_dim, cap, seq_len;
  const int* qbase_dev;
  unsigned long long* argmax_keys; /* TF_EPI_LOGITS: [m_tok] packed keys (zeroed) or NULL */
  float* workspace; size_t workspace_bytes; /* reserved (split-K reduces via DSMEM)  */
  int* counters; int n_counters;            /* reserved                              */
  int force_swap;                /* -1 auto (swap-AB when m_tok <= 256), 0, 1      */
  int splits;                    /* 0 auto; else divides ceil(k/64), <= 16 (cluster) */
  int pdl;                       /* programmatic dependent launch: 0 off, 1 on (the
                                    next kernel may launch once this one is set up),
                                    2 on, next kernel released only after this
                                    kernel's own dependency wait                   */
  /* optional LayerNorm folded into the GEMM (swap-AB only; epilogues F32 /
   * BIAS / BIAS_GELU / QKV / LOGITS): act holds the raw rows x, wt the weights
   * with gamma folded over K (W'[n][k] = q16(W[n][k] * gamma[k])), and the
   * accumulator becomes inv_t * (x_t . W'_n - mean_t * ln_c[n]) + ln_d[n]
   * (= LN(x_t) . W_n, tensor.py:153-160) before the epilogue, with
   * ln_c[n] = sum_k W'[n][k] and ln_d[n] = sum_k beta[k] W[n][k]. Row t's
   * (mean, inv) over ln_hidden features are merged from the float pairs
   * ln_stats[2 * (i * ln_stats_ld + t) + {0, 1}] = (mean, M2) of features
   * [128 i, 128 i + 128) that a TF_EPI_BIAS_RESID GEMM wrote through stats_out;
   * ln_hidden <= 2048, ln_stats_ld >= m_tok */
  const float* ln_stats; int ln_stats_ld, ln_hidden;
  const float* ln_c; const float* ln_d;
  /* TF_EPI_BIAS_RESID, swap-AB split-K: also write those per-tile (mean, M2)
   * pairs of the output rows to stats_out[2 * (tile * stats_ld + t)] */
  float* stats_out; int stats_ld;
} tf_gemm_desc;
int tf_gemm(const tf_gemm_desc* d, void* stream);

/* x = q16(tok_emb[id] + pos_emb[p] (+ type_emb[t])); h = q16(LN(x)) (h optional).
 * Type rows: type_ids[tok] when given, else type_const (type_emb NULL: none).
 * Replaces the gather-sum of model.py:453-455 / embed (model.py:521-534) and the
 * first layer_norm_f32 (tensor.py:153-160). `remap` (optional) maps original ids
 * to pruned ids (pruning.py:50-52); ids outside the map go to unk_id
 * (SPEC.md:306). */
typedef struct tf_embed_desc {
  int n_tok, hidden, vocab, max_pos;
  const int* ids; const int* pos; const int* type_ids; int type_const;
  const int* remap; int remap_n; int unk_id;
  const void* tok_emb; const void* pos_emb; const void* type_emb; int ldw;
  const float* ln_gamma; const float* ln_beta;
  void* x; void* h; int ldx;
  int* ids_out;
} tf_embed_desc;
int tf_embed_ln(const tf_embed_desc* d, void* stream);

/* h[r] = q16(LN(x[r * src_stride + src_off])) (tensor.py:153-160). */
int tf_layernorm(int n_rows, int hidden, const void* x, int ldx, int src_stride, int src_off,
                 const float* gamma, const float* beta, void* h, int ldh, void* stream);

/* Beam-search decode attention (one query row per beam; no reference
 * counterpart: SPEC.md:14 lists beam search as a non-goal, the semantics are the
 * oracle's restatement on attend_f32, kernels.py:148-180). Rows of request r are
 * beams r*beam .. r*beam+beam-1; slot s (< *qbase_dev) of row b is read from row
 * (b / beam) * beam + indir[b * cap + s] (the cache indirection the beam select
 * maintains), the newest slot *qbase_dev from indir[b * cap + *qbase_dev]; every
 * beam of a request shares the window [start[r * beam], *qbase_dev]. */
int tf_attention_beam(int requests, int beam, int heads, int head_dim, int cap, const void* q, int ldq,
                      const void* k_cache, const void* v_cache, const int* start, const int* qbase_dev,
                      const int* indir, float scale, void* out, int ldo, void* stream);

/* ---- weight packing on the device (model upload; TINF direct-to-device load,
 * replacing the host-side load_model -> Model.f32 path of model.py:177-184 /
 * 267-286 for the device mirror). All three are enqueued on `stream`.
 * tf_pack_kmajor: src [K, N] row-major (reference [in, out] layout, f32 when
 * src_f32 else f16) -> dst f16 [N, ldk] (W^T, K-major, columns >= K zeroed),
 * saturating RNE; with gamma (f32, f16-rounded values): q16(q16(src) * gamma[k]).
 * tf_fold_terms: per output feature n, c[n] = sum_k w_ln_t[n, k] and
 * d[n] = sum_k beta[k] * w_t[n, k] (f64 accumulation, rounded to f32): the
 * LayerNorm fold terms of the decode GEMMs.
 * tf_convert: dst[i] = q16(src[i]) stored as f32 (dst_f32) or f16. */
int tf_pack_kmajor(const void* src, int src_f32, int K, int N, const float* gamma, void* dst, int ldk,
                   void* stream);
int tf_fold_terms(const void* w_t, const void* w_ln_t, const float* beta, int K, int N, int ldk, float* c,
                  float* d, void* stream);
int tf_convert(const void* src, int src_f32, long long n, void* dst, int dst_f32, void* stream);

/* Masked attention over the KV cache (kernels.attend_f32, kernels.py:216-233).
 * q: [batch*seq_len, ldq] (head h at columns h*head_dim); caches [batch, heads,
 * cap, head_dim]; row t of sequence b attends slots [start[b], *qbase_dev + t].
 * seq_len == 1 selects the decode kernels of the generation path (for head_dim
 * 64 with split-KV partials + arrival counters allocated stream-ordered on
 * `stream` for the call: cudaMallocAsync / cudaFreeAsync). */
int tf_attention(int batch, int heads, int head_dim, int cap, int seq_len, const void* q, int ldq,
                 const void* k_cache, const void* v_cache, const int* start, const int* qbase_dev,
                 float scale, void* out, int ldo, void* stream);

/* ------------------------------------------------------------------ model runtime */

typedef struct tf_layer_weights {
  const float* ln1_gamma; const float* ln1_beta;
  const void* wqkv_t; const float* bqkv; /* [3H, ldk_h] f16, [3H] f32 */
  const void* wo_t; const float* bo;     /* [H, ldk_h], [H]            */
  const float* ln2_gamma; const float* ln2_beta;
  const void* w1_t; const float* b1;     /* [F, ldk_h], [F]            */
  const void* w2_t; const float* b2;     /* [H, ldk_f], [H]            */
  /* optional LayerNorm-folded copies for the decode path (see tf_gemm_desc):
   * attn_norm folded into Wqkv, ffn_norm into W1 (NULL: stand-alone LN) */
  const void* wqkv_ln_t; const float* cqkv; const float* dqkv;
  const void* w1_ln_t; const float* c1; const float* d1;
} tf_layer_weights;

typedef struct tf_model_desc {
  int vocab, hidden, layers, heads, head_dim, ffn, max_pos;
  int ldk_h, ldk_f;                      /* padded K strides for H and F inputs */
  const void* tok_emb; const void* pos_emb; const void* type_emb; int n_types; int ldw;
  const tf_layer_weights* layer;         /* [layers] */
  const float* final_gamma; const float* final_beta;
  const void* lm_head_t;                 /* [vocab, ldk_h] f16 */
  const void* lm_head_ln_t; const float* c_lm; const float* d_lm; /* final_norm folded (optional) */
} tf_model_desc;
int tf_model_create(const tf_model_desc* d, void** model);
int tf_model_destroy(void* model);

/* A generation session: one batch, its KV cache and scratch (all caller-owned). */
typedef struct tf_session_desc {
  int batch, capacity, max_tokens, max_new;
  void* k_cache; void* v_cache;          /* [layers, batch, heads, capacity, head_dim] f16 */
  void* x; void* h; void* q; void* attn; /* [batch*max_tokens, ldk_h] f16 */
  void* ffn;                             /* [batch*max_tokens, ldk_f] f16 */
  void* logits;                          /* optional [batch*max_tokens, vocab] f16 */
  float* workspace; size_t workspace_bytes; /* split-KV decode attention partials:
                                             * batch*heads*ceil(capacity/64)*66 floats */
  int* counters; int n_counters;         /* batch*heads zeroed arrival counters */
  unsigned long long* keys;              /* [batch] argmax keys (zeroed) */
  int* len_dev; int* step_dev;           /* device scalars */
  int* out_tokens;                       /* [batch, max_new] */
  const int* pads;                       /* [batch] left-pad offsets = first valid slot */
  const int* remap; int remap_n; int unk_id;  /* optional prompt-id remap */
  int* beam_indir; int beam;             /* beam search: [batch, capacity] slot->beam table, width */
  /* fused decode LayerNorms: 4 * ceil(hidden/128) * batch * max_tokens floats
   * (NULL: stand-alone LayerNorm kernels) */
  float* ln_stats; size_t ln_stats_bytes;
  /* type embeddings (model type_emb set): prompt rows' type ids [batch*max_tokens]
   * (NULL: gen_type for every row) and the type of generated tokens */
  const int* type_ids; int gen_type;
} tf_session_desc;
int tf_session_create(void* model, const tf_session_desc* d, void** session);
int tf_session_destroy(void* session);

enum tf_forward_mode {
  TF_FWD_ARGMAX = 0,      /* last-row logits -> argmax -> out_tokens[:, step]; step++ */
  TF_FWD_LOGITS_LAST = 1, /* last-row f16 logits -> logits[batch, vocab]              */
  TF_FWD_LOGITS_ALL = 2   /* every row's f16 logits -> logits[batch*T, vocab]        */
};
/* Run T new tokens per sequence through every layer (model._forward_tokens,
 * model.py:440-504): K/V appended at slots [len, len+T), len += T afterwards.
 * ids/pos: device [batch*T] (pos may be NULL -> len - pads). ids may be NULL
 * (T == 1): feed the previous argmax. */
int tf_forward(void* session, const int* ids, const int* pos, int T, int mode, int pdl,
               void* stream);
/* tf_forward that also copies the residual stream at every LayerNorm input
 * (2L+1 taps: the embedding sum, then after each layer's Wo and FFN2 residual
 * adds; the reference's layer_norm_f32 call sites model.py:460, 484, 497) into
 * taps, device f16 [2L+1][batch*T][hidden]. Diagnostics for hidden-state parity. */
int tf_forward_taps(void* session, const int* ids, const int* pos, int T, int mode, void* taps,
                    void* stream);
/* n greedy decode steps (model.py:651-666), each a T=1 TF_FWD_ARGMAX forward fed
 * by the previous argmax; with use_graph the step is captured once into a CUDA
 * graph and replayed. */
int tf_decode(void* session, int n_steps, int use_graph, void* stream);
/* Beam search (no reference implementation; semantics in DESIGN.md §6):
 * rows b = r*beam + k. After a forward that produced last-row logits, one step
 * selects, per request, the top-`beam` (beam, token) candidates by
 * score + log_softmax(f16 logits), ties to the lower flat index; finished beams
 * propose only (eos, score). Updates scores/finished/tokens, records token and
 * parent histories at step = len - prompt_len, and rewrites the cache
 * indirection table (the KV cache itself is never reordered). */
typedef struct tf_beam_desc {
  int requests, beam, max_new, prompt_len, eos;
  float* scores;              /* [requests*beam], init 0 for beam 0 and -inf otherwise */
  unsigned char* finished;    /* [requests*beam] */
  int* tokens;                /* [requests*beam] next fed ids */
  int* tok_hist; int* par_hist; /* [max_new, requests*beam] */
} tf_beam_desc;
int tf_beam_select(void* session, const tf_beam_desc* d, void* stream);
/* n steps of (T=1 forward of `tokens` -> last-row logits -> tf_beam_select),
 * captured once into a CUDA graph when use_graph. */
int tf_beam_decode(void* session, const tf_beam_desc* d, int n_steps, int use_graph, void* stream);

/* Diagnostics (host env TF_TRACE=1): kernels launched after a reset store
 * %globaltimer stamps of up to 8 points per CTA; reset != 0 clears them,
 * otherwise copies [slot][2048 CTAs][8] u64 (0 = absent; 0 = entry, 1 = past the
 * PDL wait, 7 = exit, the rest kernel-specific) for up to max_slots slots into
 * dst and their kernel names into names; returns the slot count (>= 0) or a
 * negative tf_status. */
int tf_debug_trace(int reset, unsigned long long* dst, int max_slots, const char** names);

/* Kernels launched by one decode step (for the bench's gpu_launches count). */
int tf_session_launches_per_step(void* session);

#ifdef __cplusplus
}
#endif
#endif /* TINFER_SM100_H */
