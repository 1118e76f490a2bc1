// C-ABI implementation: operator launchers + the native generation runtime
// (model / session / forward / graph-captured decode loop). See
// include/tinfer_sm100.h for the contract and the reference interfaces each
// entry point replaces.
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/tinfer_sm100.h"
#include "attention.cuh"
#include "beam.cuh"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "norm_embed.cuh"
#include "pack.cuh"

using namespace tf;

// ------------------------------------------------------------------ errors
static thread_local std::string g_last_error;

namespace {

struct TfError {
  int code;
  std::string msg;
};

#define TF_CHECK_CUDA(expr)                                                             \
  do {                                                                                  \
    cudaError_t _e = (expr);                                                            \
    if (_e != cudaSuccess)                                                              \
      throw TfError{TF_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)};   \
  } while (0)

#define TF_REQUIRE(cond, code, msg)                  \
  do {                                               \
    if (!(cond)) throw TfError{(code), (msg)};       \
  } while (0)

template <class F>
int guarded(F&& f) {
  try {
    f();
    return TF_OK;
  } catch (const TfError& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return TF_ERR_CUDA;
  }
}

int pad64(int k) { return (k + 63) / 64 * 64; }

// ------------------------------------------------------------------ TMA maps
PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;
std::once_flag g_encode_once;

void load_encoder() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  });
  TF_REQUIRE(g_encode != nullptr, TF_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
}

// K-major f16 matrix [rows, ld]; box = 64 (K) x box_rows, 128-byte swizzle,
// out-of-bounds rows/columns read as zero.
CUtensorMap make_kmajor_map(const void* ptr, int rows, int k_extent, int ld, int box_rows) {
  load_encoder();
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)k_extent, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1u, 1u};
  CUresult r = g_encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 2, const_cast<void*>(ptr), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  TF_REQUIRE(r == CUDA_SUCCESS, TF_ERR_ARG,
             "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + "): rows=" +
                 std::to_string(rows) + " k=" + std::to_string(k_extent) +
                 " ld=" + std::to_string(ld));
  return m;
}

// ------------------------------------------------------------------ launch helper
template <typename Kern, typename... Args>
void launch_cluster3(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, dim3 cluster,
                     Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  attr[n].id = cudaLaunchAttributeClusterDimension;
  attr[n].val.clusterDim.x = cluster.x;
  attr[n].val.clusterDim.y = cluster.y;
  attr[n].val.clusterDim.z = cluster.z;
  ++n;
  cfg.attrs = attr;
  cfg.numAttrs = n;
  TF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <typename Kern, typename... Args>
void launch_cluster(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
                    int cluster_z, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  int n = 0;
  if (pdl) {
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n].val.programmaticStreamSerializationAllowed = 1;
    ++n;
  }
  if (cluster_z > 1) {
    attr[n].id = cudaLaunchAttributeClusterDimension;
    attr[n].val.clusterDim.x = 1;
    attr[n].val.clusterDim.y = 1;
    attr[n].val.clusterDim.z = (unsigned)cluster_z;
    ++n;
  }
  cfg.attrs = n ? attr : nullptr;
  cfg.numAttrs = n;
  TF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern, args...));
}

template <typename Kern, typename... Args>
void launch(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl,
            Args... args) {
  launch_cluster(kern, grid, block, smem, st, pdl, 1, args...);
}

// Kernel attributes are per device: set them once per (kernel, device) pair
// (a process may drive several GPUs through several DeviceModels).
int current_device() {
  int dev = 0;
  TF_CHECK_CUDA(cudaGetDevice(&dev));
  return dev;
}
bool attr_once(const void* fn) {
  static std::mutex mu;
  static std::set<std::pair<const void*, int>> done;
  const int dev = current_device();
  std::lock_guard<std::mutex> g(mu);
  return done.insert({fn, dev}).second;
}

// Every SM keeps the maximum shared-memory carveout, whatever kernel runs on
// it: with programmatic dependent launch the next kernel's CTAs are placed
// while the current kernel's are resident, and an SM configured for a small
// carveout cannot take them until it drains.
template <typename K>
void set_max_carveout(K kern) {
  TF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                     (int)cudaSharedmemCarveoutMaxShared));
}
// max dynamic smem + carveout (+ non-portable clusters) once per (kernel, device)
template <typename K>
void ensure_attr(K kern, size_t max_smem, bool big_cluster = false) {
  if (!attr_once(reinterpret_cast<const void*>(kern))) return;
  if (max_smem > 48 * 1024)
    TF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)max_smem));
  if (big_cluster) TF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  set_max_carveout(kern);
}
template <typename Kern, typename... Args>
void launch_mc(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  ensure_attr(kern, 0);
  launch_cluster(kern, grid, block, smem, st, pdl, 1, args...);
}

int num_sms() {
  static int per_dev[64] = {0};
  const int dev = current_device();
  if (dev < 0 || dev >= 64) throw TfError{TF_ERR_UNSUPPORTED, "device ordinal >= 64"};
  if (per_dev[dev] == 0) TF_CHECK_CUDA(cudaDeviceGetAttribute(&per_dev[dev], cudaDevAttrMultiProcessorCount, dev));
  return per_dev[dev];
}

// ------------------------------------------------------------------ tracing (diagnostics)
bool trace_on() {
  static const bool on = [] {
    const char* e = getenv("TF_TRACE");
    return e && e[0] == '1';
  }();
  return on;
}
int g_trace_n = 0;
const char* g_trace_names[kTraceSlots];
int trace_next(const char* name) {
  if (!trace_on() || g_trace_n >= kTraceSlots) return 0;
  g_trace_names[g_trace_n] = name;
  return ++g_trace_n;
}

// dynamic smem budget: 227 KB per CTA minus room for the kernels' static smem
constexpr size_t kMaxSmem = 227 * 1024 - 1024;

template <int MODE, bool SWAP, int RED, int LNV>
void ensure_gemm_attr() {
  ensure_attr(gemm_tc_kernel<MODE, SWAP, RED, LNV>, kMaxSmem, true);
}

// ------------------------------------------------------------------ GEMM planning
struct GemmPlan {
  bool swap;
  int bn, tiles_a, tiles_b, k_blocks, splits, stages;
};

// Deterministic split count: a function of (features, K) for batches of <= 2
// row tiles (<= 128 rows; batch-invariant), of (features, K, row tiles) above. Splits form one cluster per
// tile: up to 8 (portable) when there are many tiles, up to 16 (non-portable,
// one cluster per GPC) when a few tiles must cover the machine.
// The largest split count whose grid stays within 128 CTAs: every cluster is
// then co-resident in one wave (a 144-CTA grid of 6-CTA clusters measured a
// second wave at batch 128: FFN1 22 -> 13 us).
int pick_splits(int tiles, int k_blocks) {
  const int target = 128;
  const int cap = tiles >= 16 ? 8 : 16;
  int best = 1;
  for (int d = 1; d <= k_blocks && d <= cap; ++d) {
    if (k_blocks % d) continue;
    if (tiles * d > target) break;
    best = d;
  }
  return best;
}

GemmPlan plan_gemm(const tf_gemm_desc& d) {
  GemmPlan p{};
  p.k_blocks = (d.k + 63) / 64;
  p.swap = d.force_swap >= 0 ? d.force_swap != 0 : d.m_tok <= 256;
  if (p.swap) {
    // decode batch tile: <= 64 rows for the split-K GEMMs (batch 128: two row
    // tiles with half the split count each -> smaller partial tiles to reduce;
    // C3 step 798 -> 714 us); the argmax lm_head keeps whole-batch tiles.
    // TF_BN_MAX overrides (A/B)
    static const int bn_max = [] {
      const char* e = getenv("TF_BN_MAX");
      return e ? atoi(e) : 64;
    }();
    static const int lm_bn = [] {  // TF_LM_BN: batch tile of the full-K logits GEMM (A/B; 128 vs 256: C4 772 vs 788 us)
      const char* e = getenv("TF_LM_BN");
      return e ? atoi(e) : 128;
    }();
    const int cap_bn = d.epilogue == TF_EPI_LOGITS ? lm_bn : bn_max;
    const int mt = d.m_tok < cap_bn ? d.m_tok : cap_bn;
    p.bn = ((mt + 15) / 16) * 16;
    if (p.bn < 16) p.bn = 16;
    p.tiles_a = (d.n_feat + 127) / 128;
    p.tiles_b = (d.m_tok + p.bn - 1) / p.bn;
  } else {
    // 128-wide feature tiles with a 3-stage ring: two CTAs per SM, so one's
    // epilogue overlaps the other's main loop (C2 prefill GEMMs 2.57 -> 1.86 ms)
    p.bn = 128;
    if (d.n_feat < p.bn) p.bn = ((d.n_feat + 15) / 16) * 16;
    if (p.bn < 16) p.bn = 16;
    p.tiles_a = (d.m_tok + 127) / 128;
    p.tiles_b = (d.n_feat + p.bn - 1) / p.bn;
  }
  if (d.splits > 0) {
    TF_REQUIRE(p.k_blocks % d.splits == 0, TF_ERR_ARG, "splits must divide ceil(k/64)");
    TF_REQUIRE(d.splits <= 16, TF_ERR_ARG, "splits (cluster size) must be <= 16");
    p.splits = d.splits;
  } else {
    // up to two 64-row batch tiles take the one-tile split count, so a row's
    // f32 summation order is the same for every batch of <= 128 rows (batched ==
    // single bitwise, model.py:8-13; C3 -2.7%); larger batches trade it for one
    // wave of clusters (at 256 rows the one-tile count costs C4 18%)
    p.splits = (p.swap && d.epilogue != TF_EPI_LOGITS)
                   ? pick_splits(p.tiles_a * (p.tiles_b <= 2 ? 1 : p.tiles_b), p.k_blocks)
                   : 1;
  }
  TF_REQUIRE(p.splits == 1 || d.epilogue != TF_EPI_LOGITS, TF_ERR_ARG,
             "argmax epilogue does not support split-K");
  const int kb_per = p.k_blocks / p.splits;
  const int stage_bytes = gemm_stage_bytes(p.bn);
  const size_t ln_bytes = (p.swap && d.ln_stats) ? gemm_ln_bytes(p.bn) : 0;
  int st = (int)((kMaxSmem - 4096 - ln_bytes - gemm_recv_bytes(p.bn, p.splits, p.swap)) / stage_bytes);
  if (!p.swap) {  // leave room for the staged output tile (smem-bytes check below)
    while (st > 1 && gemm_smem_bytes(p.bn, st, p.splits, false) > kMaxSmem) --st;
    if (st > 3) st = 3;  // two CTAs per SM (prefill)
  }
  if (st > 8) st = 8;
  // many independent full-K tiles (lm_head): a shallow ring lets 3 CTAs share
  // an SM so one CTA's epilogue overlaps the others' weight streaming
  static const int lm_st = [] {  // TF_LM_STAGES: ring depth of these many-tile full-K GEMMs (A/B)
    const char* e = getenv("TF_LM_STAGES");
    return e ? atoi(e) : 3;
  }();
  if (p.swap && p.splits == 1 && p.tiles_a * p.tiles_b > 148 && st > lm_st) st = lm_st;
  if (st > kb_per) st = kb_per;
  if (st < 1) st = 1;
  p.stages = st;
  return p;
}

// a residual GEMM of this plan can emit the row statistics of its output
// (push split-K reduction, whole token columns per warp)
bool plan_emits_stats(const GemmPlan& p) { return p.swap && gemm_push_reduce(p.bn, p.splits, true); }

template <int MODE, bool SWAP, int RED, int LNV>
void launch_gemm_v(const tf_gemm_desc& d, const GemmPlan& p, const CUtensorMap& ta, const CUtensorMap& tb,
                   const GemmArgs& args, cudaStream_t st) {
  ensure_gemm_attr<MODE, SWAP, RED, LNV>();
  dim3 grid(p.tiles_a, p.tiles_b, p.splits);
  const size_t ln_bytes = LNV == 1 ? gemm_ln_bytes(p.bn) : 0;
  const size_t smem = gemm_smem_bytes(p.bn, p.stages, p.splits, SWAP, ln_bytes);
  launch_cluster(gemm_tc_kernel<MODE, SWAP, RED, LNV>, grid, dim3(gemm_threads(MODE, SWAP, RED, LNV)), smem, st,
                 d.pdl != 0, p.splits, ta, tb, args);
}

// One kernel instantiation per (epilogue, operand order, reduction path,
// operand LayerNorm): each carries only the code it executes.
template <int MODE, bool SWAP>
void launch_gemm_t(const tf_gemm_desc& d, const GemmPlan& p, const CUtensorMap& ta,
                   const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st) {
  const int red = p.splits == 1 ? RED_ONE : (gemm_push_reduce(p.bn, p.splits, SWAP) ? RED_PUSH : RED_PULL);
  if constexpr (!SWAP) {
    if (red == RED_ONE) return launch_gemm_v<MODE, false, RED_ONE, 0>(d, p, ta, tb, args, st);
    return launch_gemm_v<MODE, false, RED_PULL, 0>(d, p, ta, tb, args, st);
  } else {
    if (!d.ln_stats) {
      if (red == RED_ONE) return launch_gemm_v<MODE, true, RED_ONE, 0>(d, p, ta, tb, args, st);
      if (red == RED_PUSH) return launch_gemm_v<MODE, true, RED_PUSH, 0>(d, p, ta, tb, args, st);
      return launch_gemm_v<MODE, true, RED_PULL, 0>(d, p, ta, tb, args, st);
    }
    constexpr bool ln_ok =
        MODE == EPI_F32 || MODE == EPI_QKV || MODE == EPI_BIAS_GELU || MODE == EPI_BIAS || MODE == EPI_LOGITS;
    if constexpr (ln_ok) {
      if (red == RED_ONE) return launch_gemm_v<MODE, true, RED_ONE, 1>(d, p, ta, tb, args, st);
      if (red == RED_PUSH) return launch_gemm_v<MODE, true, RED_PUSH, 1>(d, p, ta, tb, args, st);
      return launch_gemm_v<MODE, true, RED_PULL, 1>(d, p, ta, tb, args, st);
    }
    throw TfError{TF_ERR_UNSUPPORTED, "gemm: fused operand LayerNorm not built for this epilogue"};
  }
}

template <int MODE>
void launch_gemm_mode(const tf_gemm_desc& d, const GemmPlan& p, const CUtensorMap& ta,
                      const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st) {
  if (p.swap)
    launch_gemm_t<MODE, true>(d, p, ta, tb, args, st);
  else
    launch_gemm_t<MODE, false>(d, p, ta, tb, args, st);
}

// runtime-internal GEMM options (not part of the operator ABI)
struct GemmExtra {
  const void* l2pf = nullptr;  // HBM -> L2 prefetch range (next layer's operand)
  unsigned long long l2pf_bytes = 0;
};

void run_gemm(const tf_gemm_desc& d, cudaStream_t st, const GemmExtra& ex = GemmExtra{}) {
  TF_REQUIRE(d.m_tok > 0 && d.n_feat > 0 && d.k > 0, TF_ERR_SHAPE, "gemm: empty shape");
  TF_REQUIRE(d.act && d.wt, TF_ERR_ARG, "gemm: null operand");
  const GemmPlan p = plan_gemm(d);
  const int kext = p.k_blocks * 64;
  TF_REQUIRE(d.lda >= kext && d.ldw >= kext, TF_ERR_SHAPE,
             "gemm: leading dimensions must cover K padded to a multiple of 64");
  TF_REQUIRE(d.lda % 8 == 0 && d.ldw % 8 == 0, TF_ERR_SHAPE, "gemm: ld must be a multiple of 8");
  GemmArgs a{};
  a.rows_a = p.swap ? d.n_feat : d.m_tok;
  a.rows_b = p.swap ? d.m_tok : d.n_feat;
  a.k_blocks = p.k_blocks;
  a.splits = p.splits;
  a.kb_per_split = p.k_blocks / p.splits;
  a.bn = p.bn;
  a.stages = p.stages;
  a.m_tok = d.m_tok;
  a.n_feat = d.n_feat;
  a.bias = d.bias;
  a.out = static_cast<__half*>(d.out);
  a.out_f32 = static_cast<float*>(d.out);
  a.ldo = d.ldo;
  a.resid = static_cast<const __half*>(d.resid);
  a.ldr = d.ldr;
  a.q_out = static_cast<__half*>(d.q_out);
  a.ldq = d.ldq;
  a.kc = static_cast<__half*>(d.k_cache);
  a.vc = static_cast<__half*>(d.v_cache);
  a.H = d.hidden;
  a.NH = d.heads;
  a.D = d.head_dim;
  a.cap = d.cap;
  a.T = d.seq_len;
  a.qbase_dev = d.qbase_dev;
  a.keys = d.argmax_keys;
  a.late_trigger = d.pdl == 2 ? 1 : 0;
  a.l2pf = ex.l2pf;
  a.l2pf_bytes = ex.l2pf_bytes;
  static const char* kGemmNames[] = {"gemm_f32", "gemm_bias", "gemm_gelu", "gemm_resid", "gemm_qkv", "gemm_logits"};
  a.trace = trace_next(d.epilogue >= 0 && d.epilogue < 6 ? kGemmNames[d.epilogue] : "gemm");
  if (d.ln_stats) {
    TF_REQUIRE(p.swap, TF_ERR_UNSUPPORTED, "gemm: fused LayerNorm needs the swap-AB (decode) path");
    TF_REQUIRE(d.ln_c && d.ln_d && d.ln_hidden > 0 && d.ln_hidden <= 16 * 128 && d.ln_hidden <= d.k &&
                   d.ln_stats_ld >= d.m_tok,
               TF_ERR_ARG, "gemm: bad fused LayerNorm arguments");
    a.ln_stats = reinterpret_cast<const float2*>(d.ln_stats);
    a.ln_H = d.ln_hidden;
    a.ln_tiles = (d.ln_hidden + 127) / 128;
    a.ln_stats_ld = d.ln_stats_ld;
    a.ln_c = d.ln_c;
    a.ln_d = d.ln_d;
  }
  if (d.stats_out) {
    TF_REQUIRE(d.epilogue == TF_EPI_BIAS_RESID && plan_emits_stats(p), TF_ERR_UNSUPPORTED,
               "gemm: row statistics need a swap-AB split-K residual GEMM");
    TF_REQUIRE(d.stats_ld >= d.m_tok, TF_ERR_ARG, "gemm: stats_ld < m_tok");
    a.stats_out = reinterpret_cast<float2*>(d.stats_out);
    a.stats_ld = d.stats_ld;
  }
  switch (d.epilogue) {
    case TF_EPI_BIAS:
    case TF_EPI_BIAS_GELU:
      TF_REQUIRE(d.bias && d.out, TF_ERR_ARG, "gemm: bias/out required");
      break;
    case TF_EPI_BIAS_RESID:
      TF_REQUIRE(d.bias && d.out && d.resid, TF_ERR_ARG, "gemm: bias/out/resid required");
      break;
    case TF_EPI_QKV:
      TF_REQUIRE(d.bias && d.q_out && d.k_cache && d.v_cache && d.qbase_dev, TF_ERR_ARG,
                 "gemm: qkv routing pointers required");
      TF_REQUIRE(d.n_feat == 3 * d.hidden && d.hidden == d.heads * d.head_dim && d.seq_len > 0,
                 TF_ERR_SHAPE, "gemm: qkv shape");
      break;
    case TF_EPI_F32:
      TF_REQUIRE(d.out, TF_ERR_ARG, "gemm: out required");
      break;
    case TF_EPI_LOGITS:
      TF_REQUIRE(d.out || d.argmax_keys, TF_ERR_ARG, "gemm: logits need out or keys");
      break;
    default:
      throw TfError{TF_ERR_ARG, "gemm: unknown epilogue"};
  }
  const void* P = p.swap ? d.wt : d.act;
  const void* Q = p.swap ? d.act : d.wt;
  const int ldp = p.swap ? d.ldw : d.lda, ldq = p.swap ? d.lda : d.ldw;
  const CUtensorMap ta = make_kmajor_map(P, a.rows_a, kext, ldp, kTileA);
  const CUtensorMap tb = make_kmajor_map(Q, a.rows_b, kext, ldq, p.bn);
  // prefill on 2-CTA pairs (256 tokens x 256 features per cluster, tcgen05 cta_group::2)
  static const bool pf2_on = [] {  // TF_PF2=0: single-CTA 128x128 prefill tiles (A/B)
    const char* e = getenv("TF_PF2");
    return !(e && e[0] == '0');
  }();
  // (only when the pair grid covers the SMs: N = 768 at 4096 tokens gives 96 CTAs,
  // fewer than the 192 single-CTA tiles, and measured slower)
  const int pf2_ctas = (p.tiles_a + 1) / 2 * 2 * ((d.n_feat + 255) / 256);
  const bool pf2 = pf2_on && !p.swap && d.n_feat >= 256 && d.m_tok > 128 && pf2_ctas >= num_sms() &&
                   (d.epilogue == TF_EPI_BIAS || d.epilogue == TF_EPI_BIAS_GELU || d.epilogue == TF_EPI_BIAS_RESID ||
                    d.epilogue == TF_EPI_QKV || (d.epilogue == TF_EPI_LOGITS && d.argmax_keys == nullptr));
  if (pf2) {
    GemmArgs a2 = a;
    a2.bn = kPf2BN;
    a2.stages = kPf2Stages;
    a2.splits = 1;
    a2.kb_per_split = p.k_blocks;
    const dim3 grid((p.tiles_a + 1) / 2 * 2, (d.n_feat + kPf2BN - 1) / kPf2BN, 1);
    auto go = [&](auto kern) {
      ensure_attr(kern, gemm_pf2_smem_bytes(), true);
      launch_cluster3(kern, grid, dim3(256), gemm_pf2_smem_bytes(), st, d.pdl != 0, dim3(2, 1, 1), ta, tb, a2);
    };
    switch (d.epilogue) {
      case TF_EPI_BIAS: go(gemm_pf2_kernel<EPI_BIAS>); break;
      case TF_EPI_BIAS_GELU: go(gemm_pf2_kernel<EPI_BIAS_GELU>); break;
      case TF_EPI_BIAS_RESID: go(gemm_pf2_kernel<EPI_BIAS_RESID>); break;
      case TF_EPI_QKV: go(gemm_pf2_kernel<EPI_QKV>); break;
      default: go(gemm_pf2_kernel<EPI_LOGITS>); break;
    }
    return;
  }
  switch (d.epilogue) {
    case TF_EPI_F32: launch_gemm_mode<EPI_F32>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS: launch_gemm_mode<EPI_BIAS>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS_GELU: launch_gemm_mode<EPI_BIAS_GELU>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS_RESID: launch_gemm_mode<EPI_BIAS_RESID>(d, p, ta, tb, a, st); break;
    case TF_EPI_QKV: launch_gemm_mode<EPI_QKV>(d, p, ta, tb, a, st); break;
    case TF_EPI_LOGITS: launch_gemm_mode<EPI_LOGITS>(d, p, ta, tb, a, st); break;
  }
}

// ------------------------------------------------------------------ LN / embed / attention
int vpl_for(int H) {
  const int v = (H + 31) / 32;
  if (v <= 4) return 4;
  if (v <= 8) return 8;
  if (v <= 16) return 16;
  if (v <= 24) return 24;
  if (v <= 32) return 32;
  if (v <= 48) return 48;
  if (v <= 64) return 64;
  return -1;
}

// 16-byte path needs H % 8 == 0 and 16-byte aligned row strides
bool vec_ok(int H, int ld1, int ld2) { return H % 8 == 0 && ld1 % 8 == 0 && ld2 % 8 == 0; }

void run_embed(const EmbedArgs& a, cudaStream_t st, bool pdl) {
  const dim3 grid((a.n_tok + 7) / 8);
  if (vec_ok(a.H, a.ldw, a.ldx) && a.H <= 2048) {
    const int nc = (a.H / 8 + 31) / 32;
    switch (nc) {
      case 1: launch_mc(embed_ln_vec_kernel<1>, grid, dim3(256), 0, st, pdl, a); return;
      case 2: launch_mc(embed_ln_vec_kernel<2>, grid, dim3(256), 0, st, pdl, a); return;
      case 3: launch_mc(embed_ln_vec_kernel<3>, grid, dim3(256), 0, st, pdl, a); return;
      case 4: launch_mc(embed_ln_vec_kernel<4>, grid, dim3(256), 0, st, pdl, a); return;
      case 6: launch_mc(embed_ln_vec_kernel<6>, grid, dim3(256), 0, st, pdl, a); return;
      case 8: launch_mc(embed_ln_vec_kernel<8>, grid, dim3(256), 0, st, pdl, a); return;
      default: break;
    }
  }
  switch (vpl_for(a.H)) {
    case 4: launch_mc(embed_ln_kernel<4>, grid, dim3(256), 0, st, pdl, a); break;
    case 8: launch_mc(embed_ln_kernel<8>, grid, dim3(256), 0, st, pdl, a); break;
    case 16: launch_mc(embed_ln_kernel<16>, grid, dim3(256), 0, st, pdl, a); break;
    case 24: launch_mc(embed_ln_kernel<24>, grid, dim3(256), 0, st, pdl, a); break;
    case 32: launch_mc(embed_ln_kernel<32>, grid, dim3(256), 0, st, pdl, a); break;
    case 48: launch_mc(embed_ln_kernel<48>, grid, dim3(256), 0, st, pdl, a); break;
    case 64: launch_mc(embed_ln_kernel<64>, grid, dim3(256), 0, st, pdl, a); break;
    default: throw TfError{TF_ERR_UNSUPPORTED, "hidden size > 2048 unsupported"};
  }
}

void run_ln(const LnArgs& a0, cudaStream_t st, bool pdl) {
  LnArgs a = a0;
  a.trace = trace_next("layernorm");
  const dim3 grid((a.n_rows + 7) / 8);
  // vector form: one warp per row, 8 rows per CTA
  if (vec_ok(a.H, a.ldx, a.ldh) && a.H <= 2048) {
    const int nc = (a.H / 8 + 31) / 32;
    switch (nc) {
      case 1: launch_mc(layernorm_vec_kernel<1>, grid, dim3(256), 0, st, pdl, a); return;
      case 2: launch_mc(layernorm_vec_kernel<2>, grid, dim3(256), 0, st, pdl, a); return;
      case 3: launch_mc(layernorm_vec_kernel<3>, grid, dim3(256), 0, st, pdl, a); return;
      case 4: launch_mc(layernorm_vec_kernel<4>, grid, dim3(256), 0, st, pdl, a); return;
      case 6: launch_mc(layernorm_vec_kernel<6>, grid, dim3(256), 0, st, pdl, a); return;
      case 8: launch_mc(layernorm_vec_kernel<8>, grid, dim3(256), 0, st, pdl, a); return;
      default: break;
    }
  }
  switch (vpl_for(a.H)) {
    case 4: launch_mc(layernorm_kernel<4>, grid, dim3(256), 0, st, pdl, a); break;
    case 8: launch_mc(layernorm_kernel<8>, grid, dim3(256), 0, st, pdl, a); break;
    case 16: launch_mc(layernorm_kernel<16>, grid, dim3(256), 0, st, pdl, a); break;
    case 24: launch_mc(layernorm_kernel<24>, grid, dim3(256), 0, st, pdl, a); break;
    case 32: launch_mc(layernorm_kernel<32>, grid, dim3(256), 0, st, pdl, a); break;
    case 48: launch_mc(layernorm_kernel<48>, grid, dim3(256), 0, st, pdl, a); break;
    case 64: launch_mc(layernorm_kernel<64>, grid, dim3(256), 0, st, pdl, a); break;
    default: throw TfError{TF_ERR_UNSUPPORTED, "hidden size > 2048 unsupported"};
  }
}

// beam attention: TF_ATTN_BEAM=0 runs the per-row kernel through the
// indirection table instead of the beam-grouped tensor-core one (A/B; both are
// checked against a torch reference in tests/test_gpu_beam_attention_op.py)
int beam_attn_mode() {
  static const int mode = [] {
    const char* e = getenv("TF_ATTN_BEAM");
    return e ? atoi(e) : 1;
  }();
  return mode;
}

// greedy decode attention kernel choice: -1 (default) the tensor-core unit
// kernel for capacities > 256 slots, the per-row kernel below; TF_GREEDY_MMA=0 /
// 1 forces the per-row / unit kernel (A/B)
int greedy_mma_mode() {
  static const int m = [] {
    const char* e = getenv("TF_GREEDY_MMA");
    return e ? atoi(e) : -1;
  }();
  return m;
}

void run_attention(const AttnArgs& a, cudaStream_t st, bool pdl) {
  TF_REQUIRE(a.D >= 1 && a.D <= 128, TF_ERR_UNSUPPORTED, "head_dim must be in [1, 128]");
  const bool ws_ok = a.ws && a.cnt && a.max_chunks >= (a.cap + kPfKeysPerChunk - 1) / kPfKeysPerChunk;
  if (a.T == 1 && a.D == 64 && a.indir && a.beam >= 2 && a.beam <= 8 && a.B % a.beam == 0 &&
      a.cap * a.beam <= 4096 && beam_attn_mode() != 0) {
    // tensor-core beam attention: one CTA per (head, request), shared chunks
    // once for all beams, mma.sync with the beams as M rows
    AttnArgs t = a;
    t.trace = trace_next("attn_decode_beam");
    ensure_attr(attn_decode_beam_mma_kernel, attn_beam_mma_smem(8, 2));
    launch(attn_decode_beam_mma_kernel, dim3(1, a.NH, a.B / a.beam), dim3(kBtThreads), attn_beam_mma_smem(a.beam, 2),
           st, pdl, t);
  } else if (a.T == 1 && a.D == 64 && !a.indir && a.cap <= 4096 &&
             (greedy_mma_mode() == 1 || (greedy_mma_mode() < 0 && a.cap > 256))) {
    // long windows: greedy decode on the unit-streaming tensor-core kernel (one
    // beam per request; each warp streams its next 32-slot unit while it computes
    // the current one). Short windows keep the per-row kernel, which stages the
    // whole window before the PDL wait (C5 buckets: faster from capacity ~320 on)
    AttnArgs t = a;
    t.beam = 1;
    t.trace = trace_next("attn_decode_mma");
    ensure_attr(attn_decode_beam_mma_kernel, attn_beam_mma_smem(8, 2));
    launch(attn_decode_beam_mma_kernel, dim3(1, a.NH, a.B), dim3(kBtThreads), attn_beam_mma_smem(1, 2), st, pdl, t);
  } else if (a.T == 1 && a.D == 64 && ws_ok) {
    // prefetching split-KV decode: chunks per CTA = the whole window when it is
    // <= 4 chunks (local merge), else groups of <= 4 (64 KB of K/V each)
    // merged through the workspace
    const int gmax = 4;
    const int nch = a.max_chunks;
    const int ngr = (nch + gmax - 1) / gmax;
    AttnArgs t = a;
    t.group = (nch + ngr - 1) / ngr;
    static const bool pfm = [] {  // TF_PF_MMA=0: CUDA-core per-chunk arithmetic everywhere (A/B)
      const char* e = getenv("TF_PF_MMA");
      return !(e && e[0] == '0');
    }();
    // the tensor-core form for every greedy batch: the choice must not depend on
    // the batch (rows x heads once picked it by wave count, so a row's tokens
    // changed between batches of 32 and 64 at 12 heads); C3 538 vs 560 us,
    // C2 ~1% slower than the CUDA-core form it kept for one-wave grids
    if (pfm && !a.indir) {
      t.trace = trace_next("attn_decode_pfm");
      const int grp = t.group;
      ensure_attr(attn_decode_pfm_kernel, attn_pfm_smem_bytes(4));
      launch(attn_decode_pfm_kernel, dim3(ngr, a.NH, a.B), dim3(128), attn_pfm_smem_bytes(grp), st, pdl, t);
      return;
    }
    t.trace = trace_next("attn_decode_pf");
    ensure_attr(attn_decode_pf_kernel<128>, attn_pf_smem_bytes(kPfMaxG));
    launch(attn_decode_pf_kernel<128>, dim3(ngr, a.NH, a.B), dim3(128), attn_pf_smem_bytes(t.group), st, pdl, t);
  } else if (a.T == 1) {
    const size_t smem = (size_t)(a.D + a.cap + std::max(2 * kDecThreads, kDecWarps * a.D)) * sizeof(float);
    TF_REQUIRE(smem <= kMaxSmem, TF_ERR_UNSUPPORTED, "cache capacity too large for decode kernel");
    ensure_attr(attn_decode_kernel, kMaxSmem);
    launch(attn_decode_kernel, dim3(a.NH, a.B), dim3(kDecThreads), smem, st, pdl, a);
  } else if (a.D == 64 && a.ldq % 8 == 0 && a.ldo % 8 == 0) {
    // tcgen05 prefill attention: S and O in TMEM, softmax in registers
    ensure_attr(attn_prefill_tc_kernel, kTcSmem);
    launch(attn_prefill_tc_kernel, dim3((a.T + kTcRows - 1) / kTcRows, a.NH, a.B), dim3(kTcThreads), kTcSmem, st, pdl,
           a);
  } else {
    const size_t smem = (size_t)kPfRows * a.D * sizeof(float) + (size_t)2 * kPfKeys * (a.D + 1) * 2;
    launch(attn_prefill_kernel, dim3((a.T + kPfRows - 1) / kPfRows, a.NH, a.B), dim3(128), smem, st,
           pdl, a);
  }
}

// ------------------------------------------------------------------ runtime objects
struct Model {
  tf_model_desc d;
  std::vector<tf_layer_weights> layers;
};

struct Session {
  Model* m;
  tf_session_desc d;
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t graph_multi = nullptr;  // TF_GRAPH_STEPS decode steps
  cudaGraphExec_t beam_graph = nullptr;
  tf_beam_desc beam_key{};  // descriptor the beam graph was captured with
  int graph_launches = 0;
  int launches_last = 0;
  // per-request beam attention plans written by the cluster select; valid for
  // the next T = 1 forward only (the select sets it, every forward clears it)
  uint8_t* beam_plan = nullptr;
  bool plan_valid = false;
};

int* qbase_zero_ptr() {
  // device scalar 0 for operator calls that start at slot 0 (one per device)
  static int* per_dev[64] = {nullptr};
  static std::mutex mu;
  const int dev = current_device();
  TF_REQUIRE(dev >= 0 && dev < 64, TF_ERR_UNSUPPORTED, "device ordinal >= 64");
  std::lock_guard<std::mutex> g(mu);
  if (!per_dev[dev]) {
    TF_CHECK_CUDA(cudaMalloc(&per_dev[dev], sizeof(int)));
    TF_CHECK_CUDA(cudaMemset(per_dev[dev], 0, sizeof(int)));
  }
  return per_dev[dev];
}

// LayerNorms fused into the consuming decode GEMMs (row statistics emitted by
// the residual GEMMs). TF_LN_FUSE=0 runs them as stand-alone kernels (A/B).
bool ln_fuse_on() {
  static const bool on = [] {
    const char* e = getenv("TF_LN_FUSE");
    return !(e && e[0] == '0');
  }();
  return on;
}

// One forward of T tokens per sequence through every layer
// (model._forward_tokens, model.py:440-504). Returns the number of kernels
// launched.
//
// Per layer: QKV GEMM (K/V appended to the cache) -> attention -> Wo GEMM +
// residual -> FFN1 GEMM + GELU -> FFN2 GEMM + residual. The LayerNorms before
// QKV and FFN1 (model.py:460-462, 484-486) run either as stand-alone kernels
// writing h, or -- decode-sized batches, when the session provides the
// statistics buffer -- inside the consuming GEMM: the residual GEMMs (Wo,
// FFN2) emit per-tile row statistics of the new residual stream and the
// consumer normalises its own K slice of x (gemm_tc.cuh ln_stats_*), so a
// decode layer is five launches. Layer 0's attn_norm is computed by the
// embedding kernel, the final norm by the LN kernel (its consumer, the lm_head,
// reads whole rows in every CTA).
//
// taps (diagnostics, may be null): f16 [2L+1][batch*T][hidden] copies of the
// residual stream at every LayerNorm input (the embedding
// sum, then after each Wo and each FFN2 residual add).
int forward(Session& s, const int* ids, const int* pos, int T, int mode, bool pdl,
            cudaStream_t st, bool remap_ids = true, __half* taps = nullptr) {
  const tf_model_desc& m = s.m->d;
  const tf_session_desc& sd = s.d;
  const int B = sd.batch, M = B * T;
  const int H = m.hidden, NH = m.heads, D = m.head_dim, F = m.ffn, L = m.layers;
  TF_REQUIRE(T >= 1 && T <= sd.max_tokens, TF_ERR_SHAPE, "forward: T out of range");
  TF_REQUIRE(ids != nullptr || T == 1, TF_ERR_ARG, "forward: ids required for T > 1");
  TF_REQUIRE(mode != TF_FWD_ARGMAX || sd.out_tokens, TF_ERR_ARG, "forward: out_tokens required");
  TF_REQUIRE(mode == TF_FWD_ARGMAX || sd.logits, TF_ERR_ARG, "forward: logits buffer required");
  int launches = 0;
  const size_t layer_cache = (size_t)B * NH * sd.capacity * D;
  __half* x = static_cast<__half*>(sd.x);
  __half* h = static_cast<__half*>(sd.h);

  EmbedArgs e{};
  e.n_tok = M;
  e.H = H;
  e.V = m.vocab;
  e.P = m.max_pos;
  e.ids = ids;
  e.keys = sd.keys;
  e.remap = (ids && remap_ids) ? sd.remap : nullptr;
  e.remap_n = sd.remap_n;
  e.unk_id = sd.unk_id;
  e.pos = pos;
  e.len_dev = sd.len_dev;
  e.pads = sd.pads;
  e.tok_emb = static_cast<const __half*>(m.tok_emb);
  e.pos_emb = static_cast<const __half*>(m.pos_emb);
  e.type_emb = static_cast<const __half*>(m.type_emb);
  e.type_ids = ids ? sd.type_ids : nullptr;
  e.type_const = sd.gen_type;
  e.ldw = m.ldw;
  e.ln_g = s.m->layers[0].ln1_gamma;
  e.ln_b = s.m->layers[0].ln1_beta;
  e.x = x;
  e.h = h;
  e.ldx = m.ldk_h;
  run_embed(e, st, pdl);
  ++launches;
  int n_taps = 0;
  auto tap = [&]() {
    if (!taps) return;
    TF_CHECK_CUDA(cudaMemcpy2DAsync(taps + (size_t)n_taps * M * H, (size_t)H * 2, x, (size_t)m.ldk_h * 2,
                                    (size_t)H * 2, M, cudaMemcpyDeviceToDevice, st));
    ++n_taps;
  };
  tap();

  tf_gemm_desc g{};
  g.m_tok = M;
  // prefill (T > 1): the layer GEMMs always take the full-K token-tile form, so a
  // prompt's hidden states do not depend on how many tokens its batch has (the
  // swap-AB split-K form, whose split count follows the token count, is for
  // decode steps, where it is fixed for every batch of <= 128 rows)
  g.force_swap = T > 1 ? 0 : -1;
  g.pdl = pdl ? 1 : 0;

  // decode: every kernel of layer l streams the next layer's copy of its own
  // operand (weights; the attention its KV window) HBM -> L2, so the chain of
  // latency-bound kernels reads L2 while HBM runs a layer ahead. The last
  // layer's GEMMs stream a quarter of the lm_head each instead.
  static const bool l2pf_on = [] {  // TF_L2PF=0 disables (A/B diagnostics)
    const char* e = getenv("TF_L2PF");
    return !(e && e[0] == '0');
  }();
  const bool l2pf = l2pf_on && T == 1;
  const unsigned long long lm_bytes = (unsigned long long)m.vocab * m.ldk_h * 2;
  const unsigned long long lm_q = ((lm_bytes / 4) + 255) & ~255ull;
  // diagnostics: TF_SPLITS="q,o,f1,f2" forces the decode split counts (0 = auto)
  static const std::vector<int> force_splits = [] {
    std::vector<int> v(4, 0);
    if (const char* e = getenv("TF_SPLITS")) sscanf(e, "%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3]);
    return v;
  }();
  const bool fs = T == 1;

  // the layer's GEMM descriptors (pointers filled per layer below)
  tf_gemm_desc q = g;  // fused QKV projection, K/V straight into the cache (model.py:464-474)
  q.n_feat = 3 * H;
  q.k = H;
  q.lda = m.ldk_h;
  q.ldw = m.ldk_h;
  q.epilogue = TF_EPI_QKV;
  q.q_out = sd.q;
  q.ldq = m.ldk_h;
  q.hidden = H;
  q.heads = NH;
  q.head_dim = D;
  q.cap = sd.capacity;
  q.seq_len = T;
  q.qbase_dev = sd.len_dev;
  if (fs && force_splits[0]) q.splits = force_splits[0];
  // decode: attention (next) prefetches the whole KV window; release it only
  // once the QKV weights are in (after this GEMM's own dependency wait)
  if (pdl && T == 1) q.pdl = 2;
  tf_gemm_desc o = g;  // output projection + residual (model.py:478-482)
  o.n_feat = H;
  o.k = H;
  o.act = sd.attn;
  o.lda = m.ldk_h;
  o.ldw = m.ldk_h;
  o.epilogue = TF_EPI_BIAS_RESID;
  o.out = x;
  o.ldo = m.ldk_h;
  o.resid = x;
  o.ldr = m.ldk_h;
  if (fs && force_splits[1]) o.splits = force_splits[1];
  tf_gemm_desc f1 = g;  // FFN1 + GELU (model.py:488-490)
  f1.n_feat = F;
  f1.k = H;
  f1.lda = m.ldk_h;
  f1.ldw = m.ldk_h;
  f1.epilogue = TF_EPI_BIAS_GELU;
  f1.out = sd.ffn;
  f1.ldo = m.ldk_f;
  if (fs && force_splits[2]) f1.splits = force_splits[2];
  tf_gemm_desc f2 = g;  // FFN2 + residual (model.py:491-494)
  f2.n_feat = H;
  f2.k = F;
  f2.act = sd.ffn;
  f2.lda = m.ldk_f;
  f2.ldw = m.ldk_f;
  f2.epilogue = TF_EPI_BIAS_RESID;
  f2.out = x;
  f2.ldo = m.ldk_h;
  f2.resid = x;
  f2.ldr = m.ldk_h;
  if (fs && force_splits[3]) f2.splits = force_splits[3];

  // fused LayerNorms: both residual GEMMs must be able to emit statistics and
  // both consumers must take the swap-AB path
  const int ln_tiles = (H + 127) / 128;
  float* stats_a = sd.ln_stats;  // written by Wo, read by FFN1
  float* stats_b = sd.ln_stats ? sd.ln_stats + (size_t)2 * ln_tiles * M : nullptr;  // FFN2 -> next QKV
  bool lnf = ln_fuse_on() && sd.ln_stats && sd.ln_stats_bytes >= (size_t)4 * ln_tiles * M * sizeof(float) &&
             ln_tiles <= 16 && s.m->layers[0].wqkv_ln_t != nullptr;
  if (lnf)
    lnf = plan_gemm(q).swap && plan_gemm(f1).swap && plan_emits_stats(plan_gemm(o)) &&
          plan_emits_stats(plan_gemm(f2));
  // the lm_head reads the last position's rows: folded only when those are all rows
  const bool lm_fold = lnf && m.lm_head_ln_t && (T == 1 || mode == TF_FWD_LOGITS_ALL);
  auto pf_next = [&](int l, int which) {
    GemmExtra ex;
    if (!l2pf) return ex;
    if (l + 1 < L) {
      const tf_layer_weights& n = s.m->layers[l + 1];
      switch (which) {
        // the copy the consumer will read: the LayerNorm-folded weights when folded
        case 0: ex.l2pf = lnf ? n.wqkv_ln_t : n.wqkv_t; ex.l2pf_bytes = 3ull * H * m.ldk_h * 2; break;
        case 1: ex.l2pf = n.wo_t; ex.l2pf_bytes = (unsigned long long)H * m.ldk_h * 2; break;
        case 2: ex.l2pf = lnf ? n.w1_ln_t : n.w1_t; ex.l2pf_bytes = (unsigned long long)F * m.ldk_h * 2; break;
        default: ex.l2pf = n.w2_t; ex.l2pf_bytes = (unsigned long long)H * m.ldk_f * 2; break;
      }
    } else {
      const unsigned long long lo = which * lm_q;
      if (lo >= lm_bytes) return ex;
      ex.l2pf = static_cast<const uint8_t*>(lm_fold ? m.lm_head_ln_t : m.lm_head_t) + lo;
      ex.l2pf_bytes = std::min(lm_q, lm_bytes - lo);
    }
    return ex;
  };

  auto set_ln = [&](tf_gemm_desc& d, const float* stats, const void* wt_ln, const float* c, const float* dd) {
    d.act = x;
    d.wt = wt_ln;
    d.ln_stats = stats;
    d.ln_stats_ld = M;
    d.ln_hidden = H;
    d.ln_c = c;
    d.ln_d = dd;
  };
  LnArgs ln{};
  ln.n_rows = M;
  ln.H = H;
  ln.x = x;
  ln.ldx = m.ldk_h;
  ln.src_stride = 1;
  ln.src_off = 0;
  ln.h = h;
  ln.ldh = m.ldk_h;

  for (int l = 0; l < L; ++l) {
    const tf_layer_weights& w = s.m->layers[l];
    q.wt = w.wqkv_t;
    q.bias = w.bqkv;
    q.k_cache = static_cast<__half*>(sd.k_cache) + l * layer_cache;
    q.v_cache = static_cast<__half*>(sd.v_cache) + l * layer_cache;
    q.act = h;
    q.ln_stats = nullptr;
    if (lnf && l > 0) set_ln(q, stats_b, w.wqkv_ln_t, w.cqkv, w.dqkv);
    run_gemm(q, st, pf_next(l, 0));
    ++launches;
    // attention over slots [pad_b, len + t] (model.py:475-478)
    AttnArgs at{};
    at.B = B;
    at.NH = NH;
    at.D = D;
    at.cap = sd.capacity;
    at.T = T;
    at.q = static_cast<const __half*>(sd.q);
    at.ldq = m.ldk_h;
    at.kc = static_cast<const __half*>(q.k_cache);
    at.vc = static_cast<const __half*>(q.v_cache);
    at.start = sd.pads;
    at.qbase_dev = sd.len_dev;
    at.scale = (float)(1.0 / std::sqrt((double)D));
    at.out = static_cast<__half*>(sd.attn);
    at.ldo = m.ldk_h;
    if (T == 1 && sd.beam_indir) {
      at.indir = sd.beam_indir;
      at.beam = sd.beam;
      if (s.plan_valid) at.plan = s.beam_plan;
    }
    if (T == 1 && D == 64) {  // split-KV decode attention when the session provides scratch
      const int chunks = (sd.capacity + kPfKeysPerChunk - 1) / kPfKeysPerChunk;
      const size_t need = (size_t)B * NH * chunks * 66 * sizeof(float);
      if (sd.workspace && sd.workspace_bytes >= need && sd.counters && sd.n_counters >= B * NH) {
        at.ws = sd.workspace;
        at.cnt = sd.counters;
        at.max_chunks = chunks;
      }
      // the next layer's KV window is streamed into L2 only while it is small
      // next to the 126 MB L2 (measured at batch 128: 52 MB per layer is evicted
      // before use and doubles the attention's DRAM reads)
      const size_t kv_layer_bytes = 2 * layer_cache * sizeof(__half);
      if (l2pf && l + 1 < L && kv_layer_bytes <= (32u << 20)) {
        at.pf_kc = static_cast<const __half*>(sd.k_cache) + (l + 1) * layer_cache;
        at.pf_vc = static_cast<const __half*>(sd.v_cache) + (l + 1) * layer_cache;
      }
    }
    run_attention(at, st, pdl);
    ++launches;
    o.wt = w.wo_t;
    o.bias = w.bo;
    o.stats_out = lnf ? stats_a : nullptr;
    o.stats_ld = M;
    run_gemm(o, st, pf_next(l, 1));
    ++launches;
    tap();
    // ffn_norm (model.py:484-486)
    f1.wt = w.w1_t;
    f1.bias = w.b1;
    f1.act = h;
    f1.ln_stats = nullptr;
    if (lnf) {
      set_ln(f1, stats_a, w.w1_ln_t, w.c1, w.d1);
    } else {
      ln.g = w.ln2_gamma;
      ln.b = w.ln2_beta;
      run_ln(ln, st, pdl);
      ++launches;
    }
    run_gemm(f1, st, pf_next(l, 2));
    ++launches;
    f2.wt = w.w2_t;
    f2.bias = w.b2;
    f2.stats_out = (lnf && (l + 1 < L || lm_fold)) ? stats_b : nullptr;
    f2.stats_ld = M;
    run_gemm(f2, st, pf_next(l, 3));
    ++launches;
    tap();
    // next layer's attn_norm (fused into its QKV, or stand-alone)
    if (l + 1 < L && !lnf) {
      ln.g = s.m->layers[l + 1].ln1_gamma;
      ln.b = s.m->layers[l + 1].ln1_beta;
      run_ln(ln, st, pdl);
      ++launches;
    }
  }
  // final_norm (model.py:497-498): only the last position feeds the lm_head
  tf_gemm_desc lg = g;
  lg.force_swap = -1;  // full-K either way (no split-K for logits); swap-AB for <= 256 rows
  lg.m_tok = (mode == TF_FWD_LOGITS_ALL) ? M : B;
  lg.n_feat = m.vocab;
  lg.k = H;
  lg.act = h;
  lg.lda = m.ldk_h;
  lg.wt = m.lm_head_t;
  lg.ldw = m.ldk_h;
  lg.epilogue = TF_EPI_LOGITS;
  if (lm_fold) {
    set_ln(lg, stats_b, m.lm_head_ln_t, m.c_lm, m.d_lm);
  } else {
    LnArgs nl = ln;
    nl.g = m.final_gamma;
    nl.b = m.final_beta;
    if (mode != TF_FWD_LOGITS_ALL) {
      nl.n_rows = B;
      nl.src_stride = T;
      nl.src_off = T - 1;
    }
    run_ln(nl, st, pdl);
    ++launches;
  }
  // lm_head (+ argmax) (model.py:500-504, 594, 652)
  if (mode == TF_FWD_ARGMAX) {
    lg.argmax_keys = sd.keys;
  } else {
    lg.out = sd.logits;
    lg.ldo = m.vocab;
  }
  run_gemm(lg, st);
  ++launches;
  CollectArgs c{};
  c.B = B;
  c.keys = sd.keys;
  c.out_tokens = mode == TF_FWD_ARGMAX ? sd.out_tokens : nullptr;
  c.max_new = sd.max_new;
  c.step_dev = sd.step_dev;
  c.len_dev = sd.len_dev;
  c.advance = T;
  if (mode != TF_FWD_ARGMAX) {
    // only advance the cache length: reuse collect with no token output
    CollectArgs c2 = c;
    c2.B = 0;
    launch_mc(collect_kernel, dim3(1), dim3(32), 0, st, pdl, c2);
  } else {
    launch_mc(collect_kernel, dim3(1), dim3(256), 0, st, pdl, c);
  }
  ++launches;
  s.plan_valid = false;  // the cache length moved on: a plan is for one step
  return launches;
}

BeamArgs beam_args(const Session& s, const tf_beam_desc& d) {
  TF_REQUIRE(d.beam >= 1 && d.beam <= kMaxBeam, TF_ERR_UNSUPPORTED, "beam width must be in [1, 8]");
  TF_REQUIRE(d.requests * d.beam == s.d.batch, TF_ERR_SHAPE, "beam: requests*beam != session batch");
  TF_REQUIRE(s.d.beam_indir && s.d.beam == d.beam, TF_ERR_ARG, "beam: session lacks the indirection table");
  TF_REQUIRE(s.d.logits && d.scores && d.finished && d.tokens && d.tok_hist && d.par_hist, TF_ERR_ARG,
             "beam: missing buffer");
  BeamArgs a{};
  a.R = d.requests;
  a.K = d.beam;
  a.V = s.m->d.vocab;
  a.cap = s.d.capacity;
  a.max_new = d.max_new;
  a.eos = d.eos;
  a.logits = static_cast<const __half*>(s.d.logits);
  a.ldl = s.m->d.vocab;
  a.scores = d.scores;
  a.finished = d.finished;
  a.tokens = d.tokens;
  a.tok_hist = d.tok_hist;
  a.par_hist = d.par_hist;
  a.indir = s.d.beam_indir;
  a.len_dev = s.d.len_dev;
  a.prompt_len = d.prompt_len;
  a.pads = s.d.pads;
  return a;
}

bool select_cluster_on() {
  static const bool cl = [] {  // TF_SELECT_CLUSTER=0: one CTA per request (A/B)
    const char* e = getenv("TF_SELECT_CLUSTER");
    return !(e && e[0] == '0');
  }();
  return cl;
}

bool beam_plan_on() {
  static const bool on = [] {  // TF_BEAM_PLAN=0: every attention CTA derives its unit list (A/B)
    const char* e = getenv("TF_BEAM_PLAN");
    return !(e && e[0] == '0');
  }();
  return on;
}

template <int KB>
void launch_select(const BeamArgs& a, size_t smem, cudaStream_t st, bool pdl) {
  if constexpr (KB >= 2) {
    if (select_cluster_on()) {
      ensure_attr(beam_select_cluster_kernel<KB>, kMaxSmem - 8192);
      launch_cluster3(beam_select_cluster_kernel<KB>, dim3(KB, a.R), dim3(kSelCThreads), smem, st, pdl,
                      dim3(KB, 1, 1), a);
      return;
    }
  }
  ensure_attr(beam_select_kernel<KB>, kMaxSmem - 8192);
  launch(beam_select_kernel<KB>, dim3(a.R), dim3(kSelThreads), smem, st, pdl, a);
}

void run_beam_select(Session& s, const tf_beam_desc& d, cudaStream_t st, bool pdl) {
  BeamArgs a = beam_args(s, d);
  // the cluster select also writes the next step's attention plans
  const bool plan = s.beam_plan && a.K >= 2 && select_cluster_on() && beam_plan_on();
  if (plan) a.plan = s.beam_plan;
  const size_t smem = (size_t)a.K * a.cap * sizeof(int);
  TF_REQUIRE(smem <= kMaxSmem - 8192, TF_ERR_UNSUPPORTED, "beam: capacity too large");
  switch (a.K) {
    case 1: launch_select<1>(a, smem, st, pdl); break;
    case 2: launch_select<2>(a, smem, st, pdl); break;
    case 3: launch_select<3>(a, smem, st, pdl); break;
    case 4: launch_select<4>(a, smem, st, pdl); break;
    case 5: launch_select<5>(a, smem, st, pdl); break;
    case 6: launch_select<6>(a, smem, st, pdl); break;
    case 7: launch_select<7>(a, smem, st, pdl); break;
    case 8: launch_select<8>(a, smem, st, pdl); break;
    default: throw TfError{TF_ERR_UNSUPPORTED, "beam width must be in [1, 8]"};
  }
  s.plan_valid = plan;
}

// one beam step: feed `tokens` (generated ids, no remap), last-row logits, select
int beam_step(Session& s, const tf_beam_desc& d, cudaStream_t st) {
  int n = forward(s, d.tokens, nullptr, 1, TF_FWD_LOGITS_LAST, true, st, false);
  run_beam_select(s, d, st, true);
  return n + 1;
}

}  // namespace

// ====================================================================== C ABI
extern "C" {

int tf_abi_version(void) { return TF_ABI_VERSION; }

const char* tf_last_error(void) { return g_last_error.c_str(); }

int tf_device_info(int* sm_count, int* cc_major, int* cc_minor) {
  return guarded([&] {
    int dev = 0;
    TF_CHECK_CUDA(cudaGetDevice(&dev));
    if (sm_count) TF_CHECK_CUDA(cudaDeviceGetAttribute(sm_count, cudaDevAttrMultiProcessorCount, dev));
    if (cc_major) TF_CHECK_CUDA(cudaDeviceGetAttribute(cc_major, cudaDevAttrComputeCapabilityMajor, dev));
    if (cc_minor) TF_CHECK_CUDA(cudaDeviceGetAttribute(cc_minor, cudaDevAttrComputeCapabilityMinor, dev));
  });
}

int tf_gemm(const tf_gemm_desc* d, void* stream) {
  return guarded([&] {
    TF_REQUIRE(d != nullptr, TF_ERR_ARG, "null desc");
    run_gemm(*d, static_cast<cudaStream_t>(stream));
  });
}

int tf_embed_ln(const tf_embed_desc* d, void* stream) {
  return guarded([&] {
    TF_REQUIRE(d && d->ids && d->tok_emb && d->pos_emb && d->x, TF_ERR_ARG, "embed: null pointer");
    TF_REQUIRE(d->pos != nullptr, TF_ERR_ARG, "embed: positions required");
    TF_REQUIRE(!d->h || (d->ln_gamma && d->ln_beta), TF_ERR_ARG, "embed: LN params required");
    EmbedArgs e{};
    e.n_tok = d->n_tok;
    e.H = d->hidden;
    e.V = d->vocab;
    e.P = d->max_pos;
    e.ids = d->ids;
    e.pos = d->pos;
    e.type_ids = d->type_ids;
    e.type_const = d->type_const;
    e.remap = d->remap;
    e.remap_n = d->remap_n;
    e.unk_id = d->unk_id;
    e.tok_emb = static_cast<const __half*>(d->tok_emb);
    e.pos_emb = static_cast<const __half*>(d->pos_emb);
    e.type_emb = static_cast<const __half*>(d->type_emb);
    e.ldw = d->ldw;
    e.ln_g = d->ln_gamma;
    e.ln_b = d->ln_beta;
    e.x = static_cast<__half*>(d->x);
    e.h = static_cast<__half*>(d->h);
    e.ldx = d->ldx;
    e.tok_out = d->ids_out;
    if (d->n_tok > 0) run_embed(e, static_cast<cudaStream_t>(stream), false);
  });
}

int tf_layernorm(int n_rows, int hidden, const void* x, int ldx, int src_stride, int src_off,
                 const float* gamma, const float* beta, void* h, int ldh, void* stream) {
  return guarded([&] {
    TF_REQUIRE(x && h && gamma && beta, TF_ERR_ARG, "layernorm: null pointer");
    LnArgs a{n_rows, hidden, static_cast<const __half*>(x), ldx, src_stride, src_off,
             gamma,  beta,   static_cast<__half*>(h),       ldh};
    if (n_rows > 0) run_ln(a, static_cast<cudaStream_t>(stream), false);
  });
}

int tf_attention(int batch, int heads, int head_dim, int cap, int seq_len, const void* q, int ldq,
                 const void* k_cache, const void* v_cache, const int* start, const int* qbase_dev,
                 float scale, void* out, int ldo, void* stream) {
  return guarded([&] {
    TF_REQUIRE(q && k_cache && v_cache && start && out, TF_ERR_ARG, "attention: null pointer");
    AttnArgs a{};
    a.B = batch;
    a.NH = heads;
    a.D = head_dim;
    a.cap = cap;
    a.T = seq_len;
    a.q = static_cast<const __half*>(q);
    a.ldq = ldq;
    a.kc = static_cast<const __half*>(k_cache);
    a.vc = static_cast<const __half*>(v_cache);
    a.start = start;
    a.qbase_dev = qbase_dev ? qbase_dev : qbase_zero_ptr();
    a.scale = scale;
    a.out = static_cast<__half*>(out);
    a.ldo = ldo;
    if (batch <= 0 || seq_len <= 0) return;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    void* scratch = nullptr;
    if (seq_len == 1 && head_dim == 64) {
      // the split-KV decode kernels' partials + zeroed arrival counters, stream-
      // ordered for this call (sessions own theirs), so the operator runs the
      // same decode kernel as the generation path
      const int chunks = (cap + kPfKeysPerChunk - 1) / kPfKeysPerChunk;
      const size_t ws = (size_t)batch * heads * chunks * 66 * sizeof(float);
      const size_t cnt = (size_t)batch * heads * sizeof(int);
      TF_CHECK_CUDA(cudaMallocAsync(&scratch, ws + cnt, st));
      TF_CHECK_CUDA(cudaMemsetAsync(static_cast<uint8_t*>(scratch) + ws, 0, cnt, st));
      a.ws = static_cast<float*>(scratch);
      a.cnt = reinterpret_cast<int*>(static_cast<uint8_t*>(scratch) + ws);
      a.max_chunks = chunks;
    }
    run_attention(a, st, false);
    if (scratch) TF_CHECK_CUDA(cudaFreeAsync(scratch, st));
  });
}

int tf_attention_beam(int requests, int beam, int heads, int head_dim, int cap, const void* q, int ldq,
                      const void* k_cache, const void* v_cache, const int* start, const int* qbase_dev,
                      const int* indir, float scale, void* out, int ldo, void* stream) {
  return guarded([&] {
    TF_REQUIRE(q && k_cache && v_cache && start && indir && out && qbase_dev, TF_ERR_ARG,
               "attention_beam: null pointer");
    TF_REQUIRE(beam >= 1 && beam <= 8 && requests >= 0, TF_ERR_ARG, "attention_beam: beam must be in [1, 8]");
    AttnArgs a{};
    a.B = requests * beam;
    a.NH = heads;
    a.D = head_dim;
    a.cap = cap;
    a.T = 1;
    a.q = static_cast<const __half*>(q);
    a.ldq = ldq;
    a.kc = static_cast<const __half*>(k_cache);
    a.vc = static_cast<const __half*>(v_cache);
    a.start = start;
    a.qbase_dev = qbase_dev;
    a.indir = indir;
    a.beam = beam;
    a.scale = scale;
    a.out = static_cast<__half*>(out);
    a.ldo = ldo;
    if (requests > 0) run_attention(a, static_cast<cudaStream_t>(stream), false);
  });
}

int tf_pack_kmajor(const void* src, int src_f32, int K, int N, const float* gamma, void* dst, int ldk,
                   void* stream) {
  return guarded([&] {
    TF_REQUIRE(src && dst, TF_ERR_ARG, "pack: null pointer");
    TF_REQUIRE(K >= 1 && N >= 1 && ldk >= K, TF_ERR_SHAPE, "pack: bad shape");
    dim3 grid((N + 31) / 32, (ldk + 31) / 32);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (src_f32)
      pack_kmajor_kernel<true><<<grid, 256, 0, st>>>(src, K, N, gamma, static_cast<__half*>(dst), ldk);
    else
      pack_kmajor_kernel<false><<<grid, 256, 0, st>>>(src, K, N, gamma, static_cast<__half*>(dst), ldk);
    TF_CHECK_CUDA(cudaGetLastError());
  });
}

int tf_fold_terms(const void* w_t, const void* w_ln_t, const float* beta, int K, int N, int ldk, float* c,
                  float* d, void* stream) {
  return guarded([&] {
    TF_REQUIRE(w_t && w_ln_t && beta && c && d, TF_ERR_ARG, "fold_terms: null pointer");
    TF_REQUIRE(K >= 1 && N >= 1 && ldk >= K, TF_ERR_SHAPE, "fold_terms: bad shape");
    fold_terms_kernel<<<(N + 7) / 8, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const __half*>(w_t), static_cast<const __half*>(w_ln_t), beta, K, N, ldk, c, d);
    TF_CHECK_CUDA(cudaGetLastError());
  });
}

int tf_convert(const void* src, int src_f32, long long n, void* dst, int dst_f32, void* stream) {
  return guarded([&] {
    TF_REQUIRE(src && dst && n >= 1, TF_ERR_ARG, "convert: bad arguments");
    const long long blocks = std::min<long long>((n + 255) / 256, 148ll * 16);
    convert_kernel<<<(unsigned)blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(src, src_f32, n, dst, dst_f32);
    TF_CHECK_CUDA(cudaGetLastError());
  });
}

int tf_model_create(const tf_model_desc* d, void** model) {
  return guarded([&] {
    TF_REQUIRE(d && model && d->layer, TF_ERR_ARG, "model: null desc");
    TF_REQUIRE(d->hidden == d->heads * d->head_dim, TF_ERR_SHAPE, "model: hidden != heads*head_dim");
    TF_REQUIRE(d->ldk_h >= pad64(d->hidden) && d->ldk_f >= pad64(d->ffn), TF_ERR_SHAPE,
               "model: padded strides too small");
    TF_REQUIRE(vpl_for(d->hidden) > 0, TF_ERR_UNSUPPORTED, "model: hidden > 2048");
    TF_REQUIRE(d->head_dim <= 128, TF_ERR_UNSUPPORTED, "model: head_dim > 128");
    Model* m = new Model();
    m->d = *d;
    m->layers.assign(d->layer, d->layer + d->layers);
    m->d.layer = m->layers.data();
    *model = m;
  });
}

int tf_model_destroy(void* model) {
  return guarded([&] { delete static_cast<Model*>(model); });
}

int tf_session_create(void* model, const tf_session_desc* d, void** session) {
  return guarded([&] {
    TF_REQUIRE(model && d && session, TF_ERR_ARG, "session: null argument");
    TF_REQUIRE(d->batch >= 1 && d->capacity >= 1 && d->max_tokens >= 1, TF_ERR_SHAPE,
               "session: bad sizes");
    TF_REQUIRE(d->k_cache && d->v_cache && d->x && d->h && d->q && d->attn && d->ffn && d->keys &&
                   d->len_dev && d->step_dev && d->pads,
               TF_ERR_ARG, "session: missing buffer");
    Session* s = new Session();
    s->m = static_cast<Model*>(model);
    s->d = *d;
    if (d->beam_indir && d->beam >= 2 && d->batch % d->beam == 0)
      TF_CHECK_CUDA(cudaMalloc(&s->beam_plan, (size_t)(d->batch / d->beam) * kBeamPlanBytes));
    *session = s;
  });
}

int tf_session_destroy(void* session) {
  return guarded([&] {
    Session* s = static_cast<Session*>(session);
    if (s && s->graph) cudaGraphExecDestroy(s->graph);
    if (s && s->graph_multi) cudaGraphExecDestroy(s->graph_multi);
    if (s && s->beam_graph) cudaGraphExecDestroy(s->beam_graph);
    if (s && s->beam_plan) cudaFree(s->beam_plan);
    delete s;
  });
}

int tf_forward(void* session, const int* ids, const int* pos, int T, int mode, int pdl,
               void* stream) {
  return guarded([&] {
    TF_REQUIRE(session, TF_ERR_ARG, "forward: null session");
    Session& s = *static_cast<Session*>(session);
    s.launches_last = forward(s, ids, pos, T, mode, pdl != 0, static_cast<cudaStream_t>(stream));
  });
}

int tf_forward_taps(void* session, const int* ids, const int* pos, int T, int mode, void* taps, void* stream) {
  return guarded([&] {
    TF_REQUIRE(session && taps, TF_ERR_ARG, "forward_taps: null argument");
    Session& s = *static_cast<Session*>(session);
    s.launches_last = forward(s, ids, pos, T, mode, true, static_cast<cudaStream_t>(stream), true,
                              static_cast<__half*>(taps));
  });
}

int tf_decode(void* session, int n_steps, int use_graph, void* stream) {
  return guarded([&] {
    TF_REQUIRE(session, TF_ERR_ARG, "decode: null session");
    Session& s = *static_cast<Session*>(session);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_steps <= 0) return;
    if (!use_graph) {
      for (int i = 0; i < n_steps; ++i)
        s.launches_last = forward(s, nullptr, nullptr, 1, TF_FWD_ARGMAX, true, st);
      return;
    }
    // capture k decode steps on a private stream; every per-step quantity
    // (cache length, fed ids, output column) lives in device memory, so one
    // graph replays any step. Steps inside a graph are chained with PDL like
    // the kernels of a step (each step's embed kernel waits before releasing
    // its successor, which keeps whole steps ordered).
    auto capture = [&](int k, cudaGraphExec_t* out) {
      cudaStream_t cs;
      TF_CHECK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      cudaGraph_t g;
      TF_CHECK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int launches = 0;
      try {
        for (int i = 0; i < k; ++i) launches = forward(s, nullptr, nullptr, 1, TF_FWD_ARGMAX, true, cs);
      } catch (...) {
        cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        throw;
      }
      TF_CHECK_CUDA(cudaStreamEndCapture(cs, &g));
      TF_CHECK_CUDA(cudaGraphInstantiate(out, g, 0));
      TF_CHECK_CUDA(cudaGraphDestroy(g));
      TF_CHECK_CUDA(cudaStreamDestroy(cs));
      return launches;
    };
    static const int multi = [] {  // steps per multi-step graph (TF_GRAPH_STEPS, 1 disables)
      const char* e = getenv("TF_GRAPH_STEPS");
      const int v = e ? atoi(e) : 8;
      return v < 1 ? 1 : v;
    }();
    if (!s.graph) s.graph_launches = capture(1, &s.graph);
    int left = n_steps;
    if (multi > 1 && left >= multi) {
      if (!s.graph_multi) capture(multi, &s.graph_multi);
      for (; left >= multi; left -= multi) TF_CHECK_CUDA(cudaGraphLaunch(s.graph_multi, st));
    }
    for (; left > 0; --left) TF_CHECK_CUDA(cudaGraphLaunch(s.graph, st));
    s.launches_last = s.graph_launches;
  });
}

int tf_beam_select(void* session, const tf_beam_desc* d, void* stream) {
  return guarded([&] {
    TF_REQUIRE(session && d, TF_ERR_ARG, "beam_select: null argument");
    run_beam_select(*static_cast<Session*>(session), *d, static_cast<cudaStream_t>(stream), false);
  });
}

int tf_beam_decode(void* session, const tf_beam_desc* d, int n_steps, int use_graph, void* stream) {
  return guarded([&] {
    TF_REQUIRE(session && d, TF_ERR_ARG, "beam_decode: null argument");
    Session& s = *static_cast<Session*>(session);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_steps <= 0) return;
    if (!use_graph) {
      for (int i = 0; i < n_steps; ++i) s.launches_last = beam_step(s, *d, st);
      return;
    }
    if (s.beam_graph && std::memcmp(&s.beam_key, d, sizeof(*d)) != 0) {
      cudaGraphExecDestroy(s.beam_graph);
      s.beam_graph = nullptr;
    }
    if (!s.beam_graph) {
      cudaStream_t cs;
      TF_CHECK_CUDA(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
      cudaGraph_t g;
      TF_CHECK_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      int launches = 0;
      try {
        launches = beam_step(s, *d, cs);
      } catch (...) {
        cudaStreamEndCapture(cs, &g);
        cudaStreamDestroy(cs);
        throw;
      }
      TF_CHECK_CUDA(cudaStreamEndCapture(cs, &g));
      TF_CHECK_CUDA(cudaGraphInstantiate(&s.beam_graph, g, 0));
      TF_CHECK_CUDA(cudaGraphDestroy(g));
      TF_CHECK_CUDA(cudaStreamDestroy(cs));
      s.beam_key = *d;
      s.graph_launches = launches;
    }
    for (int i = 0; i < n_steps; ++i) TF_CHECK_CUDA(cudaGraphLaunch(s.beam_graph, st));
    s.launches_last = s.graph_launches;
  });
}

int tf_debug_trace(int reset, unsigned long long* dst, int max_slots, const char** names) {
  // dst: [slot][kTraceCtas][8] raw per-CTA stamps (0 = CTA absent)
  int n = 0;
  static unsigned long long* buf = nullptr;
  const size_t bytes = sizeof(unsigned long long) * (size_t)kTraceSlots * kTraceCtas * 8;
  const int rc = guarded([&] {
    if (reset) {
      if (!buf) {
        TF_CHECK_CUDA(cudaMalloc(&buf, bytes));
        TF_CHECK_CUDA(cudaMemcpyToSymbol(g_trace_buf, &buf, sizeof(buf)));
      }
      TF_CHECK_CUDA(cudaMemset(buf, 0, bytes));
      g_trace_n = 0;
      return;
    }
    n = std::min(g_trace_n, max_slots);
    if (dst && buf && n > 0)
      TF_CHECK_CUDA(cudaMemcpy(dst, buf, sizeof(unsigned long long) * (size_t)n * kTraceCtas * 8,
                               cudaMemcpyDeviceToHost));
    if (names)
      for (int i = 0; i < n; ++i) names[i] = g_trace_names[i];
  });
  return rc != TF_OK ? -rc : n;
}

int tf_session_launches_per_step(void* session) {
  if (!session) return -1;
  return static_cast<Session*>(session)->launches_last;
}

}  // extern "C"
