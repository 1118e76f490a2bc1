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
#include <string>
#include <vector>

#include "../../include/tinfer_sm100.h"
#include "attention.cuh"
#include "beam.cuh"
#include "decode_mk.cuh"
#include "common.cuh"
#include "gemm_tc.cuh"
#include "dgemm.cuh"
#include "norm_embed.cuh"

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

// max shared-memory carveout, once per kernel (see set_max_carveout)
bool carveout_on() {
  static const bool on = [] {  // TF_CARVEOUT=0 disables (A/B diagnostics)
    const char* e = getenv("TF_CARVEOUT");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <typename Kern, typename... Args>
void launch_mc(Kern kern, dim3 grid, dim3 block, size_t smem, cudaStream_t st, bool pdl, Args... args) {
  static bool done = false;  // one flag per kernel instantiation
  if (!done && carveout_on()) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
    done = true;
  }
  launch_cluster(kern, grid, block, smem, st, pdl, 1, args...);
}

int g_num_sms = 0;
int num_sms() {
  if (g_num_sms == 0) {
    int dev = 0;
    TF_CHECK_CUDA(cudaGetDevice(&dev));
    TF_CHECK_CUDA(cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev));
  }
  return g_num_sms;
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

// Every SM keeps the maximum shared-memory carveout, whatever kernel runs on
// it: with programmatic dependent launch the next kernel's CTAs are placed
// while the current kernel's are resident, and an SM configured for a small
// carveout cannot take them until it drains.
template <typename K>
void set_max_carveout(K kern) {
  if (carveout_on())
    TF_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributePreferredSharedMemoryCarveout,
                                       (int)cudaSharedmemCarveoutMaxShared));
}

template <int MODE, bool SWAP, int RED, int LNV>
void ensure_gemm_attr() {
  static bool done = false;
  if (!done) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<MODE, SWAP, RED, LNV>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
    TF_CHECK_CUDA(cudaFuncSetAttribute(gemm_tc_kernel<MODE, SWAP, RED, LNV>,
                                       cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    set_max_carveout(gemm_tc_kernel<MODE, SWAP, RED, LNV>);
    done = true;
  }
}

// ------------------------------------------------------------------ GEMM planning
struct GemmPlan {
  bool swap;
  int bn, tiles_a, tiles_b, k_blocks, splits, stages;
};

// Deterministic split count: a function of (features, K, row tiles), so
// decode results are batch-invariant for batches <= 64 (one row tile); above
// that the row-tile count can change the split (and summation) order. Splits form one cluster per
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

GemmPlan plan_gemm(const tf_gemm_desc& d, bool ln_coop = false) {
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
    const int cap_bn = d.epilogue == TF_EPI_LOGITS ? 256 : bn_max;
    const int mt = d.m_tok < cap_bn ? d.m_tok : cap_bn;
    p.bn = ((mt + 15) / 16) * 16;
    if (p.bn < 16) p.bn = 16;
    p.tiles_a = (d.n_feat + 127) / 128;
    p.tiles_b = (d.m_tok + p.bn - 1) / p.bn;
  } else {
    static const int pf_bn = [] {  // TF_PF_BN: prefill feature tile (A/B)
      const char* e = getenv("TF_PF_BN");
      return e ? atoi(e) : 0;
    }();
    // 128-wide feature tiles with a 3-stage ring: two CTAs per SM, so one's
    // epilogue overlaps the other's main loop (C2 prefill GEMMs 2.57 -> 1.86 ms)
    p.bn = pf_bn ? pf_bn : 128;
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
    p.splits = (p.swap && d.epilogue != TF_EPI_LOGITS) ? pick_splits(p.tiles_a * p.tiles_b, p.k_blocks) : 1;
    static const int kb_target = [] {  // diagnostics: TF_KB_PER=n -> fewest splits with <= n K-blocks each
      const char* e = getenv("TF_KB_PER");
      return e ? atoi(e) : 0;
    }();
    if (kb_target > 0 && p.swap && d.epilogue != TF_EPI_LOGITS && !d.ln_x) {
      int best = p.k_blocks <= 16 ? p.k_blocks : 16;
      for (int dd = 1; dd <= 16 && dd <= p.k_blocks; ++dd)
        if (p.k_blocks % dd == 0 && p.k_blocks / dd <= kb_target) {
          best = dd;
          break;
        }
      p.splits = best;
    }
    if (p.swap && d.ln_x && d.epilogue != TF_EPI_LOGITS && !ln_coop) {
      // fused LN: the CTA's normalised K-slice must fit beside the ring
      while (gemm_ln_bytes(p.bn, p.k_blocks / p.splits, p.k_blocks) > 128 * 1024) {
        int next = p.splits + 1;
        while (next <= 16 && p.k_blocks % next) ++next;
        if (next > 16) break;
        p.splits = next;
      }
    }
  }
  TF_REQUIRE(p.splits == 1 || d.epilogue != TF_EPI_LOGITS, TF_ERR_ARG,
             "argmax epilogue does not support split-K");
  const int kb_per = p.k_blocks / p.splits;
  const int stage_bytes = gemm_stage_bytes(p.bn);
  const size_t ln_bytes = (p.swap && d.ln_x) ? (ln_coop ? gemm_ln_coop_bytes(p.bn, kb_per, p.splits)
                                                        : gemm_ln_bytes(p.bn, kb_per, p.k_blocks))
                                             : 0;
  int st = (int)((kMaxSmem - 4096 - ln_bytes - gemm_recv_bytes(p.bn, p.splits, p.swap)) / stage_bytes);
  if (!p.swap) {  // leave room for the staged output tile (smem-bytes check below)
    while (st > 1 && gemm_smem_bytes(p.bn, st, p.splits, false) > kMaxSmem) --st;
  }
  if (st > 8) st = 8;
  static const int pf_stages = [] {  // TF_PF_STAGES caps the prefill (non-swap) ring (A/B)
    const char* e = getenv("TF_PF_STAGES");
    return e ? atoi(e) : 3;
  }();
  if (!p.swap && pf_stages > 0 && st > pf_stages) st = pf_stages;
  // many independent full-K tiles (lm_head): a shallow ring lets 3 CTAs share
  // an SM so one CTA's epilogue overlaps the others' weight streaming
  static const int lm_stages = [] {  // TF_LM_STAGES (A/B)
    const char* e = getenv("TF_LM_STAGES");
    return e ? atoi(e) : 3;
  }();
  if (p.swap && p.splits == 1 && p.tiles_a * p.tiles_b > 148 && st > lm_stages) st = lm_stages;
  if (st > kb_per) st = kb_per;
  if (st < 1) st = 1;
  p.stages = st;
  return p;
}

template <int MODE, bool SWAP, int RED, int LNV>
void launch_gemm_v(const tf_gemm_desc& d, const GemmPlan& p, const CUtensorMap& ta, const CUtensorMap& tb,
                   const GemmArgs& args, cudaStream_t st) {
  ensure_gemm_attr<MODE, SWAP, RED, LNV>();
  dim3 grid(p.tiles_a, p.tiles_b, p.splits);
  const size_t ln_bytes =
      LNV == 2 ? gemm_ln_coop_bytes(p.bn, p.k_blocks / p.splits, p.splits)
               : (LNV == 1 ? gemm_ln_bytes(p.bn, p.k_blocks / p.splits, p.k_blocks) : 0);
  const size_t smem = gemm_smem_bytes(p.bn, p.stages, p.splits, SWAP, ln_bytes);
  if (RED == RED_ROWLN)
    launch_cluster3(gemm_tc_kernel<MODE, SWAP, RED, LNV>, grid, dim3(gemm_threads(MODE, SWAP, RED, LNV)), smem, st,
                    d.pdl != 0, grid, ta, tb, args);
  else
    launch_cluster(gemm_tc_kernel<MODE, SWAP, RED, LNV>, grid, dim3(gemm_threads(MODE, SWAP, RED, LNV)), smem, st,
                   d.pdl != 0, p.splits, ta, tb,
                   args);
}

// One kernel instantiation per (epilogue, operand order, reduction path,
// operand LayerNorm): each carries only the code it executes.
template <int MODE, bool SWAP>
void launch_gemm_t(const tf_gemm_desc& d, const GemmPlan& p, const CUtensorMap& ta,
                   const CUtensorMap& tb, const GemmArgs& args, cudaStream_t st) {
  const int red = args.row_ln ? RED_ROWLN
                  : args.lnf_cnt ? RED_PUSHLN
                  : (p.splits == 1 ? RED_ONE : (gemm_push_reduce(p.bn, p.splits, SWAP) ? RED_PUSH : RED_PULL));
  const int lnv = (SWAP && d.ln_x) ? (args.ln_coop ? 2 : 1) : 0;
  if constexpr (!SWAP) {
    // opt-in (TF_PF_PERSIST=1): measured slower than two one-tile CTAs per SM,
    // whose two epilogues run side by side (the ~6 us staged epilogue bounds both)
    static const bool persist = [] {
      const char* e = getenv("TF_PF_PERSIST");
      return e && e[0] == '1';
    }();
    if (red == RED_ONE && persist && (MODE != EPI_LOGITS || args.keys == nullptr)) {
      // persistent tile loop, two TMEM accumulators, ring as deep as smem allows
      static bool done = false;
      if (!done) {
        TF_CHECK_CUDA(cudaFuncSetAttribute(gemm_pf_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           (int)kMaxSmem));
        done = true;
      }
      GemmArgs a2 = args;
      const size_t fixed = gemm_pf_smem_bytes(p.bn, 0, MODE == EPI_F32);
      int stages = (int)((kMaxSmem - fixed) / gemm_stage_bytes(p.bn));
      stages = std::max(2, std::min(stages, 8));
      a2.stages = stages;
      const int n_tiles = p.tiles_a * p.tiles_b;
      const dim3 grid(std::min(n_tiles, num_sms()));
      return launch_cluster(gemm_pf_kernel<MODE>, grid, dim3(kPfThreadsGemm),
                            gemm_pf_smem_bytes(p.bn, stages, MODE == EPI_F32), st, d.pdl != 0, 1, ta, tb, a2);
    }
    if (red == RED_ONE) return launch_gemm_v<MODE, false, RED_ONE, 0>(d, p, ta, tb, args, st);
    return launch_gemm_v<MODE, false, RED_PULL, 0>(d, p, ta, tb, args, st);
  } else {
    if (red == RED_ROWLN) {
      if constexpr (MODE == EPI_BIAS_RESID) return launch_gemm_v<MODE, true, RED_ROWLN, 0>(d, p, ta, tb, args, st);
      throw TfError{TF_ERR_UNSUPPORTED, "gemm: row-LN epilogue needs EPI_BIAS_RESID"};
    }
    if (red == RED_PUSHLN) {
      if constexpr (MODE == EPI_BIAS_RESID) return launch_gemm_v<MODE, true, RED_PUSHLN, 0>(d, p, ta, tb, args, st);
      throw TfError{TF_ERR_UNSUPPORTED, "gemm: last-arriver LN epilogue needs EPI_BIAS_RESID"};
    }
    if (lnv == 0) {
      if (red == RED_ONE) return launch_gemm_v<MODE, true, RED_ONE, 0>(d, p, ta, tb, args, st);
      if (red == RED_PUSH) return launch_gemm_v<MODE, true, RED_PUSH, 0>(d, p, ta, tb, args, st);
      return launch_gemm_v<MODE, true, RED_PULL, 0>(d, p, ta, tb, args, st);
    }
    constexpr bool ln_ok = MODE == EPI_F32 || MODE == EPI_QKV || MODE == EPI_BIAS_GELU || MODE == EPI_LOGITS;
    if constexpr (ln_ok) {
      if (lnv == 1) {
        if (red == RED_ONE) return launch_gemm_v<MODE, true, RED_ONE, 1>(d, p, ta, tb, args, st);
        if (red == RED_PUSH) return launch_gemm_v<MODE, true, RED_PUSH, 1>(d, p, ta, tb, args, st);
        return launch_gemm_v<MODE, true, RED_PULL, 1>(d, p, ta, tb, args, st);
      }
      if (red == RED_ONE) return launch_gemm_v<MODE, true, RED_ONE, 2>(d, p, ta, tb, args, st);
      if (red == RED_PUSH) return launch_gemm_v<MODE, true, RED_PUSH, 2>(d, p, ta, tb, args, st);
      return launch_gemm_v<MODE, true, RED_PULL, 2>(d, p, ta, tb, args, st);
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
  int ln_coop = 0;  // with desc.ln_x: cooperative cluster LayerNorm (gemm_tc.cuh ln_coop_build)
  int row_ln = 0;   // EPI_BIAS_RESID: whole rows in one cluster + fused LN (gemm_rowln_epilogue)
  int* lnf_cnt = nullptr;  // EPI_BIAS_RESID push split-K: LN of completed rows by their last CTA
  const float* lnf_g = nullptr;
  const float* lnf_b = nullptr;
  void* lnf_h = nullptr;
  int lnf_ldh = 0;
};


void run_gemm(const tf_gemm_desc& d, cudaStream_t st, const GemmExtra& ex = GemmExtra{}) {
  TF_REQUIRE(d.m_tok > 0 && d.n_feat > 0 && d.k > 0, TF_ERR_SHAPE, "gemm: empty shape");
  TF_REQUIRE(d.act && d.wt, TF_ERR_ARG, "gemm: null operand");
  const GemmPlan p = plan_gemm(d, d.ln_x != nullptr && ex.ln_coop != 0);
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
  if (ex.lnf_cnt) {
    TF_REQUIRE(p.swap && gemm_push_reduce(p.bn, p.splits, true) && d.epilogue == TF_EPI_BIAS_RESID &&
                   d.n_feat <= 1024 && d.n_feat % 8 == 0 && d.ldo % 8 == 0 && ex.lnf_g && ex.lnf_b && ex.lnf_h &&
                   ex.lnf_ldh % 8 == 0 && p.bn / 32 + 2 <= 64,
               TF_ERR_ARG, "gemm: last-arriver LN epilogue not applicable");
    a.lnf_cnt = ex.lnf_cnt;
    a.lnf_g = ex.lnf_g;
    a.lnf_b = ex.lnf_b;
    a.lnf_h = static_cast<__half*>(ex.lnf_h);
    a.lnf_ldh = ex.lnf_ldh;
  }
  if (ex.row_ln) {
    TF_REQUIRE(p.swap && p.splits == 2 && d.epilogue == TF_EPI_BIAS_RESID && p.tiles_b == 1 && p.bn <= 64 &&
                   p.tiles_a * 2 <= 16 && ex.lnf_g && ex.lnf_b && ex.lnf_h &&
                   gemm_ring_bytes(p.bn, p.stages, p.splits, true) >= gemm_rowln_scratch_bytes(p.bn, p.tiles_a),
               TF_ERR_ARG, "gemm: row-LN epilogue not applicable");
    a.row_ln = 1;
    a.lnf_g = ex.lnf_g;
    a.lnf_b = ex.lnf_b;
    a.lnf_h = static_cast<__half*>(ex.lnf_h);
    a.lnf_ldh = ex.lnf_ldh;
  }
  static const char* kGemmNames[] = {"gemm_f32", "gemm_bias", "gemm_gelu", "gemm_resid", "gemm_qkv", "gemm_logits"};
  a.trace = trace_next(d.epilogue >= 0 && d.epilogue < 6 ? kGemmNames[d.epilogue] : "gemm");
  if (d.ln_x) {
    TF_REQUIRE(p.swap, TF_ERR_UNSUPPORTED, "gemm: fused LayerNorm needs the swap-AB (decode) path");
    TF_REQUIRE(d.ln_gamma && d.ln_beta && d.ln_hidden > 0 && d.ln_hidden <= 1024 && d.ln_hidden % 8 == 0 &&
                   d.ln_ldx % 8 == 0 && d.ln_hidden <= kext,
               TF_ERR_ARG, "gemm: bad fused LayerNorm arguments");
    TF_REQUIRE(ex.ln_coop || gemm_ln_bytes(p.bn, p.k_blocks / p.splits, p.k_blocks) <= 128 * 1024,
               TF_ERR_UNSUPPORTED, "gemm: fused LayerNorm tile too large");
    TF_REQUIRE(!ex.ln_coop || (d.ln_hidden == d.k && p.splits <= 16), TF_ERR_ARG,
               "gemm: cooperative LayerNorm needs K == hidden");
    a.ln_coop = ex.ln_coop;
    a.ln_x = static_cast<const __half*>(d.ln_x);
    a.ln_ldx = d.ln_ldx;
    a.ln_src_stride = d.ln_src_stride;
    a.ln_src_off = d.ln_src_off;
    a.ln_H = d.ln_hidden;
    a.ln_g = d.ln_gamma;
    a.ln_b = d.ln_beta;
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
  int ldp = p.swap ? d.ldw : d.lda, ldq = p.swap ? d.lda : d.ldw;
  if (d.ln_x) {  // fused LN: the B map stages the (strided) LN source rows instead
    Q = static_cast<const __half*>(d.ln_x) + (size_t)d.ln_src_off * d.ln_ldx;
    ldq = d.ln_ldx * d.ln_src_stride;
  }
  const CUtensorMap ta = make_kmajor_map(P, a.rows_a, kext, ldp, kTileA);
  const CUtensorMap tb = make_kmajor_map(Q, a.rows_b, kext, ldq, p.bn);
  switch (d.epilogue) {
    case TF_EPI_F32: launch_gemm_mode<EPI_F32>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS: launch_gemm_mode<EPI_BIAS>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS_GELU: launch_gemm_mode<EPI_BIAS_GELU>(d, p, ta, tb, a, st); break;
    case TF_EPI_BIAS_RESID: launch_gemm_mode<EPI_BIAS_RESID>(d, p, ta, tb, a, st); break;
    case TF_EPI_QKV: launch_gemm_mode<EPI_QKV>(d, p, ta, tb, a, st); break;
    case TF_EPI_LOGITS: launch_gemm_mode<EPI_LOGITS>(d, p, ta, tb, a, st); break;
  }
}

// ------------------------------------------------------------------ small-batch decode GEMM
struct DgPlan {
  int bn, nkb, splits, tiles_f;
};

int dg_kb_max() {  // K blocks per CTA (TF_DG_KB, diagnostics)
  static const int v = [] {
    const char* e = getenv("TF_DG_KB");
    return e ? std::max(1, atoi(e)) : 12;
  }();
  return v;
}

// dgemm_kernel applies when the whole batch fits one 16..64-row operand tile and
// the CTA's K slice (<= dg_kb_max blocks, K split <= 4 ways) fits shared memory
bool dg_plan(int m_tok, int n_feat, int k, DgPlan& pl) {
  if (m_tok < 1 || m_tok > 64) return false;
  pl.bn = std::max(16, (m_tok + 15) / 16 * 16);
  const int kb = (k + 63) / 64;
  int S = 1;
  while (S <= 4 && (kb % S != 0 || kb / S > dg_kb_max())) ++S;
  if (S > 4) return false;
  pl.splits = S;
  pl.nkb = kb / S;
  pl.tiles_f = (n_feat + kDgRows - 1) / kDgRows;
  return dg_smem_bytes(pl.bn, pl.nkb) <= kMaxSmem;
}

template <int MODE, int NC>
void launch_dg(const DgPlan& pl, const CUtensorMap& tw, const CUtensorMap& ta, const DgArgs& a, cudaStream_t st,
               bool pdl) {
  static bool done = false;
  if (!done) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(dgemm_kernel<MODE, NC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kMaxSmem));
    set_max_carveout(dgemm_kernel<MODE, NC>);
    done = true;
  }
  launch_cluster(dgemm_kernel<MODE, NC>, dim3(pl.tiles_f, 1, pl.splits), dim3(kDgThreads),
                 dg_smem_bytes(pl.bn, pl.nkb), st, pdl, pl.splits, tw, ta, a);
}

template <int MODE>
void launch_dg_ln(const DgPlan& pl, const CUtensorMap& tw, const CUtensorMap& ta, const DgArgs& a, cudaStream_t st,
                  bool pdl) {
  if (a.ln_g == nullptr) return launch_dg<MODE, 0>(pl, tw, ta, a, st, pdl);
  switch ((a.ln_H / 8 + 31) / 32) {
    case 1: return launch_dg<MODE, 1>(pl, tw, ta, a, st, pdl);
    case 2: return launch_dg<MODE, 2>(pl, tw, ta, a, st, pdl);
    case 3: return launch_dg<MODE, 3>(pl, tw, ta, a, st, pdl);
    case 4: return launch_dg<MODE, 4>(pl, tw, ta, a, st, pdl);
    default: throw TfError{TF_ERR_UNSUPPORTED, "dgemm: fused LayerNorm needs hidden <= 1024"};
  }
}

// d: the usual GEMM descriptor (swap-AB decode shape, T == 1 for EPI_QKV);
// ln_g/ln_b: fused LayerNorm of the operand rows (d.k == hidden) or null
void run_dgemm(const tf_gemm_desc& d, const DgPlan& pl, const float* ln_g, const float* ln_b, const GemmExtra& ex,
               cudaStream_t st) {
  const int kext = pl.nkb * pl.splits * 64;
  TF_REQUIRE(d.lda >= kext && d.ldw >= kext && d.lda % 8 == 0 && d.ldw % 8 == 0 && d.ldo % 8 == 0, TF_ERR_SHAPE,
             "dgemm: leading dimensions");
  TF_REQUIRE(pl.splits == 1 || (d.epilogue != TF_EPI_QKV && d.n_feat % 4 == 0), TF_ERR_ARG, "dgemm: split epilogue");
  TF_REQUIRE(d.n_feat % 8 == 0, TF_ERR_SHAPE, "dgemm: features must be a multiple of 8");
  TF_REQUIRE(ln_g == nullptr || (d.k % 8 == 0 && d.k <= 1024 && pl.splits == 1), TF_ERR_ARG,
             "dgemm: fused LayerNorm needs the whole row in one CTA");
  DgArgs a{};
  a.m_tok = d.m_tok;
  a.n_feat = d.n_feat;
  a.bn = pl.bn;
  a.nkb = pl.nkb;
  a.splits = pl.splits;
  a.bias = d.bias;
  a.out = static_cast<__half*>(d.out);
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
  a.qbase_dev = d.qbase_dev;
  a.ln_g = ln_g;
  a.ln_b = ln_b;
  a.ln_H = d.k;
  a.l2pf = ex.l2pf;
  a.l2pf_bytes = ex.l2pf_bytes;
  const CUtensorMap tw = make_kmajor_map(d.wt, d.n_feat, kext, d.ldw, kDgRows);
  const CUtensorMap ta = make_kmajor_map(d.act, d.m_tok, kext, d.lda, pl.bn);
  const bool pdl = d.pdl != 0;
  switch (d.epilogue) {
    case TF_EPI_QKV:
      TF_REQUIRE(d.head_dim % 8 == 0 && d.seq_len == 1, TF_ERR_ARG, "dgemm: qkv routing");
      a.trace = trace_next("dg_qkv");
      launch_dg_ln<EPI_QKV>(pl, tw, ta, a, st, pdl);
      break;
    case TF_EPI_BIAS_RESID:
      a.trace = trace_next("dg_resid");
      launch_dg<EPI_BIAS_RESID, 0>(pl, tw, ta, a, st, pdl);
      break;
    case TF_EPI_BIAS_GELU:
      a.trace = trace_next("dg_gelu");
      launch_dg_ln<EPI_BIAS_GELU>(pl, tw, ta, a, st, pdl);
      break;
    default:
      throw TfError{TF_ERR_UNSUPPORTED, "dgemm: epilogue"};
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
  static const bool early = [] {  // TF_LN_EARLY=1: LN releases its successor before its own wait (A/B)
    const char* e = getenv("TF_LN_EARLY");
    return e && e[0] == '1';
  }();
  a.early_trigger = early ? 1 : 0;
  a.trace = trace_next("layernorm");
  const dim3 grid((a.n_rows + 7) / 8);
  static const int ln_rpc = [] {  // TF_LN_RPC: rows (warps) per CTA of the vector LN kernel (A/B)
    const char* e = getenv("TF_LN_RPC");
    const int v = e ? atoi(e) : 8;
    return v == 1 || v == 2 || v == 4 || v == 8 ? v : 8;
  }();
  const dim3 vgrid((a.n_rows + ln_rpc - 1) / ln_rpc), vblock(32 * ln_rpc);
  if (vec_ok(a.H, a.ldx, a.ldh) && a.H <= 2048) {
    const int nc = (a.H / 8 + 31) / 32;
    switch (nc) {
      case 1: launch_mc(layernorm_vec_kernel<1>, vgrid, vblock, 0, st, pdl, a); return;
      case 2: launch_mc(layernorm_vec_kernel<2>, vgrid, vblock, 0, st, pdl, a); return;
      case 3: launch_mc(layernorm_vec_kernel<3>, vgrid, vblock, 0, st, pdl, a); return;
      case 4: launch_mc(layernorm_vec_kernel<4>, vgrid, vblock, 0, st, pdl, a); return;
      case 6: launch_mc(layernorm_vec_kernel<6>, vgrid, vblock, 0, st, pdl, a); return;
      case 8: launch_mc(layernorm_vec_kernel<8>, vgrid, vblock, 0, st, pdl, a); return;
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

template <bool WO, int THREADS, int MINB = 1>
void launch_pf(dim3 grid, size_t smem, cudaStream_t st, bool pdl, const AttnArgs& t) {
  static bool attr = false;
  if (!attr) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(attn_decode_pf_kernel<WO, THREADS, MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)attn_pf_smem_bytes(kPfMaxG)));
    set_max_carveout(attn_decode_pf_kernel<WO, THREADS, MINB>);
    attr = true;
  }
  launch(attn_decode_pf_kernel<WO, THREADS, MINB>, grid, dim3(THREADS), smem, st, pdl, t);
}

template <int MINB>
void launch_beam_ring(dim3 grid, size_t smem, cudaStream_t st, bool pdl, const AttnArgs& t, int planes) {
  static bool attr = false;
  if (!attr) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(attn_decode_beam_ring_kernel<MINB>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(kMaxSmem - 2048)));
    set_max_carveout(attn_decode_beam_ring_kernel<MINB>);
    attr = true;
  }
  launch(attn_decode_beam_ring_kernel<MINB>, grid, dim3(kBmThreads), smem, st, pdl, t, planes);
}

void run_attention(const AttnArgs& a, cudaStream_t st, bool pdl) {
  TF_REQUIRE(a.D >= 1 && a.D <= 128, TF_ERR_UNSUPPORTED, "head_dim must be in [1, 128]");
  static const int pf_mode = [] {  // TF_ATTN_PF=0 selects the split kernel (A/B diagnostics)
    const char* e = getenv("TF_ATTN_PF");
    return e ? atoi(e) : 1;
  }();
  static const int beam_mode = [] {  // TF_ATTN_BEAM: 0 per-row CTAs, 1 batched staging, 2 ring (A/B)
    const char* e = getenv("TF_ATTN_BEAM");
    return e ? atoi(e) : 2;
  }();
  if (a.T == 1 && a.D == 64 && a.indir && a.beam >= 2 && a.B % a.beam == 0 && a.cap <= kBmMaxCh * 64 &&
      a.wo_t == nullptr && beam_mode) {
    // one CTA per (head, request): prompt chunks staged once for all beams.
    // Mode 2 (default): ring-pipelined, two CTAs per SM when a 6-plane ring fits
    if (beam_mode == 2) {
      const int R = a.beam;
      const size_t half = 115712 - 512;  // per-CTA share of the SM with two resident
      const int p2 = (int)((half - attn_beam_ring_aux_bytes(R)) / kPfChunkBytes);
      AttnArgs t = a;
      t.trace = trace_next("attn_decode_beam");
      const dim3 grid(1, a.NH, a.B / a.beam);
      if (p2 >= R) {
        const int planes = std::min(p2, 6);
        launch_beam_ring<2>(grid, attn_beam_ring_aux_bytes(R) + (size_t)planes * kPfChunkBytes, st, pdl, t, planes);
      } else {
        const int planes = (int)std::min<size_t>(12, (kMaxSmem - 2048 - attn_beam_ring_aux_bytes(R)) / kPfChunkBytes);
        TF_REQUIRE(planes >= R, TF_ERR_UNSUPPORTED, "beam attention: plane pool smaller than the beam");
        launch_beam_ring<1>(grid, attn_beam_ring_aux_bytes(R) + (size_t)planes * kPfChunkBytes, st, pdl, t, planes);
      }
      return;
    }
    const int planes = (int)std::min<size_t>(12, (kMaxSmem - 2048 - attn_beam_aux_bytes(a.beam)) / kPfChunkBytes);
    TF_REQUIRE(planes >= a.beam, TF_ERR_UNSUPPORTED, "beam attention: plane pool smaller than the beam");
    const size_t smem = attn_beam_smem_bytes(a.beam, planes);
    static bool attr = false;
    if (!attr) {
      TF_CHECK_CUDA(cudaFuncSetAttribute(attn_decode_beam_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kMaxSmem - 2048)));  // + the kernel's static smem
      set_max_carveout(attn_decode_beam_kernel);
      attr = true;
    }
    AttnArgs t = a;
    t.trace = trace_next("attn_decode_beam");
    launch(attn_decode_beam_kernel, dim3(1, a.NH, a.B / a.beam), dim3(kBmThreads), smem, st, pdl, t, planes);
  } else if (a.T == 1 && a.D == 64 && a.ws && a.cnt && a.max_chunks >= (a.cap + kSplitKeys - 1) / kSplitKeys &&
             pf_mode) {
    // chunks per CTA: the whole window when it is <= 4 chunks (local merge),
    // else groups of <= 4 (64 KB of K/V each) merged through the workspace
    static const int gmax = [] {  // TF_ATTN_G: max 64-slot chunks per CTA (A/B), <= kPfMaxG
      const char* e = getenv("TF_ATTN_G");
      return e ? std::max(1, std::min(kPfMaxG, atoi(e))) : 4;
    }();
    const int nch = a.max_chunks;
    const int ngr = (nch + gmax - 1) / gmax;
    TF_REQUIRE(a.wo_t == nullptr || ngr == 1, TF_ERR_ARG, "attention: fused Wo needs the window in one CTA");
    AttnArgs t = a;
    t.group = (nch + ngr - 1) / ngr;
    t.trace = trace_next("attn_decode_pf");
    const size_t smem = attn_pf_smem_bytes(t.group);
    // 128 threads by default; TF_ATTN_WIDE=1 selects 256 threads (registers
    // capped for 3 CTAs per SM while the grid fits one such wave, uncapped for
    // multi-wave grids): faster in the eager trace, within noise / slightly
    // slower in graph-replayed bench runs on the same box (C2 85.3k vs 86.5k,
    // C3 178.1k vs 181.8k)
    static const int wide_env = [] {
      const char* e = getenv("TF_ATTN_WIDE");
      return e ? atoi(e) : 0;
    }();
    const size_t ctas = (size_t)ngr * a.NH * a.B;
    const bool one_wave = ctas <= (size_t)3 * num_sms();
    const dim3 grid(ngr, a.NH, a.B);
    if (a.wo_t) {
      if (wide_env == 0)
        launch_pf<true, 128>(grid, smem, st, pdl, t);
      else if (one_wave)
        launch_pf<true, 256, 3>(grid, smem, st, pdl, t);
      else
        launch_pf<true, 256>(grid, smem, st, pdl, t);
    } else {
      if (wide_env == 0)
        launch_pf<false, 128>(grid, smem, st, pdl, t);
      else if (one_wave)
        launch_pf<false, 256, 3>(grid, smem, st, pdl, t);
      else
        launch_pf<false, 256>(grid, smem, st, pdl, t);
    }
  } else if (a.T == 1 && a.D == 64 && a.ws && a.cnt && a.max_chunks >= (a.cap + kSplitKeys - 1) / kSplitKeys) {
    AttnArgs t = a;
    t.trace = trace_next("attn_decode_split");
    launch(attn_decode_split_kernel, dim3(a.max_chunks, a.NH, a.B), dim3(kSplitThreads), 0, st, pdl, t);
  } else if (a.T == 1) {
    const size_t smem = (size_t)(a.D + a.cap + std::max(2 * kDecThreads, kDecWarps * a.D)) * sizeof(float);
    TF_REQUIRE(smem <= kMaxSmem, TF_ERR_UNSUPPORTED, "cache capacity too large for decode kernel");
    static bool attr = false;
    if (!attr) {
      TF_CHECK_CUDA(cudaFuncSetAttribute(attn_decode_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxSmem));
      attr = true;
    }
    launch(attn_decode_kernel, dim3(a.NH, a.B), dim3(kDecThreads), smem, st, pdl, a);
  } else if (a.D == 64 && a.ldq % 8 == 0 && a.ldo % 2 == 0) {
    launch(attn_prefill_mma_kernel, dim3((a.T + kFaRows - 1) / kFaRows, a.NH, a.B), dim3(128), 0, st, pdl, a);
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

// Session-owned scratch of the persistent decode megakernel (allocated on first use).
struct MkState {
  bool ready = false;
  int bn = 0, ws = 0, bs = 0, att_slots = 0, grid = 0, n_ctr = 0;
  void* mem = nullptr;  // one allocation carved into the pieces below
  __half *x, *h1, *h2, *attn, *hf, *q, *f;
  float* p_w2;
  int* ctr;
  int4* items;
  int* item_off;
  int4* aux;
  int* aux_off;
  mk::Layer* layers;
  mk::Maps maps;
};

struct Session {
  Model* m;
  tf_session_desc d;
  MkState mk;
  cudaGraphExec_t graph = nullptr;
  cudaGraphExec_t graph_multi = nullptr;  // TF_GRAPH_STEPS decode steps
  cudaGraphExec_t beam_graph = nullptr;
  tf_beam_desc beam_key{};  // descriptor the beam graph was captured with
  int graph_launches = 0;
  int launches_last = 0;
};

int* qbase_zero_ptr() {
  // device scalar 0 for operator calls that start at slot 0
  static int* p = nullptr;
  if (!p) {
    TF_CHECK_CUDA(cudaMalloc(&p, sizeof(int)));
    TF_CHECK_CUDA(cudaMemset(p, 0, sizeof(int)));
  }
  return p;
}

// One forward of T tokens per sequence through every layer. Returns the number
// of kernels launched.
int forward(Session& s, const int* ids, const int* pos, int T, int mode, bool pdl,
            cudaStream_t st, bool remap_ids = true) {
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
  e.ldw = m.ldw;
  e.ln_g = s.m->layers[0].ln1_gamma;
  e.ln_b = s.m->layers[0].ln1_beta;
  e.x = x;
  e.h = h;
  e.ldx = m.ldk_h;
  run_embed(e, st, pdl);
  ++launches;

  tf_gemm_desc g{};
  g.m_tok = M;
  g.force_swap = -1;
  g.workspace = sd.workspace;
  g.workspace_bytes = sd.workspace_bytes;
  g.counters = sd.counters;
  g.n_counters = sd.n_counters;
  g.pdl = pdl ? 1 : 0;

  // decode (every GEMM swap-AB): LayerNorms are fused into the consuming GEMM's
  // operand build instead of running as separate kernels
  // measured slower than the stand-alone LN kernel under PDL (the fused build
  // adds dependent row loads to every GEMM's critical path): opt-in only
  static const bool fuse_opt = [] {
    const char* e = getenv("TF_FUSE_LN");
    return e && e[0] == '1';
  }();
  const bool fuse_ln = fuse_opt && M <= 64 && H <= 1024 && H % 8 == 0 && m.ldk_h % 8 == 0;
  // the lm_head (argmax epilogue, no split-K) fuses only if its full-K tile fits
  const int lg_rows = (mode == TF_FWD_LOGITS_ALL) ? M : B;
  const bool fuse_final = fuse_ln && lg_rows <= 256 &&
                          gemm_ln_bytes(((std::min(lg_rows, 256) + 15) / 16) * 16, pad64(H) / 64, pad64(H) / 64) <=
                              128 * 1024;
  auto set_ln = [&](tf_gemm_desc& d, const float* gam, const float* bet, int stride, int off) {
    d.ln_x = x;
    d.ln_ldx = m.ldk_h;
    d.ln_src_stride = stride;
    d.ln_src_off = off;
    d.ln_hidden = H;
    d.ln_gamma = gam;
    d.ln_beta = bet;
  };

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
  auto pf_next = [&](int l, int which) {
    GemmExtra ex;
    const void*& ptr = ex.l2pf;
    unsigned long long& bytes = ex.l2pf_bytes;
    if (!l2pf) return ex;
    if (l + 1 < L) {
      const tf_layer_weights& n = s.m->layers[l + 1];
      switch (which) {
        case 0: ptr = n.wqkv_t; bytes = 3ull * H * m.ldk_h * 2; break;
        case 1: ptr = n.wo_t; bytes = (unsigned long long)H * m.ldk_h * 2; break;
        case 2: ptr = n.w1_t; bytes = (unsigned long long)F * m.ldk_h * 2; break;
        default: ptr = n.w2_t; bytes = (unsigned long long)H * m.ldk_f * 2; break;
      }
    } else {
      const unsigned long long lo = which * lm_q;
      if (lo >= lm_bytes) return ex;
      ptr = static_cast<const uint8_t*>(m.lm_head_t) + lo;
      bytes = std::min(lm_q, lm_bytes - lo);
    }
    return ex;
  };

  // small-batch decode: narrow-tile whole-K GEMMs with the LayerNorms fused
  // into the QKV / FFN1 operand (dgemm.cuh). Opt-in (TF_DGEMM=1): the whole-K
  // MMA chain (~35 cycles per tcgen05.mma issue) and the per-CTA LayerNorm of
  // all rows cost more than the split-K reduction they remove.
  static const bool dg_on = [] {
    const char* e = getenv("TF_DGEMM");
    return e && e[0] == '1';
  }();
  DgPlan pq{}, po{}, p1{}, p2{};
  const bool dg = dg_on && T == 1 && !fuse_ln && D % 8 == 0 && H % 8 == 0 && H <= 1024 &&
                  dg_plan(M, 3 * H, H, pq) && dg_plan(M, H, H, po) && dg_plan(M, F, H, p1) && dg_plan(M, H, F, p2) &&
                  pq.splits == 1 && p1.splits == 1;
  // decode: attn_norm / ffn_norm computed by the consuming QKV / FFN1 split-K
  // cluster (cooperative LN, gemm_tc.cuh) instead of stand-alone launches.
  // Opt-in (TF_LN_COOP=1): measured slower in the PDL-chained step
  static const bool coop_on = [] {
    const char* e = getenv("TF_LN_COOP");
    return e && e[0] == '1';
  }();
  const bool coop = coop_on && !dg && !fuse_ln && T == 1 && M <= 256 && H <= 1024 && H % 8 == 0 && m.ldk_h % 8 == 0;
  // decode: the output projection runs inside the attention kernel (per-head
  // partials of o_h @ Wo_h) and the head sum + bias + residual + ffn_norm in one
  // row kernel, replacing the Wo GEMM and the LayerNorm launch. Opt-in
  // (TF_ATTN_WO=1): every attention CTA streams its head's 98 KB Wo slice, which
  // lengthens the attention more than the two launches it removes
  static const bool attn_wo_on = [] {
    const char* e = getenv("TF_ATTN_WO");
    return e && e[0] == '1';
  }();
  const bool attn_wo = attn_wo_on && NH <= 16 && !dg && !fuse_ln && T == 1 && D == 64 && !sd.beam_indir &&
                       (sd.capacity + 63) / 64 <= 4 && H % 8 == 0 && H <= 2048 && m.ldk_h % 8 == 0 &&
                       sd.workspace && sd.workspace_bytes >= (size_t)B * NH * H * sizeof(float) && sd.counters &&
                       sd.n_counters >= B * NH;
  // decode: the LayerNorm after each residual GEMM (Wo -> ffn_norm, FFN2 ->
  // next attn_norm / final_norm) runs in that GEMM's epilogue: the CTA whose
  // stores complete a row normalises it (RED_PUSHLN), no LN launch. Opt-in
  // (TF_LN_TAIL=1): fence + counter + dependent row reload add ~4 us to each
  // residual GEMM vs the 2.4 us LN launch they replace
  static const bool lntail_on = [] {
    const char* e = getenv("TF_LN_TAIL");
    return e && e[0] == '1';
  }();
  int* ln_cnt = (lntail_on && T == 1 && !fuse_ln && !dg && !coop && H <= 1024 && H % 8 == 0 && m.ldk_h % 8 == 0 &&
                 sd.counters && sd.n_counters >= B * NH + M)
                    ? sd.counters + B * NH
                    : nullptr;
  // decode, batch <= 64: the two residual GEMMs (Wo, FFN2) run as ONE cluster
  // covering whole output rows (tiles x 2 K-halves <= 16 CTAs) and fuse the
  // following LayerNorm into their epilogue (gemm_rowln_epilogue). Opt-in
  // (TF_ROWLN=1): 12 CTAs carry the whole weight matrix and three cluster
  // exchange rounds sit on the critical path (measured 4.9 -> 20 us)
  static const bool rowln_on = [] {
    const char* e = getenv("TF_ROWLN");
    return e && e[0] == '1';
  }();
  const bool rowln = rowln_on && !dg && !coop && !fuse_ln && T == 1 && M <= 64 && (H + 127) / 128 <= 8 &&
                     (H / 64) % 2 == 0 && (F / 64) % 2 == 0 && H % 8 == 0;
  if (rowln) ln_cnt = nullptr;
  auto push_plan = [&](const tf_gemm_desc& d) {
    const GemmPlan gp = plan_gemm(d);
    return gp.swap && gemm_push_reduce(gp.bn, gp.splits, true) && gp.bn / 32 + 2 <= 64;
  };

  // diagnostics: TF_SPLITS="q,o,f1,f2" forces the decode split counts (0 = auto)
  static const std::vector<int> force_splits = [] {
    std::vector<int> v(4, 0);
    if (const char* e = getenv("TF_SPLITS")) sscanf(e, "%d,%d,%d,%d", &v[0], &v[1], &v[2], &v[3]);
    return v;
  }();
  const bool fs = T == 1;

  for (int l = 0; l < L; ++l) {
    const tf_layer_weights& w = s.m->layers[l];
    // fused QKV projection, K/V straight into the cache (model.py:464-474)
    tf_gemm_desc q = g;
    if (fuse_ln) set_ln(q, w.ln1_gamma, w.ln1_beta, 1, 0);
    q.n_feat = 3 * H;
    q.k = H;
    q.act = h;
    q.lda = m.ldk_h;
    q.wt = w.wqkv_t;
    q.ldw = m.ldk_h;
    q.epilogue = TF_EPI_QKV;
    q.bias = w.bqkv;
    q.q_out = sd.q;
    q.ldq = m.ldk_h;
    q.k_cache = static_cast<__half*>(sd.k_cache) + l * layer_cache;
    q.v_cache = static_cast<__half*>(sd.v_cache) + l * layer_cache;
    q.hidden = H;
    q.heads = NH;
    q.head_dim = D;
    q.cap = sd.capacity;
    q.seq_len = T;
    q.qbase_dev = sd.len_dev;
    if (fs && force_splits[0]) q.splits = force_splits[0];
    if (coop) set_ln(q, w.ln1_gamma, w.ln1_beta, 1, 0);
    static const bool qkv_late = [] {  // TF_QKV_LATE=0 disables (A/B diagnostics)
      const char* e = getenv("TF_QKV_LATE");
      return !(e && e[0] == '0');
    }();
    // decode: attention (next) prefetches the whole KV window; release it only
    // once the QKV weights are in (after this GEMM's own dependency wait)
    if (pdl && T == 1 && qkv_late) q.pdl = 2;
    static const int late_mask = [] {  // TF_LATE_MASK bits: 1 Wo, 2 FFN1, 4 FFN2 release late (A/B)
      const char* e = getenv("TF_LATE_MASK");
      return e ? atoi(e) : 0;
    }();
    if (dg) {
      q.act = x;  // attn_norm (model.py:460-462) runs on the operand inside the GEMM
      run_dgemm(q, pq, w.ln1_gamma, w.ln1_beta, pf_next(l, 0), st);
    } else {
      GemmExtra qex = pf_next(l, 0);
      qex.ln_coop = coop ? 1 : 0;
      run_gemm(q, st, qex);
    }
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
    }
    if (T == 1 && D == 64) {  // split-KV decode attention when the session provides scratch
      const int chunks = (sd.capacity + kSplitKeys - 1) / kSplitKeys;
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
    if (attn_wo) {
      at.wo_t = static_cast<const __half*>(w.wo_t);
      at.ldw = m.ldk_h;
      at.H = H;
      at.wo_part = sd.workspace;
      const GemmExtra wex = pf_next(l, 1);
      at.l2pf = wex.l2pf;
      at.l2pf_bytes = wex.l2pf_bytes;
    }
    run_attention(at, st, pdl);
    ++launches;
    if (attn_wo) {
      // head sum + bias + residual (model.py:478-482) and ffn_norm (model.py:484-486)
      ResLnArgs r{};
      r.B = B;
      r.NH = NH;
      r.H = H;
      r.part = sd.workspace;
      r.bias = w.bo;
      r.x = x;
      r.ldx = m.ldk_h;
      r.g = w.ln2_gamma;
      r.b = w.ln2_beta;
      r.h = h;
      r.ldh = m.ldk_h;
      r.trace = trace_next("resid_heads_ln");
      launch_mc(resid_heads_ln_kernel, dim3(B), dim3(kResThreads), 0, st, pdl, r);
      ++launches;
    }
    // output projection + residual (model.py:478-482)
    tf_gemm_desc o = g;
    const bool skip_wo = attn_wo;
    o.n_feat = H;
    o.k = H;
    o.act = sd.attn;
    o.lda = m.ldk_h;
    o.wt = w.wo_t;
    o.ldw = m.ldk_h;
    o.epilogue = TF_EPI_BIAS_RESID;
    o.bias = w.bo;
    o.out = x;
    o.ldo = m.ldk_h;
    o.resid = x;
    o.ldr = m.ldk_h;
    if (fs && force_splits[1]) o.splits = force_splits[1];
    GemmExtra oex = pf_next(l, 1);
    if (rowln) {
      o.splits = 2;
      oex.row_ln = 1;
      oex.lnf_g = w.ln2_gamma;
      oex.lnf_b = w.ln2_beta;
      oex.lnf_h = h;
      oex.lnf_ldh = m.ldk_h;
    }
    if (pdl && T == 1 && (late_mask & 1)) o.pdl = 2;
    const bool o_tail = ln_cnt && !skip_wo && push_plan(o);
    if (o_tail) {
      oex.lnf_cnt = ln_cnt;
      oex.lnf_g = w.ln2_gamma;
      oex.lnf_b = w.ln2_beta;
      oex.lnf_h = h;
      oex.lnf_ldh = m.ldk_h;
    }
    if (skip_wo) {
    } else if (dg) {
      run_dgemm(o, po, nullptr, nullptr, oex, st);
      ++launches;
    } else {
      run_gemm(o, st, oex);
      ++launches;
    }
    // ffn_norm (model.py:484-486)
    LnArgs ln{};
    ln.n_rows = M;
    ln.H = H;
    ln.x = x;
    ln.ldx = m.ldk_h;
    ln.src_stride = 1;
    ln.src_off = 0;
    ln.g = w.ln2_gamma;
    ln.b = w.ln2_beta;
    ln.h = h;
    ln.ldh = m.ldk_h;
    if (!fuse_ln && !dg && !coop && !rowln && !skip_wo && !o_tail) {
      run_ln(ln, st, pdl);
      ++launches;
    }
    // FFN1 + GELU (model.py:488-490)
    tf_gemm_desc f1 = g;
    if (fuse_ln) set_ln(f1, w.ln2_gamma, w.ln2_beta, 1, 0);
    f1.n_feat = F;
    f1.k = H;
    f1.act = h;
    f1.lda = m.ldk_h;
    f1.wt = w.w1_t;
    f1.ldw = m.ldk_h;
    f1.epilogue = TF_EPI_BIAS_GELU;
    f1.bias = w.b1;
    f1.out = sd.ffn;
    f1.ldo = m.ldk_f;
    if (fs && force_splits[2]) f1.splits = force_splits[2];
    if (dg) {
      f1.act = x;  // ffn_norm (model.py:484-486) inside the GEMM
      run_dgemm(f1, p1, w.ln2_gamma, w.ln2_beta, pf_next(l, 2), st);
    } else {
      GemmExtra f1ex = pf_next(l, 2);
      if (pdl && T == 1 && (late_mask & 2)) f1.pdl = 2;
      if (coop) {
        set_ln(f1, w.ln2_gamma, w.ln2_beta, 1, 0);
        f1ex.ln_coop = 1;
      }
      run_gemm(f1, st, f1ex);
    }
    ++launches;
    // FFN2 + residual (model.py:491-494)
    tf_gemm_desc f2 = g;
    f2.n_feat = H;
    f2.k = F;
    f2.act = sd.ffn;
    f2.lda = m.ldk_f;
    f2.wt = w.w2_t;
    f2.ldw = m.ldk_f;
    f2.epilogue = TF_EPI_BIAS_RESID;
    f2.bias = w.b2;
    f2.out = x;
    f2.ldo = m.ldk_h;
    f2.resid = x;
    f2.ldr = m.ldk_h;
    if (fs && force_splits[3]) f2.splits = force_splits[3];
    // next layer's attn_norm, or final_norm (model.py:460-462, 497-498)
    LnArgs nl = ln;
    if (l + 1 < L) {
      nl.g = s.m->layers[l + 1].ln1_gamma;
      nl.b = s.m->layers[l + 1].ln1_beta;
    } else {
      nl.g = m.final_gamma;
      nl.b = m.final_beta;
      if (mode != TF_FWD_LOGITS_ALL) {  // only the last position feeds the lm_head
        nl.n_rows = B;
        nl.src_stride = T;
        nl.src_off = T - 1;
      }
    }
    GemmExtra f2ex = pf_next(l, 3);
    if (rowln) {  // T == 1: every row is the last position
      f2.splits = 2;
      f2ex.row_ln = 1;
      f2ex.lnf_g = nl.g;
      f2ex.lnf_b = nl.b;
      f2ex.lnf_h = h;
      f2ex.lnf_ldh = m.ldk_h;
    }
    if (pdl && T == 1 && (late_mask & 4)) f2.pdl = 2;
    const bool f2_tail = ln_cnt && push_plan(f2);
    if (f2_tail) {  // T == 1: every row is the last position
      f2ex.lnf_cnt = ln_cnt;
      f2ex.lnf_g = nl.g;
      f2ex.lnf_b = nl.b;
      f2ex.lnf_h = h;
      f2ex.lnf_ldh = m.ldk_h;
    }
    if (dg)
      run_dgemm(f2, p2, nullptr, nullptr, f2ex, st);
    else
      run_gemm(f2, st, f2ex);
    ++launches;
    if (rowln || f2_tail) continue;
    if ((dg || coop) && l + 1 < L) continue;  // the next QKV normalises its own operand
    if (l + 1 < L ? !fuse_ln : !fuse_final) {
      run_ln(nl, st, pdl);
      ++launches;
    }
  }
  // lm_head (+ argmax) (model.py:500-504, 594, 652)
  tf_gemm_desc lg = g;
  if (fuse_final) {
    if (mode == TF_FWD_LOGITS_ALL)
      set_ln(lg, m.final_gamma, m.final_beta, 1, 0);
    else
      set_ln(lg, m.final_gamma, m.final_beta, T, T - 1);
  }
  lg.m_tok = (mode == TF_FWD_LOGITS_ALL) ? M : B;
  lg.n_feat = m.vocab;
  lg.k = H;
  lg.act = h;
  lg.lda = m.ldk_h;
  lg.wt = m.lm_head_t;
  lg.ldw = m.ldk_h;
  lg.epilogue = TF_EPI_LOGITS;
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
  return launches;
}

// ---------------------------------------------------------------- megakernel
long long* g_mk_trace = nullptr;  // tf_debug_set_trace (diagnostics only)

bool mk_enabled() {  // opt-in until it beats the graph path (TF_MEGAKERNEL=1)
  const char* e = getenv("TF_MEGAKERNEL");
  return e && e[0] == '1';
}

bool mk_eligible(const Session& s) {
  const tf_model_desc& m = s.m->d;
  return m.head_dim == 64 && m.hidden % 128 == 0 && m.ffn % m.hidden == 0 && m.layers <= mk::kMaxLayers &&
         m.hidden <= 1024 && s.d.batch <= 128 && s.d.beam_indir == nullptr && s.d.out_tokens &&
         mk::smem_bytes(4, 3, ((s.d.batch + 15) / 16) * 16, s.d.capacity, 16) <= kMaxSmem;
}

void mk_prepare(Session& s) {
  MkState& k = s.mk;
  if (k.ready) return;
  const tf_model_desc& m = s.m->d;
  const int L = m.layers, H = m.hidden, F = m.ffn, NH = m.heads, V = m.vocab, B = s.d.batch;
  const int bn = ((B + 15) / 16) * 16;
  const int nth = H / 128, nff = F / 128, nqkv = 3 * H / 128, nsplit = F / H, lmt = (V + 127) / 128;
  int dev = 0;
  TF_CHECK_CUDA(cudaGetDevice(&dev));
  int sms = 0;
  TF_CHECK_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  k.bn = bn;
  k.grid = sms;
  // smem: weight ring, activation ring, then as many attention K slots as fit
  k.ws = 6;
  k.bs = 4;
  auto slots_for = [&](int ws, int bs) {
    const long left = (long)kMaxSmem - (long)mk::smem_bytes(ws, bs, bn, s.d.capacity, 0);
    return (int)std::max(0L, left / (4 * 128));
  };
  if (slots_for(k.ws, k.bs) < 64) k.ws = 4;
  k.att_slots = std::min(slots_for(k.ws, k.bs), s.d.capacity);
  // ---- static plan: GEMM items and aux tasks in one topological order,
  // dealt to CTAs so every CTA's list is a subsequence of that order
  std::vector<std::vector<int4>> gi(k.grid), ai(k.grid);
  std::vector<long> load(k.grid, 0);
  int next_g = 0;
  auto put_gemm = [&](int type, int layer, int tile, int split) {
    // all items stream the same bytes; deal round-robin (least loaded == next)
    gi[next_g].push_back(make_int4(type, layer, tile, split));
    load[next_g] += 1;
    next_g = (next_g + 1) % k.grid;
  };
  int rr = 0;
  auto put_aux = [&](int type, int layer, int b, int h) {
    ai[rr % k.grid].push_back(make_int4(type, layer, b, h));
    ++rr;
  };
  for (int b = 0; b < B; ++b) put_aux(mk::A_EMB, 0, b, 0);
  for (int l = 0; l < L; ++l) {
    for (int t = 0; t < nqkv; ++t) put_gemm(mk::G_QKV, l, t, 0);
    for (int id = 0; id < NH * B; id += 4) put_aux(mk::A_ATT, l, id, std::min(4, NH * B - id));
    for (int t = 0; t < nth; ++t) put_gemm(mk::G_WO, l, t, 0);
    for (int b = 0; b < B; ++b) put_aux(mk::A_R2, l, b, 0);
    for (int t = 0; t < nff; ++t) put_gemm(mk::G_W1, l, t, 0);
    for (int c = 0; c < nsplit; ++c)
      for (int t = 0; t < nth; ++t) put_gemm(mk::G_W2, l, t, c);
    for (int b = 0; b < B; ++b) put_aux(mk::A_R1, l, b, 0);
  }
  for (int t = 0; t < lmt; ++t) put_gemm(mk::G_LM, 0, t, 0);
  std::vector<int4> items, aux;
  std::vector<int> ioff(k.grid + 1, 0), aoff(k.grid + 1, 0);
  for (int c = 0; c < k.grid; ++c) {
    ioff[c] = (int)items.size();
    items.insert(items.end(), gi[c].begin(), gi[c].end());
    aoff[c] = (int)aux.size();
    aux.insert(aux.end(), ai[c].begin(), ai[c].end());
  }
  ioff[k.grid] = (int)items.size();
  aoff[k.grid] = (int)aux.size();
  // ---- one device allocation for everything
  const int ldx = m.ldk_h, ldf = m.ldk_f;
  k.n_ctr = mk::ctr_count(L, nqkv, NH, nff);
  const size_t act = (size_t)bn * ldx * sizeof(__half);
  size_t off = 0;
  auto take = [&](size_t n) {
    size_t o = off;
    off += (n + 255) / 256 * 256;
    return o;
  };
  const size_t o_x = take(act), o_h1 = take(act), o_h2 = take(act), o_at = take(act), o_hf = take(act);
  const size_t o_q = take(act), o_f = take((size_t)bn * ldf * sizeof(__half));
  const size_t o_pw2 = take((size_t)nth * bn * nsplit * 128 * sizeof(float));
  const size_t o_ctr = take(sizeof(int) * k.n_ctr);
  const size_t o_it = take(sizeof(int4) * items.size()), o_io = take(sizeof(int) * ioff.size());
  const size_t o_ax = take(sizeof(int4) * aux.size()), o_ao = take(sizeof(int) * aoff.size());
  const size_t o_ly = take(sizeof(mk::Layer) * L);
  TF_CHECK_CUDA(cudaMalloc(&k.mem, off));
  TF_CHECK_CUDA(cudaMemset(k.mem, 0, off));
  uint8_t* base = static_cast<uint8_t*>(k.mem);
  k.x = reinterpret_cast<__half*>(base + o_x);
  k.h1 = reinterpret_cast<__half*>(base + o_h1);
  k.h2 = reinterpret_cast<__half*>(base + o_h2);
  k.attn = reinterpret_cast<__half*>(base + o_at);
  k.hf = reinterpret_cast<__half*>(base + o_hf);
  k.q = reinterpret_cast<__half*>(base + o_q);
  k.f = reinterpret_cast<__half*>(base + o_f);
  k.p_w2 = reinterpret_cast<float*>(base + o_pw2);
  k.ctr = reinterpret_cast<int*>(base + o_ctr);
  k.items = reinterpret_cast<int4*>(base + o_it);
  k.item_off = reinterpret_cast<int*>(base + o_io);
  k.aux = reinterpret_cast<int4*>(base + o_ax);
  k.aux_off = reinterpret_cast<int*>(base + o_ao);
  k.layers = reinterpret_cast<mk::Layer*>(base + o_ly);
  std::vector<mk::Layer> ly(L);
  for (int l = 0; l < L; ++l) {
    const tf_layer_weights& w = s.m->layers[l];
    ly[l] = mk::Layer{w.ln1_gamma, w.ln1_beta, w.bqkv, w.bo, w.ln2_gamma, w.ln2_beta, w.b1, w.b2};
  }
  TF_CHECK_CUDA(cudaMemcpy(k.items, items.data(), sizeof(int4) * items.size(), cudaMemcpyHostToDevice));
  TF_CHECK_CUDA(cudaMemcpy(k.item_off, ioff.data(), sizeof(int) * ioff.size(), cudaMemcpyHostToDevice));
  TF_CHECK_CUDA(cudaMemcpy(k.aux, aux.data(), sizeof(int4) * aux.size(), cudaMemcpyHostToDevice));
  TF_CHECK_CUDA(cudaMemcpy(k.aux_off, aoff.data(), sizeof(int) * aoff.size(), cudaMemcpyHostToDevice));
  TF_CHECK_CUDA(cudaMemcpy(k.layers, ly.data(), sizeof(mk::Layer) * L, cudaMemcpyHostToDevice));
  // ---- tensor maps
  for (int l = 0; l < L; ++l) {
    const tf_layer_weights& w = s.m->layers[l];
    k.maps.w[4 * l + 0] = make_kmajor_map(w.wqkv_t, 3 * H, H, m.ldk_h, 128);
    k.maps.w[4 * l + 1] = make_kmajor_map(w.wo_t, H, H, m.ldk_h, 128);
    k.maps.w[4 * l + 2] = make_kmajor_map(w.w1_t, F, H, m.ldk_h, 128);
    k.maps.w[4 * l + 3] = make_kmajor_map(w.w2_t, H, F, m.ldk_f, 128);
  }
  k.maps.w[4 * L] = make_kmajor_map(m.lm_head_t, V, H, m.ldk_h, 128);
  k.maps.act[0] = make_kmajor_map(k.h1, bn, H, ldx, bn);
  k.maps.act[1] = make_kmajor_map(k.attn, bn, H, ldx, bn);
  k.maps.act[2] = make_kmajor_map(k.h2, bn, H, ldx, bn);
  k.maps.act[3] = make_kmajor_map(k.f, bn, F, ldf, bn);
  k.maps.act[4] = make_kmajor_map(k.hf, bn, H, ldx, bn);
  TF_CHECK_CUDA(cudaFuncSetAttribute(mk::decode_megakernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)kMaxSmem));
  k.ready = true;
}

int mk_decode(Session& s, int n_steps, cudaStream_t st) {
  mk_prepare(s);
  MkState& k = s.mk;
  const tf_model_desc& m = s.m->d;
  mk::Params p{};
  p.L = m.layers;
  p.H = m.hidden;
  p.F = m.ffn;
  p.NH = m.heads;
  p.V = m.vocab;
  p.B = s.d.batch;
  p.bn = k.bn;
  p.cap = s.d.capacity;
  p.n_steps = n_steps;
  p.ws = k.ws;
  p.bs = k.bs;
  p.nkb = m.hidden / 64;
  p.nth = m.hidden / 128;
  p.nqkv = 3 * m.hidden / 128;
  p.nff = m.ffn / 128;
  p.nsplit = m.ffn / m.hidden;
  p.lm_tiles = (m.vocab + 127) / 128;
  p.att_slots = k.att_slots;
  p.layers = k.layers;
  p.fin_g = m.final_gamma;
  p.fin_b = m.final_beta;
  p.tok_emb = static_cast<const __half*>(m.tok_emb);
  p.pos_emb = static_cast<const __half*>(m.pos_emb);
  p.ldw = m.ldw;
  p.x = k.x;
  p.h1 = k.h1;
  p.h2 = k.h2;
  p.attn = k.attn;
  p.hf = k.hf;
  p.q = k.q;
  p.f = k.f;
  p.ldx = m.ldk_h;
  p.ldf = m.ldk_f;
  p.p_w2 = k.p_w2;
  p.kc = static_cast<__half*>(s.d.k_cache);
  p.vc = static_cast<__half*>(s.d.v_cache);
  p.pads = s.d.pads;
  p.len_dev = s.d.len_dev;
  p.step_dev = s.d.step_dev;
  p.keys = s.d.keys;
  p.out_tokens = s.d.out_tokens;
  p.max_new = s.d.max_new;
  p.ctr = k.ctr;
  p.items = k.items;
  p.item_off = k.item_off;
  p.aux = k.aux;
  p.aux_off = k.aux_off;
  p.scale = 0.125f;
  p.trace = g_mk_trace;
  p.trace_step = 1;
  const char* fl = getenv("TF_MK_FLAGS");
  p.flags = fl ? atoi(fl) : 1;
  TF_CHECK_CUDA(cudaMemsetAsync(k.ctr, 0, sizeof(int) * k.n_ctr, st));
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(k.grid);
  cfg.blockDim = dim3(mk::kThreads);
  cfg.dynamicSmemBytes = mk::smem_bytes(k.ws, k.bs, k.bn, s.d.capacity, k.att_slots);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // all CTAs co-resident (spin-waits are safe)
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  TF_CHECK_CUDA(cudaLaunchKernelEx(&cfg, mk::decode_megakernel, k.maps, p));
  return 2;  // memset + kernel
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
  return a;
}

template <int KB>
void launch_select(const BeamArgs& a, size_t smem, cudaStream_t st, bool pdl) {
  static bool attr = false;
  if (!attr) {
    TF_CHECK_CUDA(cudaFuncSetAttribute(beam_select_kernel<KB>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kMaxSmem - 8192));
    attr = true;
  }
  launch(beam_select_kernel<KB>, dim3(a.R), dim3(kSelThreads), smem, st, pdl, a);
}

void run_beam_select(const Session& s, const tf_beam_desc& d, cudaStream_t st, bool pdl) {
  const BeamArgs a = beam_args(s, d);
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
    if (batch > 0 && seq_len > 0) run_attention(a, static_cast<cudaStream_t>(stream), false);
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
    *session = s;
  });
}

int tf_session_destroy(void* session) {
  return guarded([&] {
    Session* s = static_cast<Session*>(session);
    if (s && s->graph) cudaGraphExecDestroy(s->graph);
    if (s && s->graph_multi) cudaGraphExecDestroy(s->graph_multi);
    if (s && s->beam_graph) cudaGraphExecDestroy(s->beam_graph);
    if (s && s->mk.mem) cudaFree(s->mk.mem);
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

int tf_decode(void* session, int n_steps, int use_graph, void* stream) {
  return guarded([&] {
    TF_REQUIRE(session, TF_ERR_ARG, "decode: null session");
    Session& s = *static_cast<Session*>(session);
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (n_steps <= 0) return;
    if (use_graph && mk_enabled() && mk_eligible(s)) {
      mk_decode(s, n_steps, st);
      s.launches_last = 1;  // one persistent kernel for all n steps
      return;
    }
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

int tf_debug_mk_trace(void* session, void* trace_buf, int* n_items, int* n_aux, void* plan_out) {
  return guarded([&] {
    TF_REQUIRE(session, TF_ERR_ARG, "trace: null session");
    Session& s = *static_cast<Session*>(session);
    g_mk_trace = static_cast<long long*>(trace_buf);
    if (s.mk.ready && n_items && n_aux) {
      int off[2];
      TF_CHECK_CUDA(cudaMemcpy(off, s.mk.item_off + s.mk.grid, sizeof(int), cudaMemcpyDeviceToHost));
      TF_CHECK_CUDA(cudaMemcpy(off + 1, s.mk.aux_off + s.mk.grid, sizeof(int), cudaMemcpyDeviceToHost));
      *n_items = off[0];
      *n_aux = off[1];
      if (plan_out) {
        TF_CHECK_CUDA(cudaMemcpy(plan_out, s.mk.items, sizeof(int4) * off[0], cudaMemcpyDeviceToHost));
        TF_CHECK_CUDA(cudaMemcpy(static_cast<int4*>(plan_out) + off[0], s.mk.aux, sizeof(int4) * off[1],
                                 cudaMemcpyDeviceToHost));
      }
    }
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
