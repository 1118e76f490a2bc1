"""ctypes binding of ``libtinfer_sm100.so`` (include/tinfer_sm100.h).

The shared library is built in-tree by ``build.py`` (nvcc, sm_100a). There is no
CPU fallback: if the library or a CUDA device is missing, :func:`lib` raises
:class:`~.errors.DeviceError`. ctypes releases the GIL for the duration of each
call, preserving the reference kernels' ``nogil=True`` threading contract.
"""

from __future__ import annotations

import ctypes as C
import os

from .errors import DeviceError, raise_for_status

LIB_NAME = "libtinfer_sm100.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

c_int_p = C.POINTER(C.c_int)
c_float_p = C.POINTER(C.c_float)


class GemmDesc(C.Structure):
    _fields_ = [
        ("m_tok", C.c_int), ("n_feat", C.c_int), ("k", C.c_int),
        ("act", C.c_void_p), ("lda", C.c_int),
        ("wt", C.c_void_p), ("ldw", C.c_int),
        ("epilogue", C.c_int),
        ("bias", C.c_void_p),
        ("out", C.c_void_p), ("ldo", C.c_int),
        ("resid", C.c_void_p), ("ldr", C.c_int),
        ("q_out", C.c_void_p), ("ldq", C.c_int),
        ("k_cache", C.c_void_p), ("v_cache", C.c_void_p),
        ("hidden", C.c_int), ("heads", C.c_int), ("head_dim", C.c_int), ("cap", C.c_int),
        ("seq_len", C.c_int),
        ("qbase_dev", C.c_void_p),
        ("argmax_keys", C.c_void_p),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("counters", C.c_void_p), ("n_counters", C.c_int),
        ("force_swap", C.c_int), ("splits", C.c_int), ("pdl", C.c_int),
        ("ln_stats", C.c_void_p), ("ln_stats_ld", C.c_int), ("ln_hidden", C.c_int),
        ("ln_c", C.c_void_p), ("ln_d", C.c_void_p),
        ("stats_out", C.c_void_p), ("stats_ld", C.c_int),
    ]


class EmbedDesc(C.Structure):
    _fields_ = [
        ("n_tok", C.c_int), ("hidden", C.c_int), ("vocab", C.c_int), ("max_pos", C.c_int),
        ("ids", C.c_void_p), ("pos", C.c_void_p), ("type_ids", C.c_void_p), ("type_const", C.c_int),
        ("remap", C.c_void_p), ("remap_n", C.c_int), ("unk_id", C.c_int),
        ("tok_emb", C.c_void_p), ("pos_emb", C.c_void_p), ("type_emb", C.c_void_p),
        ("ldw", C.c_int),
        ("ln_gamma", C.c_void_p), ("ln_beta", C.c_void_p),
        ("x", C.c_void_p), ("h", C.c_void_p), ("ldx", C.c_int),
        ("ids_out", C.c_void_p),
    ]


class LayerWeights(C.Structure):
    _fields_ = [
        ("ln1_gamma", C.c_void_p), ("ln1_beta", C.c_void_p),
        ("wqkv_t", C.c_void_p), ("bqkv", C.c_void_p),
        ("wo_t", C.c_void_p), ("bo", C.c_void_p),
        ("ln2_gamma", C.c_void_p), ("ln2_beta", C.c_void_p),
        ("w1_t", C.c_void_p), ("b1", C.c_void_p),
        ("w2_t", C.c_void_p), ("b2", C.c_void_p),
        ("wqkv_ln_t", C.c_void_p), ("cqkv", C.c_void_p), ("dqkv", C.c_void_p),
        ("w1_ln_t", C.c_void_p), ("c1", C.c_void_p), ("d1", C.c_void_p),
    ]


class ModelDesc(C.Structure):
    _fields_ = [
        ("vocab", C.c_int), ("hidden", C.c_int), ("layers", C.c_int), ("heads", C.c_int),
        ("head_dim", C.c_int), ("ffn", C.c_int), ("max_pos", C.c_int),
        ("ldk_h", C.c_int), ("ldk_f", C.c_int),
        ("tok_emb", C.c_void_p), ("pos_emb", C.c_void_p), ("type_emb", C.c_void_p),
        ("n_types", C.c_int), ("ldw", C.c_int),
        ("layer", C.POINTER(LayerWeights)),
        ("final_gamma", C.c_void_p), ("final_beta", C.c_void_p),
        ("lm_head_t", C.c_void_p),
        ("lm_head_ln_t", C.c_void_p), ("c_lm", C.c_void_p), ("d_lm", C.c_void_p),
    ]


class SessionDesc(C.Structure):
    _fields_ = [
        ("batch", C.c_int), ("capacity", C.c_int), ("max_tokens", C.c_int), ("max_new", C.c_int),
        ("k_cache", C.c_void_p), ("v_cache", C.c_void_p),
        ("x", C.c_void_p), ("h", C.c_void_p), ("q", C.c_void_p), ("attn", C.c_void_p),
        ("ffn", C.c_void_p), ("logits", C.c_void_p),
        ("workspace", C.c_void_p), ("workspace_bytes", C.c_size_t),
        ("counters", C.c_void_p), ("n_counters", C.c_int),
        ("keys", C.c_void_p), ("len_dev", C.c_void_p), ("step_dev", C.c_void_p),
        ("out_tokens", C.c_void_p), ("pads", C.c_void_p),
        ("remap", C.c_void_p), ("remap_n", C.c_int), ("unk_id", C.c_int),
        ("beam_indir", C.c_void_p), ("beam", C.c_int),
        ("ln_stats", C.c_void_p), ("ln_stats_bytes", C.c_size_t),
        ("type_ids", C.c_void_p), ("gen_type", C.c_int),
    ]


class BeamDesc(C.Structure):
    _fields_ = [
        ("requests", C.c_int), ("beam", C.c_int), ("max_new", C.c_int), ("prompt_len", C.c_int),
        ("eos", C.c_int),
        ("scores", C.c_void_p), ("finished", C.c_void_p), ("tokens", C.c_void_p),
        ("tok_hist", C.c_void_p), ("par_hist", C.c_void_p),
    ]


# exported symbol -> (restype, argtypes); the single source for the CPU-side
# "library loads and exports every declared symbol" test
SIGNATURES = {
    "tf_abi_version": (C.c_int, []),
    "tf_last_error": (C.c_char_p, []),
    "tf_device_info": (C.c_int, [c_int_p, c_int_p, c_int_p]),
    "tf_gemm": (C.c_int, [C.POINTER(GemmDesc), C.c_void_p]),
    "tf_embed_ln": (C.c_int, [C.POINTER(EmbedDesc), C.c_void_p]),
    "tf_layernorm": (C.c_int, [C.c_int, C.c_int, C.c_void_p, C.c_int, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]),
    "tf_attention": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float,
                               C.c_void_p, C.c_int, C.c_void_p]),
    "tf_model_create": (C.c_int, [C.POINTER(ModelDesc), C.POINTER(C.c_void_p)]),
    "tf_model_destroy": (C.c_int, [C.c_void_p]),
    "tf_session_create": (C.c_int, [C.c_void_p, C.POINTER(SessionDesc), C.POINTER(C.c_void_p)]),
    "tf_session_destroy": (C.c_int, [C.c_void_p]),
    "tf_forward": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                             C.c_void_p]),
    "tf_forward_taps": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                  C.c_void_p]),
    "tf_decode": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p]),
    "tf_beam_select": (C.c_int, [C.c_void_p, C.POINTER(BeamDesc), C.c_void_p]),
    "tf_beam_decode": (C.c_int, [C.c_void_p, C.POINTER(BeamDesc), C.c_int, C.c_int, C.c_void_p]),
    "tf_debug_trace": (C.c_int, [C.c_int, C.c_void_p, C.c_int, C.c_void_p]),
    "tf_session_launches_per_step": (C.c_int, [C.c_void_p]),
    "tf_attention_beam": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                    C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_float,
                                    C.c_void_p, C.c_int, C.c_void_p]),
    "tf_pack_kmajor": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_int,
                                 C.c_void_p]),
    "tf_fold_terms": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_void_p,
                                C.c_void_p, C.c_void_p]),
    "tf_convert": (C.c_int, [C.c_void_p, C.c_int, C.c_longlong, C.c_void_p, C.c_int, C.c_void_p]),
}

ABI_VERSION = 2

# tf_epilogue / tf_forward_mode (include/tinfer_sm100.h)
EPI_F32, EPI_BIAS, EPI_BIAS_GELU, EPI_BIAS_RESID, EPI_QKV, EPI_LOGITS = range(6)
FWD_ARGMAX, FWD_LOGITS_LAST, FWD_LOGITS_ALL = range(3)

_lib = None


def load_library(path: str = LIB_PATH) -> C.CDLL:
    """dlopen the library and bind every declared symbol (no GPU needed)."""
    if not os.path.exists(path):
        raise DeviceError(f"{LIB_NAME} not built (expected at {path}); run build.py")
    handle = C.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    if handle.tf_abi_version() != ABI_VERSION:
        raise DeviceError("libtinfer_sm100 ABI version mismatch")
    return handle


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        _lib = load_library()
    return _lib


def check(status: int, what: str) -> None:
    if status != 0:
        detail = lib().tf_last_error().decode("utf-8", "replace")
        raise_for_status(status, what, detail)
