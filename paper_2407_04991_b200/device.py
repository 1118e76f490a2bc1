"""Device mirror of a host ``Model`` and per-batch generation sessions.

``DeviceModel`` packs the reference weights (``[in, out]`` row-major, reference
model.py:190-207) into the layout the sm_100a kernels stream:

* every projection as f16 ``W^T [out, pad64(in)]`` (K-major, zero-padded K) so
  TMA can fetch 64-wide K slabs with a 128-byte swizzle;
* Q, K and V fused into one ``[3H, pad64(H)]`` matrix (one GEMM, K/V written
  straight into the cache by the epilogue);
* LayerNorm parameters and biases as f32 (they hold f16-representable values
  for F16 models, and the epilogues add them in f32 like the reference);
* the untied lm_head transposed to ``[V, pad64(H)]``.

F32 models are rounded to f16 on upload (saturating RNE, tensor.py:95-100): the
device path always stores f16 and accumulates in f32.

``Session`` owns one batch's KV cache ``[L, B, NH, cap, D]`` (reference layout,
model.py:316-317) and activation scratch, plus the native ``tf_session`` whose
decode step is captured into a CUDA graph on first use and replayed.
"""

from __future__ import annotations

import ctypes as C
import threading

import numpy as np
import torch

from . import _native as N
from . import workspace
from .ops import pad64
from .tensor import round_to, DType


def _raw(t) -> np.ndarray:
    """The stored array of a ``Tensor`` (or an array), C-contiguous, F32 or F16."""
    a = t.array if hasattr(t, "array") else t
    if a.dtype not in (np.float32, np.float16):
        a = a.astype(np.float32)
    return np.ascontiguousarray(a)


class DeviceModel:
    """Packed, device-resident weights + the native ``tf_model`` handle.

    Packing runs on the device (csrc/pack.cuh through tf_pack_kmajor /
    tf_fold_terms / tf_convert): each reference tensor is uploaded as stored and
    transposed / rounded / LayerNorm-folded in HBM. ``source`` (optional) maps
    tensor names to arrays to read instead of ``model``'s — the TINF
    direct-to-device loader passes memory-mapped file slices."""

    def __init__(self, model, device: torch.device, source: dict | None = None):
        c = model.config
        self.config = c
        self.device = device
        self.H, self.F, self.V = c.hidden_size, c.ffn_size, c.vocab_size
        self.L, self.NH, self.D, self.P = c.num_layers, c.num_heads, c.head_dim, c.max_position
        self.ldk_h, self.ldk_f = pad64(self.H), pad64(self.F)
        # re-entrant: session() takes it too, so a session can never be evicted
        # (and closed) while another thread holding the lock uses it
        self.lock = threading.RLock()
        arrays = dict(model.named_tensors()) if source is None else source
        raw = lambda name: _raw(arrays[name])  # noqa: E731  (reference layout, F32 or F16)
        self._keep = []
        st = C.c_void_p(torch.cuda.current_stream(device).cuda_stream)

        def keep(t):
            self._keep.append(t)
            return t

        def upload(a: np.ndarray) -> torch.Tensor:
            """Raw tensor -> HBM as stored (one H2D copy; from a memory-mapped
            TINF file the bytes go page cache -> device)."""
            return torch.from_numpy(a).to(device)

        def vec(name, as_f32=True):  # q16 values, f32 (biases / LN params) or f16
            a = raw(name)
            src = upload(a)
            out = torch.empty(a.shape, dtype=torch.float32 if as_f32 else torch.float16, device=device)
            N.check(N.lib().tf_convert(C.c_void_p(src.data_ptr()), int(a.dtype == np.float32), a.size,
                                       C.c_void_p(out.data_ptr()), int(as_f32), st), "tf_convert")
            return out

        def pack(names, ldk, gamma=None, out=None):
            """[in, out] tensors stacked along out -> f16 W^T [sum(out), ldk]."""
            n_tot = sum(arrays[n].shape[1] for n in names)
            dst = out if out is not None else torch.empty((n_tot, ldk), dtype=torch.float16, device=device)
            row = 0
            for n in names:
                a = raw(n)
                k, nn = a.shape
                src = upload(a)
                N.check(N.lib().tf_pack_kmajor(C.c_void_p(src.data_ptr()), int(a.dtype == np.float32), k, nn,
                                               None if gamma is None else C.c_void_p(gamma.data_ptr()),
                                               C.c_void_p(dst[row:].data_ptr()), ldk, st), "tf_pack_kmajor")
                row += nn
            return dst

        def fold(names, ldk, gamma, beta, w_t):
            """LayerNorm folded into the projection (decode path, gemm_tc.cuh
            ln_fold): W' = q16(W * gamma), c = sum_k W', d = sum_k beta_k W."""
            w_ln = pack(names, ldk, gamma=gamma)
            n = w_ln.shape[0]
            c_ = torch.empty(n, dtype=torch.float32, device=device)
            d_ = torch.empty(n, dtype=torch.float32, device=device)
            N.check(N.lib().tf_fold_terms(C.c_void_p(w_t.data_ptr()), C.c_void_p(w_ln.data_ptr()),
                                          C.c_void_p(beta.data_ptr()), self.H, n, ldk, C.c_void_p(c_.data_ptr()),
                                          C.c_void_p(d_.data_ptr()), st), "tf_fold_terms")
            return w_ln, c_, d_

        self.tok_emb = keep(vec("token_embedding", as_f32=False))
        self.type_emb = None
        if model.type_embedding is not None:  # extension: word + position + type gather-sum
            te = model.type_embedding.array
            self.type_emb = keep(torch.from_numpy(round_to(te.astype(np.float32), DType.F16)).to(device))
        self.pos_emb = keep(vec("position_embedding", as_f32=False))
        layers = (N.LayerWeights * self.L)()
        self.layers = []
        for i in range(self.L):
            p = f"layers.{i}."
            g1, be1 = vec(p + "attn_norm.gamma"), vec(p + "attn_norm.beta")
            g2, be2 = vec(p + "ffn_norm.gamma"), vec(p + "ffn_norm.beta")
            qkv = [p + "attn.wq", p + "attn.wk", p + "attn.wv"]
            wqkv_t = pack(qkv, self.ldk_h)
            w1_t = pack([p + "ffn.w1"], self.ldk_h)
            wqkv_ln, cqkv, dqkv = fold(qkv, self.ldk_h, g1, be1, wqkv_t)
            w1_ln, c1, d1 = fold([p + "ffn.w1"], self.ldk_h, g2, be2, w1_t)
            lw = dict(
                ln1_gamma=g1, ln1_beta=be1,
                wqkv_t=wqkv_t, bqkv=torch.cat([vec(p + "attn.bq"), vec(p + "attn.bk"), vec(p + "attn.bv")]),
                wo_t=pack([p + "attn.wo"], self.ldk_h), bo=vec(p + "attn.bo"),
                ln2_gamma=g2, ln2_beta=be2,
                w1_t=w1_t, b1=vec(p + "ffn.b1"),
                w2_t=pack([p + "ffn.w2"], self.ldk_f), b2=vec(p + "ffn.b2"),
                wqkv_ln_t=wqkv_ln, cqkv=cqkv, dqkv=dqkv,
                w1_ln_t=w1_ln, c1=c1, d1=d1,
            )
            self.layers.append(lw)
            for k, t in lw.items():
                setattr(layers[i], k, t.data_ptr())
        self.final_gamma = keep(vec("final_norm.gamma"))
        self.final_beta = keep(vec("final_norm.beta"))
        self.lm_head_t = keep(pack(["lm_head"], self.ldk_h))
        lm_ln, c_lm, d_lm = fold(["lm_head"], self.ldk_h, self.final_gamma, self.final_beta, self.lm_head_t)
        self.lm_head_ln_t, self.c_lm, self.d_lm = keep(lm_ln), keep(c_lm), keep(d_lm)
        torch.cuda.current_stream(device).synchronize()  # staging copies may be released
        self._layer_structs = layers
        d = N.ModelDesc()
        d.vocab, d.hidden, d.layers, d.heads = self.V, self.H, self.L, self.NH
        d.head_dim, d.ffn, d.max_pos = self.D, self.F, self.P
        d.ldk_h, d.ldk_f = self.ldk_h, self.ldk_f
        d.tok_emb, d.pos_emb = self.tok_emb.data_ptr(), self.pos_emb.data_ptr()
        if self.type_emb is not None:
            d.type_emb, d.n_types = self.type_emb.data_ptr(), self.type_emb.shape[0]
        d.ldw = self.tok_emb.stride(0)
        d.layer = layers
        d.final_gamma, d.final_beta = self.final_gamma.data_ptr(), self.final_beta.data_ptr()
        d.lm_head_t = self.lm_head_t.data_ptr()
        d.lm_head_ln_t, d.c_lm, d.d_lm = self.lm_head_ln_t.data_ptr(), self.c_lm.data_ptr(), self.d_lm.data_ptr()
        h = C.c_void_p()
        N.check(N.lib().tf_model_create(C.byref(d), C.byref(h)), "tf_model_create")
        self.handle = h
        # reserved C-ABI scratch fields (split-K reduces through DSMEM; kept tiny)
        self.ws_bytes = 1 << 12
        self.ws = torch.empty(self.ws_bytes // 4, dtype=torch.float32, device=device)
        self.n_counters = 16
        self.counters = torch.zeros(self.n_counters, dtype=torch.int32, device=device)
        self._sessions: dict[tuple, Session] = {}

    def weight_bytes(self) -> int:
        """Bytes of weights one decode step streams (all layers + lm_head)."""
        n = 0
        for lw in self.layers:
            for k in ("wqkv_t", "wo_t", "w1_t", "w2_t"):
                n += lw[k].numel() * 2
        return n + self.lm_head_t.numel() * 2

    def session(self, batch: int, capacity: int, max_tokens: int, max_new: int,
                logits=False, beam: int = 0) -> "Session":
        """The calling thread's session of this shape. Sessions are owned per host
        thread (its KV cache, scratch, step state and captured graphs), so
        inference workers sharing one GPU run concurrently on their own streams
        without touching each other's buffers; each thread keeps at most 16."""
        tid = threading.get_ident()
        key = (tid, batch, capacity, max_tokens, max_new, logits, beam)
        with self.lock:
            s = self._sessions.get(key)
            if s is None:
                mine = [k for k in self._sessions if k[0] == tid]
                if len(mine) >= 16:  # bound this thread's cache; drop its oldest
                    self._sessions.pop(mine[0]).close()
                s = Session(self, batch, capacity, max_tokens, max_new, logits, beam=beam)
                self._sessions[key] = s
            return s

    def close(self):
        for s in self._sessions.values():
            s.close()
        self._sessions.clear()
        if self.handle:
            N.lib().tf_model_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Session:
    """One batch shape: KV cache, activations, device step state, native handle."""

    def __init__(self, dm: DeviceModel, batch: int, capacity: int, max_tokens: int, max_new: int,
                 logits, k_cache: torch.Tensor | None = None,
                 v_cache: torch.Tensor | None = None, beam: int = 0):
        """``logits``: False (argmax only), "last" ([batch, V] buffer) or True/"all"
        ([batch*max_tokens, V]); ``beam`` > 0 adds the beam-search state."""
        dev = dm.device
        self.dm, self.batch, self.capacity = dm, batch, capacity
        self.max_tokens, self.max_new = max_tokens, max(1, max_new)
        rows = batch * max_tokens
        shape = (dm.L, batch, dm.NH, capacity, dm.D)
        self.k_cache = k_cache if k_cache is not None else torch.zeros(shape, dtype=torch.float16, device=dev)
        self.v_cache = v_cache if v_cache is not None else torch.zeros(shape, dtype=torch.float16, device=dev)
        z16 = lambda n, ld: torch.zeros((n, ld), dtype=torch.float16, device=dev)  # noqa: E731
        # activation buffers: one zeroed arena, lifetime-disjoint buffers share
        # storage (workspace.py: {ffn, q}, {h, attn}, {x})
        self.plan = workspace.session_plan(rows, dm.H, dm.F, dm.ldk_h, dm.ldk_f, dm.L)
        self.arena = torch.zeros(self.plan.arena_bytes(), dtype=torch.uint8, device=dev)
        offs = self.plan.offsets()
        for name, ld in (("x", dm.ldk_h), ("h", dm.ldk_h), ("q", dm.ldk_h), ("attn", dm.ldk_h), ("ffn", dm.ldk_f)):
            o = offs[self.plan.assignment[name]]
            setattr(self, name, self.arena[o:o + rows * ld * 2].view(torch.float16).view(rows, ld))
        logit_rows = batch if logits == "last" else rows
        self.logits = z16(logit_rows, dm.V) if logits else None
        self.keys = torch.zeros(batch, dtype=torch.int64, device=dev)
        # int32 state: [len, step] + pads[B] + ids[rows] + pos[rows] + types[rows]
        self.state = torch.zeros(2 + batch + 3 * rows, dtype=torch.int32, device=dev)
        self.len_dev, self.step_dev = self.state[0:1], self.state[1:2]
        self.pads = self.state[2:2 + batch]
        self.ids = self.state[2 + batch:2 + batch + rows]
        self.pos = self.state[2 + batch + rows:2 + batch + 2 * rows]
        self.types = self.state[2 + batch + 2 * rows:]
        self.out_tokens = torch.zeros((batch, self.max_new), dtype=torch.int32, device=dev)
        self.host_in = torch.zeros(self.state.numel(), dtype=torch.int32).pin_memory()
        self.host_out = torch.zeros((batch, self.max_new), dtype=torch.int32).pin_memory()
        self.remap = None
        self.beam = beam
        if beam:
            self.indir = torch.zeros((batch, capacity), dtype=torch.int32, device=dev)
            self.scores = torch.zeros(batch, dtype=torch.float32, device=dev)
            self.finished = torch.zeros(batch, dtype=torch.uint8, device=dev)
            self.beam_tokens = torch.zeros(batch, dtype=torch.int32, device=dev)
            self.tok_hist = torch.zeros((self.max_new, batch), dtype=torch.int32, device=dev)
            self.par_hist = torch.zeros((self.max_new, batch), dtype=torch.int32, device=dev)
        d = N.SessionDesc()
        d.batch, d.capacity, d.max_tokens, d.max_new = batch, capacity, max_tokens, self.max_new
        d.k_cache, d.v_cache = self.k_cache.data_ptr(), self.v_cache.data_ptr()
        d.x, d.h, d.q, d.attn = self.x.data_ptr(), self.h.data_ptr(), self.q.data_ptr(), self.attn.data_ptr()
        d.ffn = self.ffn.data_ptr()
        d.logits = self.logits.data_ptr() if logits else None
        # split-KV decode attention scratch: per (row, head, 64-slot chunk) {m, z, o[64]}
        # and one arrival counter per (row, head)
        chunks = (capacity + 63) // 64
        self.att_ws = torch.empty(max(1, batch * dm.NH * chunks * 66), dtype=torch.float32, device=dev)
        self.att_cnt = torch.zeros(batch * dm.NH, dtype=torch.int32, device=dev)
        d.workspace, d.workspace_bytes = self.att_ws.data_ptr(), self.att_ws.numel() * 4
        d.counters, d.n_counters = self.att_cnt.data_ptr(), self.att_cnt.numel()
        # row statistics of the residual stream for the LayerNorms fused into the
        # decode GEMMs: two [ceil(H/128), rows] arrays of (mean, M2) pairs
        tiles = (dm.H + 127) // 128
        self.ln_stats = torch.zeros(4 * tiles * rows, dtype=torch.float32, device=dev)
        d.ln_stats, d.ln_stats_bytes = self.ln_stats.data_ptr(), self.ln_stats.numel() * 4
        d.keys = self.keys.data_ptr()
        d.len_dev, d.step_dev = self.len_dev.data_ptr(), self.step_dev.data_ptr()
        d.out_tokens = self.out_tokens.data_ptr()
        d.pads = self.pads.data_ptr()
        d.remap, d.remap_n, d.unk_id = None, 0, 0
        if beam:
            d.beam_indir, d.beam = self.indir.data_ptr(), beam
        if dm.type_emb is not None:
            d.type_ids, d.gen_type = self.types.data_ptr(), 0
        self.desc = d
        h = C.c_void_p()
        N.check(N.lib().tf_session_create(dm.handle, C.byref(d), C.byref(h)), "tf_session_create")
        self.handle = h
        self.len = 0  # host mirror of the device cache length

    def set_remap(self, table):
        """Install (or clear, table=None) the prompt-id remap applied by the
        embedding kernel to prefill ids (int32 old id -> new id, -1 = dropped)."""
        import numpy as np
        if table is None:
            if self.remap is not None:
                self.desc.remap, self.desc.remap_n = None, 0
                self.remap = None
                self._push_desc()
            return
        t = torch.from_numpy(np.ascontiguousarray(table, dtype=np.int32)).to(self.k_cache.device)
        self.remap = t
        self.desc.remap, self.desc.remap_n, self.desc.unk_id = t.data_ptr(), t.numel(), 0
        self._push_desc()

    def set_gen_type(self, gen_type: int):
        """Type row of generated tokens (models with a type table)."""
        if self.dm.type_emb is not None and self.desc.gen_type != gen_type:
            self.desc.gen_type = gen_type
            self._push_desc()

    def _push_desc(self):
        """Re-create the native session with the updated descriptor (buffers kept)."""
        N.lib().tf_session_destroy(self.handle)
        h = C.c_void_p()
        N.check(N.lib().tf_session_create(self.dm.handle, C.byref(self.desc), C.byref(h)),
                "tf_session_create")
        self.handle = h

    # ------------------------------------------------------------------ steps
    @staticmethod
    def stream():
        return C.c_void_p(torch.cuda.current_stream().cuda_stream)

    def load_inputs(self, ids: np.ndarray, pos: np.ndarray, pads: np.ndarray, length: int = 0,
                    types: np.ndarray | None = None):
        """One H2D copy of [len, step, pads, ids, pos(, types)] from pinned memory."""
        B, rows, R = self.batch, ids.size, self.batch * self.max_tokens
        buf = self.host_in.numpy()
        buf[0], buf[1] = length, 0
        buf[2:2 + B] = pads
        buf[2 + B:2 + B + rows] = ids.reshape(-1)
        buf[2 + B + R:2 + B + R + rows] = pos.reshape(-1)
        n = 2 + B + R + rows
        if self.dm.type_emb is not None:
            buf[2 + B + 2 * R:2 + B + 2 * R + rows] = 0 if types is None else np.asarray(types).reshape(-1)
            n = 2 + B + 2 * R + rows
        self.state[:n].copy_(self.host_in[:n], non_blocking=True)
        self.keys.zero_()
        self.len = length
        return (2 + B + (3 if self.dm.type_emb is not None else 2) * rows) * 4

    def forward(self, T: int, mode: int, use_ids: bool = True, pdl: bool = True):
        ids = C.c_void_p(self.ids.data_ptr()) if use_ids else None
        pos = C.c_void_p(self.pos.data_ptr()) if use_ids else None
        N.check(N.lib().tf_forward(self.handle, ids, pos, T, mode, 1 if pdl else 0, self.stream()),
                "tf_forward")
        self.len += T
        return N.lib().tf_session_launches_per_step(self.handle)

    def forward_taps(self, T: int, mode: int) -> torch.Tensor:
        """forward() that also returns the residual stream at every LayerNorm
        input, f16 [2L+1, batch*T, H] (tf_forward_taps)."""
        dm = self.dm
        taps = torch.empty((2 * dm.L + 1, self.batch * T, dm.H), dtype=torch.float16, device=self.k_cache.device)
        N.check(N.lib().tf_forward_taps(self.handle, C.c_void_p(self.ids.data_ptr()), C.c_void_p(self.pos.data_ptr()),
                                        T, mode, C.c_void_p(taps.data_ptr()), self.stream()), "tf_forward_taps")
        self.len += T
        return taps

    def decode(self, n_steps: int, use_graph: bool = True) -> int:
        if n_steps <= 0:
            return 0
        N.check(N.lib().tf_decode(self.handle, n_steps, 1 if use_graph else 0, self.stream()),
                "tf_decode")
        self.len += n_steps
        return n_steps * N.lib().tf_session_launches_per_step(self.handle)

    def fetch_tokens(self, n: int) -> np.ndarray:
        self.host_out[:, :n].copy_(self.out_tokens[:, :n], non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return self.host_out[:, :n].numpy().copy()

    def close(self):
        if getattr(self, "handle", None):
            N.lib().tf_session_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
