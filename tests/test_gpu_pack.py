"""Device-side weight packing (csrc/pack.cuh) and TINF direct-to-device loading.

The packed buffers the kernels stream must be bit-identical to the host
restatement below (the previous host packer: transpose + saturating RNE to f16,
LayerNorm fold W' = q16(W * gamma), c = sum W', d = sum beta * W in f64), for F32
and F16 models; and a model loaded with ``load_model(path, device=...)`` (memory-
mapped file, raw upload, device packing) generates exactly what the host-loaded
model generates."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

import paper_2407_04991_b200 as P  # noqa: E402
from paper_2407_04991_b200.ops import pad64  # noqa: E402
from paper_2407_04991_b200.tensor import DType, round_to  # noqa: E402


def host_kmajor(w_in_out, ld):
    k, n = w_in_out.shape
    buf = np.zeros((n, ld), dtype=np.float16)
    buf[:, :k] = round_to(np.asarray(w_in_out, dtype=np.float32), DType.F16).T
    return buf


def host_vec(v):
    return round_to(np.asarray(v, dtype=np.float32), DType.F16).astype(np.float32)


def host_fold(w_t, k, gamma, beta):
    w = w_t[:, :k].astype(np.float32)
    wf = round_to(w * gamma[None, :k].astype(np.float32), DType.F16)
    buf = np.zeros_like(w_t)
    buf[:, :k] = wf
    c = wf.astype(np.float64).sum(axis=1).astype(np.float32)
    d = (w.astype(np.float64) @ beta[:k].astype(np.float64)).astype(np.float32)
    return buf, c, d


@pytest.mark.parametrize("dtype,H,F,NH", [(P.DType.F32, 96, 200, 3), (P.DType.F16, 128, 512, 2)])
def test_device_packing_bitwise_equals_host(cuda_device, dtype, H, F, NH):
    m = P.init_random(P.ModelConfig(300, H, 2, NH, H // NH, F, 40, dtype, 1, 2), 5)
    dm = m.device_model()
    f32 = {n: t.array.astype(np.float32) for n, t in m.named_tensors()}
    lh, lf = pad64(H), pad64(F)
    for i, lw in enumerate(dm.layers):
        p = f"layers.{i}."
        wqkv = np.concatenate([f32[p + "attn.wq"], f32[p + "attn.wk"], f32[p + "attn.wv"]], axis=1)
        wqkv_t = host_kmajor(wqkv, lh)
        assert np.array_equal(lw["wqkv_t"].cpu().numpy(), wqkv_t)
        assert np.array_equal(lw["wo_t"].cpu().numpy(), host_kmajor(f32[p + "attn.wo"], lh))
        w1_t = host_kmajor(f32[p + "ffn.w1"], lh)
        assert np.array_equal(lw["w1_t"].cpu().numpy(), w1_t)
        assert np.array_equal(lw["w2_t"].cpu().numpy(), host_kmajor(f32[p + "ffn.w2"], lf))
        g1, b1 = host_vec(f32[p + "attn_norm.gamma"]), host_vec(f32[p + "attn_norm.beta"])
        assert np.array_equal(lw["ln1_gamma"].cpu().numpy(), g1)
        bq = np.concatenate([f32[p + "attn.bq"], f32[p + "attn.bk"], f32[p + "attn.bv"]])
        assert np.array_equal(lw["bqkv"].cpu().numpy(), host_vec(bq))
        for key, wt, g, b in (("wqkv_ln_t", wqkv_t, g1, b1),
                              ("w1_ln_t", w1_t, host_vec(f32[p + "ffn_norm.gamma"]),
                               host_vec(f32[p + "ffn_norm.beta"]))):
            buf, c, d = host_fold(wt, H, g, b)
            pre = "q" if key.startswith("wqkv") else "1"
            assert np.array_equal(lw[key].cpu().numpy(), buf)
            assert np.array_equal(lw[f"c{'qkv' if pre == 'q' else '1'}"].cpu().numpy(), c)
            assert np.array_equal(lw[f"d{'qkv' if pre == 'q' else '1'}"].cpu().numpy(), d)
    lm_t = host_kmajor(f32["lm_head"], lh)
    assert np.array_equal(dm.lm_head_t.cpu().numpy(), lm_t)
    buf, c, d = host_fold(lm_t, H, host_vec(f32["final_norm.gamma"]), host_vec(f32["final_norm.beta"]))
    assert np.array_equal(dm.lm_head_ln_t.cpu().numpy(), buf)
    assert np.array_equal(dm.c_lm.cpu().numpy(), c) and np.array_equal(dm.d_lm.cpu().numpy(), d)
    assert np.array_equal(dm.tok_emb.cpu().numpy(), round_to(f32["token_embedding"], DType.F16))


def test_tinf_direct_to_device(cuda_device, tmp_path):
    m = P.init_random(P.ModelConfig(2048, 256, 2, 4, 64, 1024, 256, P.DType.F16, 1, 2), 9)
    P.save_model(m, str(tmp_path / "m.tinf"))
    direct = P.load_model(str(tmp_path / "m.tinf"), device="cuda:0")
    host = P.load_model(str(tmp_path / "m.tinf"))
    prompts = [[5, 9, 11, 20, 7] * 6, [3, 4] * 10, list(range(40, 70))]
    assert P.batched_greedy_decode(direct, prompts, 16) == P.batched_greedy_decode(host, prompts, 16)
    dd, dh = direct.device_model(), host.device_model()
    assert dd is not dh
    for a, b in zip(dd.layers, dh.layers):
        assert all(bool((a[k] == b[k]).all()) for k in a)
    # the returned model's host tensors are the file's bytes
    for (na, ta), (nb, tb) in zip(direct.named_tensors(), host.named_tensors()):
        assert na == nb and np.array_equal(ta.array, tb.array)
