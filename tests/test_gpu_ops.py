"""Kernel-level numerics on the GPU: every CUDA operator against a plain PyTorch
fp32 reference of the same op (f16 inputs, f32 math)."""

import math

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2407_04991_b200 import _native as N  # noqa: E402
from paper_2407_04991_b200 import ops  # noqa: E402


def rand16(*shape, scale=1.0, seed=0):
    g = torch.Generator().manual_seed(seed)
    return (torch.randn(*shape, generator=g) * scale).half()


def q16(x):
    return x.clamp(-65504, 65504).half().float()


def gelu_ref(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x * x * x)))


@pytest.mark.parametrize("m,n,k,swap,splits", [
    (128, 256, 64, 0, 1), (256, 512, 768, 0, 1), (300, 200, 200, 0, 1),
    (4096, 768, 768, 0, 1), (32, 2304, 768, 1, 0), (32, 768, 3072, 1, 0),
    (7, 100, 70, 1, 1), (128, 1000, 256, 1, 4), (256, 768, 768, 1, 0), (16, 64, 32, 1, 1),
    (512, 2304, 768, 0, 1), (4096, 3072, 768, 0, 1), (300, 1100, 192, 0, 1),  # bn = 256 tiles
])
def test_gemm_f32_matches_torch(cuda_device, m, n, k, swap, splits):
    kp = ops.pad64(k)
    a = torch.zeros(m, kp, dtype=torch.half)
    a[:, :k] = rand16(m, k, seed=1)
    w = torch.zeros(n, kp, dtype=torch.half)
    w[:, :k] = rand16(n, k, scale=0.05, seed=2)
    a, w = a.to(cuda_device), w.to(cuda_device)
    out = torch.full((m, n), float("nan"), dtype=torch.float32, device=cuda_device)
    scr = ops.Scratch(cuda_device, 64 << 20)
    ops.gemm(a, w, k, N.EPI_F32, out=out, scratch=scr, force_swap=swap, splits=splits)
    torch.cuda.synchronize()
    ref = a.float()[:, :k] @ w.float()[:, :k].T
    err = (out - ref).abs().max().item()
    assert err <= 1e-3 * max(1.0, ref.abs().max().item()), err
    assert int(scr.counters.abs().sum().item()) == 0  # split-K counters self-reset


@pytest.mark.parametrize("swap,m,n", [(0, 64, 384), (1, 64, 384), (0, 300, 640), (0, 4096, 2304)])
def test_gemm_epilogues(cuda_device, swap, m, n):
    """Bias / GELU / residual epilogues; (0, 300, 640) and (0, 4096, 2304) run the
    2-CTA prefill kernel (odd 128-row tile count, partial 256-feature tile)."""
    k = 256
    a = rand16(m, k, seed=3).to(cuda_device)
    w = rand16(n, k, scale=0.05, seed=4).to(cuda_device)
    bias = (torch.randn(n) * 0.1).half().float().to(cuda_device)
    resid = rand16(m, n, seed=5).to(cuda_device)
    acc = a.float() @ w.float().T
    scr = ops.Scratch(cuda_device, 16 << 20)
    out = torch.empty(m, n, dtype=torch.half, device=cuda_device)
    ops.gemm(a, w, k, N.EPI_BIAS, out=out, bias=bias, scratch=scr, force_swap=swap)
    assert (out.float() - q16(acc + bias)).abs().max().item() <= 2e-3
    ops.gemm(a, w, k, N.EPI_BIAS_GELU, out=out, bias=bias, scratch=scr, force_swap=swap)
    assert (out.float() - q16(gelu_ref(acc + bias))).abs().max().item() <= 2e-3
    x = resid.clone()
    ops.gemm(a, w, k, N.EPI_BIAS_RESID, out=x, resid=x, bias=bias, scratch=scr, force_swap=swap)
    assert (x.float() - q16(resid.float() + q16(acc + bias))).abs().max().item() <= 4e-3
    torch.cuda.synchronize()


@pytest.mark.parametrize("swap", [0, 1])
def test_gemm_logits_argmax_lowest_id_ties(cuda_device, swap):
    m, n, k = 16, 1000, 64
    a = rand16(m, k, seed=6).to(cuda_device)
    w = rand16(n, k, scale=0.05, seed=7)
    w[500] = w[3]  # duplicated column -> exact tie, lowest id must win
    w[900] = w[3]
    w = w.to(cuda_device)
    keys = torch.zeros(m, dtype=torch.int64, device=cuda_device)
    logits = torch.empty(m, n, dtype=torch.half, device=cuda_device)
    scr = ops.Scratch(cuda_device, 16 << 20)
    ops.gemm(a, w, k, N.EPI_LOGITS, out=logits, keys=keys, scratch=scr, force_swap=swap)
    torch.cuda.synchronize()
    ids = (0xFFFFFFFF - (keys & 0xFFFFFFFF)).cpu().numpy()
    want = np.argmax(logits.float().cpu().numpy(), axis=1)  # first max = lowest id
    assert (ids == want).all()
    ref = q16(a.float() @ w.float().T)
    assert (logits.float() - ref).abs().max().item() <= 2e-3


def test_layernorm(cuda_device):
    rows, H = 37, 768
    x = rand16(rows, H, seed=8).to(cuda_device)
    g = (1 + 0.05 * torch.randn(H)).half().float().to(cuda_device)
    b = (0.05 * torch.randn(H)).half().float().to(cuda_device)
    h = torch.empty_like(x)
    ops.layernorm(x, H, g, b, h)
    torch.cuda.synchronize()
    xf = x.float()
    mean = xf.mean(-1, keepdim=True)
    c = xf - mean
    var = (c * c).mean(-1, keepdim=True)
    ref = q16(c * (1.0 / torch.sqrt(var + 1e-5)) * g + b)
    assert (h.float() - ref).abs().max().item() <= 4e-3


def _attn_ref(q, kc, vc, start, qbase, T, scale):
    B, NH, cap, D = kc.shape
    out = torch.zeros(B, T, NH, D)
    for b in range(B):
        for t in range(T):
            lo, hi = int(start[b]), qbase + t
            if hi < lo:
                continue
            qq = q[b * T + t].float().view(NH, D)
            k = kc[b, :, lo:hi + 1].float()
            v = vc[b, :, lo:hi + 1].float()
            s = torch.einsum("hd,hsd->hs", qq, k) * scale
            w = torch.softmax(s, dim=-1)
            out[b, t] = torch.einsum("hs,hsd->hd", w, v)
    return q16(out.reshape(B * T, NH * D))


@pytest.mark.parametrize("T,D,qbase", [(1, 64, 40), (1, 16, 5), (1, 4, 3), (16, 64, 0), (37, 64, 0),
                                       (5, 32, 7), (130, 64, 0), (128, 64, 0), (200, 64, 60), (300, 64, 0),
                                       (1, 64, 700)])
def test_attention(cuda_device, T, D, qbase):
    """T > 1 with D = 64 runs the tcgen05 prefill kernel (S, O in TMEM); T = 1
    with a capacity > 256 the tensor-core unit kernel (one beam per request)."""
    B, NH, cap = 3, 2, max(192, qbase + T + 8)
    H = NH * D
    q = rand16(B * T, H, seed=9).to(cuda_device)
    kc = rand16(B, NH, cap, D, seed=10).to(cuda_device)
    vc = rand16(B, NH, cap, D, seed=11).to(cuda_device)
    start = torch.tensor([0, 3, min(qbase + T + 2, 20)], dtype=torch.int32)
    qb = torch.tensor([qbase], dtype=torch.int32, device=cuda_device)
    out = torch.full((B * T, H), float("nan"), dtype=torch.half, device=cuda_device)
    scale = 1.0 / math.sqrt(D)
    ops.attention(q, None, kc, vc, start.to(cuda_device), qb, scale, out, batch=B, heads=NH,
                  head_dim=D, cap=cap, seq_len=T)
    torch.cuda.synchronize()
    ref = _attn_ref(q.cpu(), kc.cpu(), vc.cpu(), start, qbase, T, scale)
    assert (out.float().cpu() - ref).abs().max().item() <= 4e-3


@pytest.mark.parametrize("B,NH,cap,qbase", [(64, 12, 192, 150), (128, 12, 256, 255), (8, 4, 192, 100),
                                             (8, 4, 320, 300)])
def test_decode_attention_per_row_kernels(cuda_device, B, NH, cap, qbase):
    """T = 1, D = 64 through the operator runs the generation path's decode
    kernels: capacities <= 256 the tensor-core per-row kernel (whatever the
    grid: one wave at (8, 4, 192), several at (64, 12, 192)), capacity 320 the
    unit kernel; windows start at per-row left pads."""
    D = 64
    H = NH * D
    q = rand16(B, H, seed=21).to(cuda_device)
    kc = rand16(B, NH, cap, D, seed=22).to(cuda_device)
    vc = rand16(B, NH, cap, D, seed=23).to(cuda_device)
    start = torch.randint(0, qbase // 2, (B,), generator=torch.Generator().manual_seed(5), dtype=torch.int32)
    start[0] = 0
    qb = torch.tensor([qbase], dtype=torch.int32, device=cuda_device)
    out = torch.full((B, H), float("nan"), dtype=torch.half, device=cuda_device)
    scale = 1.0 / math.sqrt(D)
    ops.attention(q, None, kc, vc, start.to(cuda_device), qb, scale, out, batch=B, heads=NH,
                  head_dim=D, cap=cap, seq_len=1)
    torch.cuda.synchronize()
    ref = _attn_ref(q.cpu(), kc.cpu(), vc.cpu(), start, qbase, 1, scale)
    assert (out.float().cpu() - ref).abs().max().item() <= 4e-3


def test_decode_attention_capacity_invariant(cuda_device):
    """A row's decode attention output does not depend on the capacity of the
    cache it sits in (which the batch's longest prompt sets): the same windows
    placed in caches of 192 ... 1024 slots give bitwise equal outputs within
    each kernel class, and the per-row (<= 256 slots) and unit (> 256 slots)
    kernels are reported against each other."""
    B, NH, D, qbase = 16, 12, 64, 180
    H = NH * D
    q = rand16(B, H, seed=31).to(cuda_device)
    k0 = rand16(B, NH, 192, D, seed=32)
    v0 = rand16(B, NH, 192, D, seed=33)
    start = torch.randint(0, 150, (B,), generator=torch.Generator().manual_seed(6), dtype=torch.int32).to(cuda_device)
    qb = torch.tensor([qbase], dtype=torch.int32, device=cuda_device)
    outs = {}
    for cap in (192, 256, 320, 448, 1024):
        kc = torch.zeros(B, NH, cap, D, dtype=torch.half)
        vc = torch.zeros(B, NH, cap, D, dtype=torch.half)
        kc[:, :, :192], vc[:, :, :192] = k0, v0
        out = torch.empty(B, H, dtype=torch.half, device=cuda_device)
        ops.attention(q, None, kc.to(cuda_device), vc.to(cuda_device), start, qb, 0.125, out, batch=B, heads=NH,
                      head_dim=D, cap=cap, seq_len=1)
        torch.cuda.synchronize()
        outs[cap] = out.cpu()
    assert torch.equal(outs[192], outs[256])
    assert torch.equal(outs[320], outs[448]) and torch.equal(outs[320], outs[1024])
    diff = (outs[192].float() - outs[320].float()).abs().max().item()
    print(f"per-row vs unit kernel max-abs {diff:.3e}, bitwise {torch.equal(outs[192], outs[320])}")
    assert diff <= 2e-3


def test_embed_gather_sum_bit_exact_and_remap(cuda_device):
    V, P, H, n = 50, 20, 96, 13
    tok = rand16(V, H, seed=12, scale=0.05)
    pos = rand16(P, H, seed=13, scale=0.05)
    ids = torch.randint(0, 40, (n,), dtype=torch.int32)
    ps = torch.randint(0, P, (n,), dtype=torch.int32)
    remap = torch.full((40,), -1, dtype=torch.int32)
    remap[::2] = torch.arange(20, dtype=torch.int32)
    dev = cuda_device
    x = torch.empty(n, H, dtype=torch.half, device=dev)
    used = torch.empty(n, dtype=torch.int32, device=dev)
    ops.embed_ln(ids.to(dev), ps.to(dev), tok.to(dev), pos.to(dev), H, x, remap=remap.to(dev),
                 unk_id=0, ids_out=used)
    torch.cuda.synchronize()
    want_ids = torch.where(remap[ids.long()] >= 0, remap[ids.long()], torch.zeros_like(ids))
    assert torch.equal(used.cpu(), want_ids)
    ref = (tok[want_ids.long()].float() + pos[ps.long()].float()).clamp(-65504, 65504).half()
    assert torch.equal(x.cpu(), ref)  # bit-exact gather-sum


@pytest.mark.parametrize("m,n,h", [(32, 2304, 768), (5, 200, 256), (64, 3072, 768), (100, 640, 384),
                                   (256, 2304, 768), (16, 384, 200)])
def test_fused_layernorm_statistics(cuda_device, m, n, h):
    """The decode LayerNorm fusion (tensor.py:153-160 restated over tiles): a
    residual GEMM (swap-AB split-K) writes per-128-feature (mean, M2) pairs of
    its output rows; a consuming GEMM with gamma folded into its weights applies
    inv * (x . W' - mean * c) + d. The pairs match numpy (fp64) per tile; the
    consumer matches LN(x) . W in fp64 within 5e-3 (the folded weights are
    f16-rounded and the LN output is not)."""
    kin = 256
    tiles = (h + 127) // 128
    a = rand16(m, kin, seed=30).to(cuda_device)
    wo = rand16(h, kin, scale=0.05, seed=31).to(cuda_device)
    bo = (0.1 * torch.randn(h, generator=torch.Generator().manual_seed(3))).half().float().to(cuda_device)
    hp = ops.pad64(h)
    x = torch.zeros(m, hp, dtype=torch.half)
    x[:, :h] = rand16(m, h, seed=32)
    x = x.to(cuda_device)
    stats = torch.full((2 * tiles * m,), float("nan"), dtype=torch.float32, device=cuda_device)
    ops.gemm(a, wo, kin, N.EPI_BIAS_RESID, out=x, bias=bo, resid=x, force_swap=1, stats=(stats, m))
    torch.cuda.synchronize()
    xs = x[:, :h].double().cpu().numpy()
    got = stats.view(tiles, m, 2).double().cpu().numpy()
    for i in range(tiles):
        seg = xs[:, 128 * i:min(h, 128 * i + 128)]
        mu = seg.mean(axis=1)
        m2 = ((seg - mu[:, None]) ** 2).sum(axis=1)
        assert np.allclose(got[i, :, 0], mu, rtol=1e-5, atol=1e-6)
        assert np.allclose(got[i, :, 1], m2, rtol=1e-4, atol=1e-5)
    from test_gpu_pack import host_fold as _fold_ln
    g = (1 + 0.05 * torch.randn(h, generator=torch.Generator().manual_seed(4))).half().float()
    b = (0.05 * torch.randn(h, generator=torch.Generator().manual_seed(5))).half().float()
    w = rand16(n, hp, scale=0.05, seed=33)
    wf, c, dd = _fold_ln(w.numpy(), h, g.numpy(), b.numpy())
    wf, c, dd = (torch.from_numpy(v).to(cuda_device) for v in (wf, c, dd))
    out = torch.full((m, n), float("nan"), dtype=torch.float32, device=cuda_device)
    ops.gemm(x, wf, h, N.EPI_F32, out=out, force_swap=1, ln=(stats, m, h, c, dd))
    torch.cuda.synchronize()
    xd = x[:, :h].double().cpu()
    mu = xd.mean(dim=1, keepdim=True)
    var = ((xd - mu) ** 2).mean(dim=1, keepdim=True)
    ln = (xd - mu) / torch.sqrt(var + 1e-5) * g.double() + b.double()
    ref = (ln @ w[:, :h].double().T).float().to(cuda_device)
    assert (out - ref).abs().max().item() <= 5e-3
