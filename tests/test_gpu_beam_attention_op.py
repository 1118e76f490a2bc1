"""Beam-search decode attention as an operator (tf_attention_beam) against a
torch fp32 reference: rows gathered through the cache indirection table, the
window shared by the beams of a request, f16 output within 4e-3. Cases mix
fully shared prompt chunks, partially shared ancestry, per-beam tails, ragged
left pads and windows up to 8 chunks; both kernels (TF_ATTN_BEAM=1, the
tensor-core beam-grouped default, and 0, the per-row kernel reading through
the indirection table) run in their own processes."""

import math
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CASE = r'''
import math, sys, torch
sys.path.insert(0, ROOT)
from paper_2407_04991_b200 import ops
torch.manual_seed(0)
dev = torch.device("cuda:0")
fails = []
for (req, R, hi, starts, share) in CASES:
    NH, D, cap = 3, 64, 1024 if hi >= 512 else 512
    rows = req * R
    q = (torch.randn(rows, NH * D) * 0.5).half()
    kc = (torch.randn(rows, NH, cap, D) * 0.5).half()
    vc = torch.randn(rows, NH, cap, D).half()
    start = torch.tensor([starts[r // R] for r in range(rows)], dtype=torch.int32)
    indir = torch.zeros(rows, cap, dtype=torch.int32)
    g = torch.Generator().manual_seed(hi)
    for b in range(rows):
        r = b % R
        for s in range(cap):
            # slots < share: beam 0's row for everyone (shared prompt); later: a
            # random ancestor, the newest slot: the row itself
            indir[b, s] = 0 if s < share else (r if s >= hi else int(torch.randint(0, R, (1,), generator=g)))
    out = torch.full((rows, NH * D), float("nan"), dtype=torch.half, device=dev)
    qb = torch.tensor([hi], dtype=torch.int32, device=dev)
    ops.attention_beam(q.to(dev), kc.to(dev), vc.to(dev), start.to(dev), qb, indir.to(dev), 1.0 / math.sqrt(D),
                       out, requests=req, beam=R, heads=NH, head_dim=D, cap=cap)
    torch.cuda.synchronize()
    ref = torch.zeros(rows, NH * D)
    for b in range(rows):
        lo = int(start[b])
        if hi < lo:
            continue
        base = (b // R) * R
        src = [base + int(indir[b, s]) for s in range(lo, hi + 1)]
        k = torch.stack([kc[src[i], :, lo + i].float() for i in range(len(src))], dim=1)  # [NH, n, D]
        v = torch.stack([vc[src[i], :, lo + i].float() for i in range(len(src))], dim=1)
        qq = q[b].float().view(NH, D)
        w = torch.softmax(torch.einsum("hd,hsd->hs", qq, k) / math.sqrt(D), dim=-1)
        ref[b] = torch.einsum("hs,hsd->hd", w, v).reshape(-1)
    err = (out.float().cpu() - ref.half().float()).abs().max().item()
    if not err <= 4e-3:
        fails.append((req, R, hi, err))
print("FAILS", fails)
assert not fails
'''

CASES = [(3, 4, 300, [0, 5, 40], 256), (2, 3, 140, [0, 17], 130), (1, 8, 460, [3], 400), (4, 2, 66, [0, 1, 2, 64], 64),
         (2, 4, 200, [0, 0], 0), (2, 4, 511, [0, 100], 448), (2, 2, 900, [0, 37], 700), (1, 4, 1000, [9], 512)]


@pytest.mark.parametrize("mode", ["1", "0"])
def test_beam_attention_operator(cuda_device, mode):
    code = f"ROOT = {ROOT!r}\nCASES = {CASES!r}\n" + CASE
    env = dict(os.environ, TF_ATTN_BEAM=mode)
    r = subprocess.run([sys.executable, "-c", code], cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
