"""Per-kernel timeline of one decode step (diagnostics; needs TF_TRACE=1).

Runs a workload's prefill, warms the decode path, then launches ONE decode step
without a graph (same kernels, same PDL chaining) with trace slots enabled and
prints, per kernel, each trace point's latest CTA time relative to the previous
kernel's last exit (the critical-path view). GEMM points: 1 past the PDL wait,
2 MMA done, 3 partial tile parked, 4 past the cluster barrier, 5 first unit
reduced, 6 stores issued, 7 exit. Usage: TF_TRACE=1 python tools/trace_step.py [workload] [rows]"""

import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TF_TRACE", "1")

import warnings  # noqa: E402

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402

NP = 16


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "c2"
    nrows = int(sys.argv[2]) if len(sys.argv) > 2 else 14
    w = bench.WORKLOADS[wname]
    model = bench.build_model(w)
    prompts = bench.make_prompts(model.config.vocab_size, w, 0)
    run = bench.Runner(model, prompts, w)
    lib = N.lib()
    run.stage()
    if run.beam:  # beam: prefill + select + warm steps; each traced step = T=1 forward + select
        br, s = run.beam, run.sess
        st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
        s.forward(br.L, N.FWD_LOGITS_LAST)
        N.check(lib.tf_beam_select(s.handle, C.byref(br.desc), st), "tf_beam_select")
        N.check(lib.tf_beam_decode(s.handle, C.byref(br.desc), 8, 0, st), "tf_beam_decode")

        def one():
            N.check(lib.tf_beam_decode(s.handle, C.byref(br.desc), 1, 0, st), "tf_beam_decode")
    else:
        run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
        run.sess.decode(8, use_graph=False)

        def one():
            run.sess.decode(1, use_graph=False)
    torch.cuda.synchronize()
    reps = int(os.environ.get("TRACE_REPS", "10"))
    agg = {}
    step_us = []
    for rep in range(reps):
        lib.tf_debug_trace(1, None, 0, None)
        one()
        torch.cuda.synchronize()
        raw = np.zeros((256, 2048, 8), dtype=np.uint64)
        names = (C.c_char_p * 256)()
        n = lib.tf_debug_trace(0, raw.ctypes.data, 256, names)
        r = raw[:n].astype(np.float64)
        r[r == 0] = np.nan
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            mx = np.nanmax(r[:, :, 7], axis=1)
            mn0 = np.nanmin(r[:, :, 0], axis=1)
        for i in range(n):
            prev = mx[i - 1] if i > 0 else mn0[0]
            agg.setdefault(names[i].decode(), []).append((mx[i] - prev) / 1e3)
        step_us.append((mx[n - 1] - mn0[0]) / 1e3)
    print(f"mean over {reps} traced steps: step {np.mean(step_us):.1f} us (median {np.median(step_us):.1f})")
    for k, v in agg.items():
        print(f"  {k:<18} mean incr {np.nanmean(v):6.2f} us  x{len(v) // reps:3d}/step = {np.nansum(v) / reps:7.1f} us")
    r = raw[:n].astype(np.float64)
    r[r == 0] = np.nan
    if os.environ.get("PER_CTA"):  # per-CTA phase durations of the attention launches
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            for i in range(n):
                if not names[i].decode().startswith("attn_decode"):
                    continue
                c = r[i]
                c = c[~np.isnan(c[:, 0])]
                ph = lambda x, y: np.nanmedian(c[:, y] - c[:, x]) / 1e3  # noqa: E731
                life = (c[:, 7] - c[:, 0]) / 1e3
                print(f"attn #{i}: ctas traced {len(c)} span {(np.nanmax(c[:, 7]) - np.nanmin(c[:, 0])) / 1e3:.1f} us; "
                      f"median life {np.nanmedian(life):.2f} (p90 {np.nanpercentile(life, 90):.2f}); "
                      f"0-1 {ph(0, 1):.2f} 1-2 {ph(1, 2):.2f} 2-4 {ph(2, 4):.2f} 4-5 {ph(4, 5):.2f} 5-7 {ph(5, 7):.2f}; "
                      f"QK cycles median {np.nanmedian(c[:, 6]):.0f}; 0-6 {ph(0, 6):.2f} 1-3 {ph(1, 3):.2f} 3-2 {ph(3, 2):.2f}")
                st = np.sort(c[:, 0])
                print(f"   entry times rel: p10 {(st[len(st) // 10] - st[0]) / 1e3:.1f} p50 {(st[len(st) // 2] - st[0]) / 1e3:.1f} "
                      f"p90 {(st[9 * len(st) // 10] - st[0]) / 1e3:.1f} us")
                break
    t = np.full((n, NP), np.nan)
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        t[:, :8] = np.nanmax(r, axis=1)
        t[:, 8:] = np.nanmin(r, axis=1)
    nm = [names[i].decode() for i in range(n)]
    base = np.nanmin(t[:, 8])
    print(f"{'#':>3} {'kernel':<18} {'entry':>7} " + " ".join(f"{'p' + str(i):>6}" for i in range(0, 8)) + f" {'incr':>6}")
    prev = None
    tot = {}
    for i in range(n):
        ref = prev if prev is not None else t[i, 8]
        rel = [(t[i, k] - ref) / 1e3 for k in range(0, 8)]
        incr = (t[i, 7] - ref) / 1e3
        if i < nrows:
            print(f"{i:3d} {nm[i]:<18} {(t[i, 8] - base) / 1e3:7.2f} " + " ".join(f"{v:6.2f}" for v in rel)
                  + f" {incr:6.2f}")
            mins = [(t[i, 8 + k] - ref) / 1e3 for k in range(0, 8)]
            print(f"{'':3} {'  (min over CTAs)':<18} {'':7} " + " ".join(f"{v:6.2f}" for v in mins))
        tot.setdefault(nm[i], []).append(incr)
        if nm[i] == "attn_decode_pf" and i < nrows:
            print(f"      scores: SM cycles max {t[i, 6]:.0f} min {t[i, 14]:.0f}; globaltimer p2->p4 "
                  f"{(t[i, 4] - t[i, 2]) / 1e3:.2f} us (max)")
        prev = t[i, 7]
    print("\ncritical-path increment (exit_i - exit_{i-1}) per kernel type, us:")
    for k, v in tot.items():
        print(f"  {k:<18} n={len(v):3d} mean {np.nanmean(v):6.2f} total {np.nansum(v):7.1f}")
    print(f"step (first entry -> last exit): {(t[-1, 7] - base) / 1e3:.1f} us (traced kernels only)")


if __name__ == "__main__":
    main()
