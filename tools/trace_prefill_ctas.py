"""Per-CTA phase times of the prefill GEMMs of one forward (TF_TRACE=1):
for each of the first layer's GEMM launches, the distribution over CTAs of
(MMA done - start) and (exit - MMA done), and the launch span."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("TF_TRACE", "1")

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2407_04991_b200 import _native as N  # noqa: E402


def main():
    w = bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    model = bench.build_model(w)
    run = bench.Runner(model, bench.make_prompts(model.config.vocab_size, w, 0), w)
    lib = N.lib()
    for _ in range(2):
        run.stage()
        run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
    torch.cuda.synchronize()
    run.stage()
    lib.tf_debug_trace(1, None, 0, None)
    run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
    torch.cuda.synchronize()
    raw = np.zeros((256, 2048, 8), dtype=np.uint64)
    names = (C.c_char_p * 256)()
    n = lib.tf_debug_trace(0, raw.ctypes.data, 256, names)
    for i in range(min(n, 9)):
        nm = names[i].decode()
        r = raw[i].astype(np.float64)
        ok = r[:, 0] > 0
        r = r[ok]
        if not len(r):
            continue
        t0 = r[:, 0].min()
        span = (r[:, 7].max() - t0) / 1e3
        if "gemm" in nm:
            main_ = (r[:, 2] - r[:, 0]) / 1e3
            epi = (r[:, 7] - r[:, 2]) / 1e3
            start = (r[:, 0] - t0) / 1e3
            print(f"{nm:<16} ctas {len(r):4d} span {span:7.1f} us | start p50 {np.median(start):6.1f} max {start.max():6.1f}"
                  f" | mainloop p50 {np.median(main_):5.1f} max {main_.max():5.1f} | epilogue p50 {np.median(epi):5.1f}"
                  f" max {epi.max():5.1f}")
        else:
            print(f"{nm:<16} ctas {len(r):4d} span {span:7.1f} us")


if __name__ == "__main__":
    main()
