"""Probe: does one batch split into S row groups, each generated on its own host
thread / CUDA stream, finish sooner than the whole batch on one stream?

    python tools/split_probe.py [c2|c3] [reps]

Prints the median wall time of the public batched_greedy_decode for S = 1, 2, 4
(outputs are checked equal to the S = 1 result: batch invariance holds for <= 128 rows).
"""

import os
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2407_04991_b200 as P  # noqa: E402


def main():
    wname = sys.argv[1] if len(sys.argv) > 1 else "c2"
    reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
    w = bench.WORKLOADS[wname]
    model = bench.build_model(w)
    prompts = bench.make_prompts(model.config.vocab_size, w, 0)
    model.device_model(torch.device("cuda", 0))
    ref = P.batched_greedy_decode(model, prompts, w["new"])

    def run_split(S):
        n = (len(prompts) + S - 1) // S
        groups = [prompts[i * n:(i + 1) * n] for i in range(S)]
        out = [None] * S
        streams = [torch.cuda.Stream() for _ in range(S)]

        def work(i):
            with torch.cuda.stream(streams[i]):
                out[i] = P.batched_greedy_decode(model, groups[i], w["new"])

        ts = [threading.Thread(target=work, args=(i,)) for i in range(S)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        return [r for o in out for r in o]

    for S in (1, 2, 4):
        for _ in range(3):
            got = run_split(S)
        assert got == ref, f"S={S}: tokens differ"
        times = []
        for _ in range(reps):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            run_split(S)
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        ms = float(np.median(times)) * 1e3
        toks = len(prompts) * w["new"]
        print(f"{wname} S={S}: {ms:.2f} ms per generate, {toks / ms * 1e3:.0f} tok/s", flush=True)


if __name__ == "__main__":
    main()
