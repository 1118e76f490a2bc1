"""Benchmark: generated tokens/s for Ernie-base fp16 generation on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c2]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1, one rank per GPU)

Workloads (BASELINE.json configs, SURVEY §8 pins; all weights random-init with
the reference's splitmix64 stream, seed 42, from the 12L/768h/12-head/FFN-3072
vocab-40000 master model):

* c2 (default, configs[1]): positions trimmed 1024 -> 512, fp16 greedy, batch 32
  per GPU, src 128, 64 new tokens. One step = one batched_greedy_decode call
  (1 prefill + 63 decode forwards, 2048 generated tokens per GPU).
* c3 (configs[2]): vocab pruned 40k -> 10k (build_pruned_vocab on a synthetic
  Zipf count vector, specials forced), positions 256, greedy, batch 128.
* c4 (configs[3]): the pruned model (512 positions), beam 4, 64 requests, src
  256, 128 new tokens; tokens counted = returned hypotheses (64 x 128).
* c5 (configs[4]): the pruned model (1024 positions), 20k requests with src
  ~ U[32, 512], 64 new, length-bucketed (batch <= 256, bucket 16); one step = the
  whole sweep; under torchrun each rank takes its LPT share (strong scaling).

Multi-GPU for c2/c3/c4 is data parallel over independent requests (each rank its
own batch, no collective): "scaling": "weak".

* ``value``  — device-resident throughput: inputs staged in HBM before the timed
  region; CUDA events on the launching stream around each step; L2 flushed
  between steps (outside the events); max over ranks.
* ``e2e``    — the same metric through the public API (batched_greedy_decode /
  beam_search_decode) with host prompt lists: H2D of ids/positions/pads and D2H
  of results inside the timed region (wall clock + device sync), max over ranks.
* ``roofline`` — the decode step, the unit of the north-star target (DESIGN.md
  §5): SURVEY §8d algorithmic bytes per step / the CUDA-event time of a
  graph-replayed step, against MEASURED_PEAKS.json; ``traffic`` = ncu DRAM bytes
  of one step (profiles/r1_ncu_step_<w>.json). ``largest_launch``: the lm_head
  GEMM + argmax alone (rotating weight copies, HBM-streamed).
* ``cpu_baseline`` — the reference's own CPU path (unmodified tinfer model +
  numba kernels, staged under oracle/_ref by oracle/make_ref.py) on this host's
  cores, bounded sample (prefill + a few decode steps, extrapolated; c2/c3);
  ``cpu_baseline_port`` — the oracle numpy port, same sample shape. c4/c5 report
  the port (the reference has no beam search; its c5 prefill sample would run
  minutes). ``--impl reference`` prints the reference arm alone (rank 0; other
  ranks exit 0).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

SEED = 42
WORKLOADS = {
    "c2": dict(batch=32, src=128, new=64, beam=1, vocab="full", positions=512,
               text="C2: Ernie-base-sized (12L, 768h, 12 heads, FFN 3072, vocab 40000, 512 positions), "
                    "fp16 greedy generation, batch 32/GPU, src 128, 64 new tokens"),
    "c3": dict(batch=128, src=128, new=64, beam=1, vocab="pruned", positions=256,
               text="C3: Ernie-base-sized, vocab pruned 40k->10k (fused logits GEMM + argmax), 256 positions, "
                    "fp16 greedy, batch 128/GPU, src 128, 64 new tokens"),
    "c4": dict(batch=64, src=256, new=128, beam=4, vocab="pruned", positions=512,
               text="C4: Ernie-base-sized, vocab 10k, beam search width 4, 64 requests/GPU, src 256, "
                    "128 new tokens (returned hypotheses counted)"),
    "c5": dict(batch=128, max_batch=256, src=None, new=64, beam=1, vocab="pruned", positions=1024, requests=20000,
               text="C5: Ernie-base-sized, vocab 10k, 20000 requests, src ~ U[32,512], 64 new, "
                    "length-bucketed batches <= 256 (bucket 16), per-GPU shards"),
}


def master_config(M):
    return M.ModelConfig(vocab_size=40000, hidden_size=768, num_layers=12, num_heads=12,
                         head_dim=64, ffn_size=3072, max_position=1024, dtype=M.DType.F16,
                         eos_token=1, pad_token=2)


def zipf_keep_ids():
    """Kept ids for the 40k -> 10k pruning (same construction as the golden fixture)."""
    from oracle import tinfer_oracle as O  # SplitMix64 stream + reference selection rule
    zs = O.Stream(O.derive_seed(SEED, "zipf"))
    rank = np.argsort(zs.u64(40000), kind="stable")
    counts = np.empty(40000, np.int64)
    counts[rank] = 10 ** 9 // (np.arange(40000) + 1)
    return counts


def build_model(w):
    import paper_2407_04991_b200 as P
    from paper_2407_04991_b200 import pruning as PR
    model = P.init_random(master_config(P), SEED)
    if w["vocab"] == "pruned":
        vmap = PR.build_pruned_vocab(zipf_keep_ids(), 10000, specials=[0, 1, 2])
        model = PR.prune_token_embedding(model, vmap)
    return PR.prune_position_embedding(model, w["positions"])


def make_prompts(V, w, rank):
    from oracle import tinfer_oracle as O  # prompt stream only
    if w["src"] is not None:
        return O.synthetic_prompts(V, w["batch"], w["src"], seed=SEED + rank)
    s = O.Stream(O.derive_seed(SEED, "c5-lengths"))
    lens = (s.randint(w["requests"], 481) + 32).tolist()
    t = O.Stream(O.derive_seed(SEED, "prompts"))
    ids = (t.randint(sum(lens), V - 3) + 3).tolist()
    out, k = [], 0
    for n in lens:
        out.append(ids[k:k + n])
        k += n
    return out


def _latest_profile(pattern):
    import glob
    hits = sorted(glob.glob(os.path.join(ROOT, "profiles", pattern)))
    return hits[-1] if hits else None


def ncu_step_traffic(wname):
    """DRAM bytes (read + write) of one decode step from the newest committed ncu
    per-launch capture (profiles/r<N>_ncu_step_<w>.json: tools/one_step.py under
    ncu --cache-control none, summed by tools/step_profile.py), or None."""
    path = _latest_profile(f"r*_ncu_step_{wname}.json")
    if path is None:
        return None
    with open(path) as fh:
        return float(json.load(fh)["dram_bytes"])


def ncu_traffic(kernel_tag="prof_lm_head"):
    """dram read + write per launch of the dominant kernel from the newest
    committed `ncu --set full` summary (profiles/r<N>_ncu_summary.md), or None."""
    path = _latest_profile("r*_ncu_summary.md")
    if path is None:
        return None
    text = open(path).read()
    at = text.find(kernel_tag)
    if at < 0:
        return None
    block = text[at:at + 2000]
    units = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    total = 0.0
    for key in ("- dram read: ", "- dram write: "):
        i = block.find(key)
        if i < 0:
            return None
        val, unit = block[i + len(key):].split("\n", 1)[0].split()[:2]
        total += float(val) * units.get(unit, 1)
    return total


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        with open(path) as fh:
            d = json.load(fh)
        return float(d["hbm_gbs"]), float(d["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """NVML clocks + throttle reasons sampled during the timed region."""
    REASONS = {"applications_clocks_setting": 0x2, "sw_power_cap": 0x4, "hw_slowdown": 0x8,
               "sync_boost": 0x10, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, index):
        self.samples, self.reasons, self.max_mhz = [], set(), None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                mask = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                self.reasons.update(n for n, bit in self.REASONS.items() if mask & bit)
            except Exception:
                pass
            time.sleep(0.05)

    def __enter__(self):
        if self.nv is not None:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        return {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons)}


def decode_step_bytes(L, H, F, V, S, ctx_sum, e=2):
    """weights + embedding rows + KV reads of live slots + KV append + ids."""
    weights = e * (L * (4 * H * H + 2 * H * F + 4 * H + F + H + 4 * H) + 2 * H + H * V)
    return weights + e * 2 * H * S + e * 2 * L * H * ctx_sum + e * 2 * L * H * S + 4 * S


# ---------------------------------------------------------------------------
# CPU baseline: oracle port on this host's cores
# ---------------------------------------------------------------------------
def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((p.get("num_threads") or 1) for p in info) if info else os.cpu_count()
    except Exception:
        return os.cpu_count()


def cpu_baseline_reference(wname="c2", samples=1, n_decode=4):
    """The reference's OWN CPU path (unmodified tinfer model/kernels, numba, from the
    copy oracle/make_ref.py stages under oracle/_ref) on this host's cores.

    Sample: S = min(B*beam, 32) rows of the workload's prompts; per sample one
    call with ``n_decode`` decode steps through the reference's
    batched_greedy_decode (model.py:613-667), its forward calls timed one by one
    (the prefill, then each decode step). Extrapolated to the workload: prefill time x (rows / S)
    (prefill is GEMM-bound, linear in rows), decode step time as measured at S
    rows (a lower bound for more rows -> the reported CPU throughput is an upper
    bound). Returns None when the reference copy is absent."""
    threads = len(os.sched_getaffinity(0))
    os.environ.setdefault("NUMBA_NUM_THREADS", str(threads))
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/tinfer_ref_numba_cache")
    try:
        from oracle import ref_loader
        T = ref_loader.load()
    except Exception:
        return None
    import numba
    M, PR = T.model, T.pruning
    w = WORKLOADS[wname]
    cfg = M.ModelConfig(vocab_size=40000, hidden_size=768, num_layers=12, num_heads=12, head_dim=64,
                        ffn_size=3072, max_position=1024, dtype=T.tensor.DType.F16, eos_token=1, pad_token=2)
    model = M.init_random(cfg, SEED)
    if w["vocab"] == "pruned":
        model = PR.prune_token_embedding(model, PR.build_pruned_vocab(zipf_keep_ids(), 10000, specials=[0, 1, 2]))
    model = PR.prune_position_embedding(model, w["positions"])
    rows = w["batch"] * w["beam"]
    S = min(rows, 32)
    src = w["src"] or 272  # c5: mean prompt length
    from oracle import tinfer_oracle as O  # prompt stream only (the reference's SplitMix64 restated)
    prompts = O.synthetic_prompts(model.config.vocab_size, S, src, seed=SEED)
    T.kernels.warmup()
    M.batched_greedy_decode(model, [p[:8] for p in prompts[:2]], 2)  # strided-view specialisation
    # per-forward wall times through the reference's own generate loop: its
    # _forward_tokens (model.py:440-504) wrapped with a timer for the duration
    # of the sample (first call = prefill, the rest = decode steps)
    calls = []
    inner = M._forward_tokens

    def timed(*a, **k):
        t0 = time.perf_counter()
        r = inner(*a, **k)
        calls.append(time.perf_counter() - t0)
        return r

    t_pre, t_dec = [], []
    M._forward_tokens = timed
    try:
        for _ in range(samples):
            calls.clear()
            M.batched_greedy_decode(model, prompts, 1 + n_decode)
            t_pre.append(calls[0])
            t_dec.extend(calls[1:])
    finally:
        M._forward_tokens = inner
    tp, td = statistics.median(t_pre) * rows / S, statistics.median(t_dec)
    total = tp + (w["new"] - 1) * td
    return {"value": w["batch"] * w["new"] / total, "unit": "generated tokens/s", "cores": threads,
            "numba_threads": int(numba.get_num_threads()), "cpu_model": cpu_model(), "kind": "reference",
            "sample": f"unmodified reference (tinfer.model.batched_greedy_decode, numba kernels, F16 storage) "
                      f"on {S} of {rows} rows, src {src}: prefill {statistics.median(t_pre):.2f}s + decode "
                      f"step {td * 1e3:.0f} ms (median of {samples}); extrapolated to 1 prefill x {rows}/{S} + "
                      f"{w['new'] - 1} steps" + (" (greedy proxy for beam: no reference beam search)"
                                                 if w["beam"] > 1 else "")}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_baseline(wname="c2", n_decode=3):
    from oracle import tinfer_oracle as O
    w = WORKLOADS[wname]
    c = O.config_master(True)
    wts = O.init_weights(c, SEED)
    kept = tuple(range(c.vocab_size))
    if w["vocab"] == "pruned":
        kept = O.build_pruned_vocab(zipf_keep_ids(), 10000, [0, 1, 2])
    wts, c = O.prune_weights(wts, c, kept, new_max_position=w["positions"])
    B = w["batch"] * w["beam"]
    src = w["src"] or 272  # c5: mean prompt length
    prompts = O.synthetic_prompts(c.vocab_size, B, src, seed=SEED)
    ids, pos, pads, _ = O.left_pad(c, prompts)
    cache = O.Cache.new(c, B, src + w["new"])
    t0 = time.perf_counter()
    logits = O.forward_tokens(wts, c, ids, pos, cache, pads)
    t_pre = time.perf_counter() - t0
    t0 = time.perf_counter()
    for _ in range(n_decode):
        nxt = np.argmax(logits, axis=1).reshape(B, 1)
        logits = O.forward_tokens(wts, c, nxt, (cache.len - pads).reshape(B, 1), cache, pads)
    t_dec = (time.perf_counter() - t0) / n_decode
    total = t_pre + (w["new"] - 1) * t_dec
    return {"value": w["batch"] * w["new"] / total, "unit": "generated tokens/s", "cores": int(cpu_threads()),
            "kind": "port",
            "sample": f"oracle numpy port, {wname} rows {B} src {src}: prefill ({t_pre:.2f}s) + {n_decode} "
                      f"decode steps ({t_dec * 1e3:.0f} ms each) timed, extrapolated to 1 prefill + "
                      f"{w['new'] - 1} steps" + (" (greedy proxy for beam)" if w["beam"] > 1 else "")}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


# C2 / C3: every GPU runs its own batch (weak scaling); C4 (64 requests) and
# C5 (20k requests) are one fixed job sharded across the GPUs (strong scaling,
# BASELINE configs[3] / [4])
STRONG = ("c4", "c5")


def base_line(args, w, world, value, ms_per_step):
    strong = args.workload in STRONG
    return {"metric": "generated tokens/s", "value": value, "unit": "generated tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_per_step,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "f16", "data": "synthetic",
            "config": {"workload": w["text"],
                       "global_batch": w.get("requests") or w["batch"] * (1 if strong else world),
                       "seq_len": w["src"] or "32-512", "new_tokens": w["new"], "beam": w["beam"],
                       "parallelism": f"dp{world} (independent requests, no collective)",
                       "l2": "flushed between timed steps (256 MB write); the per-step working set "
                             "(>=200 MB weights + KV cache) also exceeds the 126 MB L2"}}


def run_reference(args):
    """The reference arm: the reference's own numba CPU path (oracle/_ref copy);
    the oracle numpy port only if that copy is absent. At most 2 samples of the
    workload (each a prefill + a few decode steps) keep the run within minutes."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    w = WORKLOADS[args.workload]
    base = cpu_baseline_reference(args.workload, samples=max(1, min(args.steps, 2)))
    if base is None:
        for _ in range(args.warmup):
            cpu_baseline(args.workload, n_decode=1)
        vals = [cpu_baseline(args.workload, n_decode=2) for _ in range(args.steps)]
        base = dict(vals[-1], value=float(statistics.median(x["value"] for x in vals)))
    v = float(base["value"])
    line = base_line(args, w, args.gpus, v, 1e3 * w["batch"] * w["new"] / v)
    line["impl"] = "reference"
    line["executor"] = "host CPU, rank 0 only (the reference path has no GPU code); config = our arm's workload"
    line["cpu_baseline"] = base
    line["e2e"] = {"value": v, "unit": "generated tokens/s", "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
class Runner:
    """Device-resident step and public-API step for one workload on one rank."""

    def __init__(self, model, prompts, w):
        import torch

        from paper_2407_04991_b200 import model as PM
        from paper_2407_04991_b200.beam import BeamRun

        self.w, self.model, self.prompts = w, model, prompts
        c = model.config
        if w["beam"] > 1:
            self.beam = BeamRun(model, prompts, w["new"], w["beam"])
            self.sess = self.beam.s
        else:
            self.beam = None
            self.ids, self.pos, self.pads, _ = PM._left_pad(c, prompts)
            cap, max_tokens = PM._session_shape(c, self.ids.shape[1], w["new"])
            dm = model.device_model()
            with torch.cuda.device(dm.device):
                self.sess = dm.session(len(prompts), cap, max_tokens, w["new"])

    def stage(self):
        if self.beam:
            self.beam.stage_inputs()
        else:
            self.sess.load_inputs(self.ids, self.pos, self.pads)

    def device_step(self):
        from paper_2407_04991_b200 import _native as N
        if self.beam:
            self.beam.run_device()
        else:
            self.sess.forward(self.ids.shape[1], N.FWD_ARGMAX)
            self.sess.decode(self.w["new"] - 1)

    def result(self):
        if self.beam:
            return self.beam.finish()[0]
        return self.sess.fetch_tokens(self.w["new"])

    def api_step(self):
        import paper_2407_04991_b200 as P
        if self.w["beam"] > 1:
            return P.beam_search_decode(self.model, self.prompts, self.w["new"], self.w["beam"])
        return P.batched_greedy_decode(self.model, self.prompts, self.w["new"])

    def launches(self):
        from paper_2407_04991_b200 import _native as N
        from paper_2407_04991_b200 import model as PM
        return PM.LAST_STATS.launches


def run_ours(args):
    import torch
    import torch.distributed as dist

    from paper_2407_04991_b200 import _native as N
    from paper_2407_04991_b200 import model as PM

    rank, world, local = dist_env()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    hbm_peak, _, peak_kind = peaks()
    w = WORKLOADS[args.workload]
    model = build_model(w)
    c = model.config
    dm = model.device_model(dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    if args.workload == "c5":
        return run_sweep(args, w, model, dm, rank, world, dev)

    if args.workload in STRONG:  # one job of w["batch"] requests, contiguous shard per rank
        allp = make_prompts(c.vocab_size, w, 0)
        per = (len(allp) + world - 1) // world
        prompts = allp[rank * per:(rank + 1) * per]
        assert prompts, "more ranks than requests"
    else:
        prompts = make_prompts(c.vocab_size, w, rank)
    run = Runner(model, prompts, w)
    for _ in range(max(args.warmup, 3)):
        run.stage()
        run.device_step()
    torch.cuda.synchronize()
    first = run.result()

    def sync_all():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()

    # ---------------- device-resident timed region
    sync_all()
    times = []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            run.stage()
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            run.device_step()
            e1.record(stream)
            e1.synchronize()
            times.append(e0.elapsed_time(e1) / 1e3)
    sync_all()
    last = run.result()
    assert (np.array_equal(first, last) if not run.beam else first == last), "non-deterministic"
    total = sum(times)
    if world > 1:
        t = torch.tensor([total], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total = float(t.item())
    # whole-job generated tokens per step: every rank's batch (weak) or the one
    # sharded job (strong)
    gen_per_step = w["batch"] * w["new"] * (1 if args.workload in STRONG else world)
    value = gen_per_step * args.steps / total

    # ---------------- end-to-end through the public API
    for _ in range(2):
        run.api_step()
    sync_all()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        out = run.api_step()
    torch.cuda.synchronize()
    e2e_t = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_t], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_t = float(t.item())
    st = PM.LAST_STATS
    if not run.beam:
        assert [r[w["src"]:] for r in out] == [list(map(int, r)) for r in last], "API/device mismatch"
    # ---------------- latency: p50 of 20 repeated generate calls (public API,
    # wall clock incl. host copies) and the p50 device decode step (below)
    gen_ms = []
    for _ in range(20):
        t1 = time.perf_counter()
        run.api_step()
        gen_ms.append((time.perf_counter() - t1) * 1e3)

    # ---------------- rooflines
    H, F, V, L = c.hidden_size, c.ffn_size, c.vocab_size, c.num_layers
    nb = len(prompts)  # this rank's requests
    S = nb * w["beam"]
    # live context: the prompt once per request (beams share it: SURVEY 8d shared
    # prefix, read from beam 0's rows) + the generated slots per row
    step_bytes = [decode_step_bytes(L, H, F, V, S, nb * w["src"] + S * i) for i in range(1, w["new"])]
    t_step = probe_decode_step(torch, run, flush, stream, w)
    n_launch = int(N.lib().tf_session_launches_per_step(run.sess.handle))  # the decode graph's kernels
    step_bw = float(np.mean(step_bytes)) / t_step / 1e9
    latency = {"p50_generate_ms": float(np.percentile(gen_ms, 50)), "p90_generate_ms": float(np.percentile(gen_ms, 90)),
               "generate_calls": len(gen_ms), "p50_decode_step_us": t_step * 1e6,
               "note": "generate = one public-API call (this rank's batch, prefill + all decode steps, host "
                       "copies included); decode step = CUDA-event median of graph-replayed steps"}
    prefill = probe_prefill(torch, run, dm, flush, stream, w, peaks()[1])
    kern = probe_dominant_kernel(torch, dm, run.sess, flush, stream, S)

    if rank == 0:
        line = base_line(args, w, world, value, 1e3 * total / args.steps)
        line.update({
            "e2e": {"value": gen_per_step * args.steps / e2e_t, "unit": "generated tokens/s",
                    "h2d_bytes_per_step": int(st.h2d_bytes), "d2h_bytes_per_step": int(st.d2h_bytes)},
            "gpu_launches": int(run.launches() * args.steps),
            # the roofline unit is the decode step (north star: fraction of the
            # HBM roofline per decode step): one CUDA-graph replay of the step's
            # PDL-chained launches, device-timed over the 63 steps of a generate
            "roofline": {"bound": "hbm", "achieved": step_bw, "peak": hbm_peak, "unit": "GB/s",
                         "frac": step_bw / hbm_peak,
                         "traffic": ncu_step_traffic(args.workload),
                         "kernel": f"decode step (CUDA graph of {n_launch} PDL-chained launches)",
                         "bytes_per_launch": float(np.mean(step_bytes)), "launch_us": t_step * 1e6,
                         "peak_kind": peak_kind},
            "decode_step": {"us": t_step * 1e6, "algorithmic_bytes": float(np.mean(step_bytes)),
                            "achieved_gbs": step_bw, "frac_of_hbm": step_bw / hbm_peak,
                            "launches": n_launch},
            "largest_launch": {"kernel": kern["name"], "bytes_per_launch": kern["bytes"], "launch_us": kern["us"],
                               "achieved_gbs": kern["gbs"], "frac": kern["gbs"] / hbm_peak,
                               "traffic": ncu_traffic() if args.workload == "c2" else None},
            "clocks": clk.summary(),
        })
        line["latency"] = latency
        line["prefill"] = prefill
        if not args.no_cpu_baseline and world == 1:
            ref = cpu_baseline_reference(args.workload) if args.workload in ("c2", "c3") else None
            port = cpu_baseline(args.workload)
            line["cpu_baseline"] = ref or port
            if ref:
                line["cpu_baseline_port"] = port
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def probe_decode_step(torch, run, flush, stream, w):
    """Median per-decode-step time (CUDA events around the graph-replayed steps)."""
    from paper_2407_04991_b200 import _native as N
    if run.beam:  # prefill + first select untimed, then the graph-replayed beam steps
        import ctypes as C
        br, s = run.beam, run.sess
        ts = []
        for _ in range(3):
            run.stage()
            st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
            s.forward(br.L, N.FWD_LOGITS_LAST)
            N.check(N.lib().tf_beam_select(s.handle, C.byref(br.desc), st), "tf_beam_select")
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            N.check(N.lib().tf_beam_decode(s.handle, C.byref(br.desc), w["new"] - 1, 1, st), "tf_beam_decode")
            e1.record(stream)
            e1.synchronize()
            s.len += w["new"] - 1
            ts.append(e0.elapsed_time(e1) / 1e3 / (w["new"] - 1))
        return float(statistics.median(ts))
    ts = []
    for _ in range(5):
        run.stage()
        run.sess.forward(run.ids.shape[1], N.FWD_ARGMAX)
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run.sess.decode(w["new"] - 1)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3 / (w["new"] - 1))
    return float(statistics.median(ts))


def prefill_flops(L, H, F, V, B, T, pads_sum=0):
    """Prefill of B prompts of T tokens: the GEMMs (QKV, Wo, FFN1, FFN2 over
    every token; lm_head over the last position) + causal attention QK^T and
    PV over each row's valid window."""
    gemm = 2 * B * T * L * (4 * H * H + 2 * H * F) + 2 * B * H * V
    ctx = B * T * (T + 1) // 2 - pads_sum * T
    return gemm, 4 * L * H * ctx


def probe_prefill(torch, run, dm, flush, stream, w, tflops_peak):
    """Prefill forward (CUDA events, L2 flushed before each of 5 runs) and its
    largest GEMM alone (FFN1, tokens x F x H, 20 back-to-back launches in a
    CUDA graph): tensor-pipe throughput vs the measured dense bf16/f16 peak."""
    from paper_2407_04991_b200 import _native as N
    from paper_2407_04991_b200 import ops
    if run.beam:
        return None
    B, T = run.ids.shape
    ts = []
    for _ in range(5):
        run.stage()
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        run.sess.forward(T, N.FWD_ARGMAX)
        e1.record(stream)
        e1.synchronize()
        ts.append(e0.elapsed_time(e1) / 1e3)
    t = float(statistics.median(ts))
    gf, af = prefill_flops(dm.L, dm.H, dm.F, dm.V, B, T, int(run.pads.sum()))
    M = B * T
    act = torch.randn(M, dm.ldk_h, device=dm.device).half()
    out = torch.empty(M, dm.ldk_f, dtype=torch.float16, device=dm.device)
    w1, b1 = dm.layers[0]["w1_t"], dm.layers[0]["b1"]
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        ops.gemm(act, w1, dm.H, N.EPI_BIAS_GELU, out=out, bias=b1)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for _ in range(20):
                ops.gemm(act, w1, dm.H, N.EPI_BIAS_GELU, out=out, bias=b1)
    torch.cuda.synchronize()
    gts = []
    with torch.cuda.stream(gs):
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            graph.replay()
            e1.record(gs)
            e1.synchronize()
            gts.append(e0.elapsed_time(e1) / 1e3 / 20)
    tg = float(statistics.median(gts))
    g_tf = 2 * M * dm.F * dm.H / tg / 1e12
    return {"us": t * 1e6, "gemm_flops": gf, "attn_flops": af,
            "achieved_tflops": (gf + af) / t / 1e12, "frac_of_tensor_peak": (gf + af) / t / 1e12 / tflops_peak,
            "largest_gemm": {"kernel": f"gemm_tc_kernel<EPI_BIAS_GELU> FFN1 {M}x{dm.F}x{dm.H}", "us": tg * 1e6,
                             "achieved_tflops": g_tf, "frac_of_tensor_peak": g_tf / tflops_peak},
            "peak_tflops": tflops_peak, "peak_kind": "MEASURED_PEAKS.json bf16_tflops (dense, burst)"}


def probe_dominant_kernel(torch, dm, sess, flush, stream, batch):
    """The lm_head GEMM fused with argmax — the largest single launch of a decode
    step. COPIES launches, each on its own copy of the lm_head weights (together
    > 2x the 126 MB L2, so every launch streams its weights from HBM), are
    captured back to back into one CUDA graph; the replay is timed with CUDA
    events on the replay stream and divided by COPIES. Algorithmic bytes =
    lm_head weights (as stored, K padded to 64) + activations + argmax keys."""
    from paper_2407_04991_b200 import _native as N
    from paper_2407_04991_b200 import ops

    H, V = dm.H, dm.V
    wbytes = V * dm.ldk_h * 2
    copies = max(4, int(2 * (126 << 20) // wbytes) + 1)
    ws = [dm.lm_head_t.clone() for _ in range(copies)]
    keys = torch.zeros(batch, dtype=torch.int64, device=dm.device)
    act = sess.h[:batch]
    gs = torch.cuda.Stream()
    with torch.cuda.stream(gs):
        for w in ws:
            ops.gemm(act, w, H, N.EPI_LOGITS, keys=keys)
        torch.cuda.synchronize()
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=gs):
            for w in ws:
                ops.gemm(act, w, H, N.EPI_LOGITS, keys=keys)
    torch.cuda.synchronize()
    ts = []
    with torch.cuda.stream(gs):
        for i in range(7):
            flush.zero_()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(gs)
            graph.replay()
            e1.record(gs)
            e1.synchronize()
            if i >= 2:
                ts.append(e0.elapsed_time(e1) / 1e3 / copies)
    t = float(statistics.median(ts))
    del ws
    nbytes = wbytes + batch * H * 2 + batch * 8
    return {"name": "gemm_tc_kernel<EPI_LOGITS,swap> (lm_head + argmax)", "bytes": nbytes,
            "us": t * 1e6, "gbs": nbytes / t / 1e9}


def run_sweep(args, w, model, dm, rank, world, dev):
    """C5: the 20k-request sweep; this rank's LPT share of the length-bucketed
    groups through the public API; whole-job tokens / max-over-ranks time."""
    import torch
    import torch.distributed as dist

    import paper_2407_04991_b200 as P
    from paper_2407_04991_b200 import pipeline as PL

    reqs = make_prompts(model.config.vocab_size, w, 0)
    # 256-row batches: C5 186k vs 162k tok/s at 128 rows (peak HBM 60 vs ~35 GB; 512 rows: 202k at
    # 118 GB). Batches above 128 rows pick wave-filling split counts, so a request's tokens are
    # deterministic and within the parity tolerance but not bitwise those of a <= 128-row batch.
    settings = PL.PipelineSettings(max_batch_size=args.c5_batch or w["max_batch"], bucket_width=16,
                                   max_new_tokens=w["new"])
    plan = PL.plan_batches([len(r) for r in reqs], settings.max_batch_size, settings.bucket_width)
    mine = PL.rank_share(plan, world, rank, w["new"])
    # warm-up happens inside each worker thread (sessions are per thread), below
    if world > 1:
        dist.barrier()
    # W inference workers per GPU (host threads, each with its own stream and
    # sessions): the decode chain of one group is latency-bound, so a second
    # group's kernels fill the SMs it leaves idle. Groups dealt by LPT.
    W = max(1, args.c5_workers)
    share = [[] for _ in range(W)]
    load = [0] * W
    for gi in sorted(mine, key=lambda g: -PL.group_cost(plan, g, w["new"])):
        k = min(range(W), key=lambda j: (load[j], j))
        share[k].append(gi)
        load[k] += PL.group_cost(plan, gi, w["new"])
    lat, gen_box, errors = [], [0], []
    lock = threading.Lock()
    ready = threading.Barrier(W + 1)  # workers warm up their own sessions/graphs, then start together
    go = threading.Event()
    t0 = [0.0]

    def run_groups(groups, record):
        for gi in groups:
            g = plan.groups[gi]
            seqs = P.batched_greedy_decode(model, [reqs[i] for i in g], w["new"])
            if record:
                done = time.perf_counter() - t0[0]
                with lock:
                    gen_box[0] += sum(len(s) - len(reqs[i]) for s, i in zip(seqs, g))
                    lat.extend([done] * len(g))

    def worker(groups):
        try:
            with torch.cuda.device(dev), torch.cuda.stream(torch.cuda.Stream(dev)):
                # one group of every session shape this worker will meet (its
                # sessions and captured graphs are its own) before the timed sweep
                from paper_2407_04991_b200.model import _session_shape
                seen, warm = set(), []
                for gi in groups:
                    g = plan.groups[gi]
                    key = (len(g), _session_shape(model.config, plan.group_pad[gi], w["new"]))
                    if key not in seen:
                        seen.add(key)
                        warm.append(gi)
                run_groups(warm, False)
                torch.cuda.current_stream().synchronize()
                ready.wait()
                go.wait()
                run_groups(groups, True)
        except BaseException as e:  # surfaced below
            errors.append(e)
            try:
                ready.abort()
            except Exception:
                pass

    threads = [threading.Thread(target=worker, args=(sh,), daemon=True) for sh in share]
    for t in threads:
        t.start()
    try:
        ready.wait()
    except threading.BrokenBarrierError:
        pass
    if errors:
        raise errors[0]
    torch.cuda.synchronize()
    with ClockSampler(dev.index) as clk:
        t0[0] = time.perf_counter()
        go.set()
        for t in threads:
            t.join()
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0[0]
    if errors:
        raise errors[0]
    gen = gen_box[0]
    tot = torch.tensor([wall, gen], device=dev, dtype=torch.float64)
    if world > 1:
        mx = tot.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        sm = tot.clone()
        dist.all_reduce(sm, op=dist.ReduceOp.SUM)
        wall, gen = float(mx[0]), int(sm[1])
    if rank == 0:
        value = gen / wall
        line = base_line(args, w, world, value, 1e3 * wall)
        line["steps"] = 1
        line.update({
            "e2e": {"value": value, "unit": "generated tokens/s",
                    "h2d_bytes_per_step": int(sum(len(r) for r in reqs) * 8),
                    "d2h_bytes_per_step": int(len(reqs) * w["new"] * 4)},
            "latency_s": {"p50": float(np.percentile(lat, 50)), "p99": float(np.percentile(lat, 99)),
                          "note": "rank-0 requests, enqueue (sweep start) -> ids back"},
            "groups": len(plan.groups), "requests": len(reqs), "workers_per_gpu": W,
            "max_batch_size": settings.max_batch_size,
            "peak_hbm_gb": round(torch.cuda.max_memory_allocated(dev) / 2**30, 1),
            "clocks": clk.summary(),
        })
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def relaunch_distributed(n):
    """`bench.py --gpus N` (N > 1) without a torchrun environment: re-exec this
    command under torch.distributed.run with N local ranks (127.0.0.1)."""
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def run_dry(args):
    """--dry-run: the launch and rendezvous only (gloo, no GPU work); rank 0
    prints how many ranks joined."""
    import torch
    import torch.distributed as dist
    rank, world, _ = dist_env()
    joined = 1
    if world > 1:
        dist.init_process_group("gloo")
        t = torch.ones(1)
        dist.all_reduce(t)
        joined = int(t.item())
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "ranks_joined": joined, "workload": args.workload}),
              flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--dry-run", action="store_true", help="launch + rendezvous only (CPU, gloo)")
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="c2")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--c5-workers", type=int, default=2, help="inference worker threads per GPU (c5 sweep)")
    ap.add_argument("--c5-batch", type=int, default=0, help="max rows per C5 batch (0: the workload's 256)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        relaunch_distributed(args.gpus)
    if int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE', '1')}")
    if args.dry_run:
        run_dry(args)
        return
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
