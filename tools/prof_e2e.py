"""Host-side cost of the public-API generate call: median wall time per call,
then a cProfile of 10 calls. usage: python tools/prof_e2e.py [c2|c4]"""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import bench, torch
import paper_2407_04991_b200 as P
wname = sys.argv[1] if len(sys.argv) > 1 else "c2"
w = bench.WORKLOADS[wname]
model = bench.build_model(w)
prompts = bench.make_prompts(model.config.vocab_size, w, 0)
if w["beam"] > 1:
    call = lambda: P.beam_search_decode(model, prompts, w["new"], w["beam"])
else:
    call = lambda: P.batched_greedy_decode(model, prompts, w["new"])
for _ in range(3): call()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(10): call()
torch.cuda.synchronize()
print("per call ms", (time.perf_counter() - t) / 10 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): call()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(16)
