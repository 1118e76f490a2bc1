import cProfile, pstats, sys, os, time
sys.path.insert(0, os.getcwd())
import bench, torch
import paper_2407_04991_b200 as P
w = bench.WORKLOADS["c2"]
model = bench.build_model(w)
prompts = bench.make_prompts(model.config.vocab_size, w, 0)
for _ in range(3): P.batched_greedy_decode(model, prompts, w["new"])
torch.cuda.synchronize()
t=time.perf_counter()
for _ in range(10): P.batched_greedy_decode(model, prompts, w["new"])
torch.cuda.synchronize()
print("per call ms", (time.perf_counter()-t)/10*1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(10): P.batched_greedy_decode(model, prompts, w["new"])
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
