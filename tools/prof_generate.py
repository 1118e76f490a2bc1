"""Host-side cost of one public-API generate call (C2): median wall time of
batched_greedy_decode after warm-up, then a cProfile of 5 calls (the device
sync dominates; the rest is validation, padding and launches). GPU box only."""
import cProfile, pstats, time, sys
sys.path.insert(0, '.')
import bench
import paper_2407_04991_b200 as P
w = bench.WORKLOADS["c2"]
m = bench.build_model(w)
prompts = bench.make_prompts(m.config.vocab_size, w, 0)
for _ in range(3): P.batched_greedy_decode(m, prompts, w["new"])
ts=[]
for _ in range(10):
    t=time.perf_counter(); P.batched_greedy_decode(m, prompts, w["new"]); ts.append(time.perf_counter()-t)
print("generate ms", sorted(ts)[5]*1e3)
pr=cProfile.Profile(); pr.enable()
for _ in range(5): P.batched_greedy_decode(m, prompts, w["new"])
pr.disable()
st=pstats.Stats(pr); st.sort_stats('tottime').print_stats(14)
