"""One C2 generate with the megakernel (for ncu)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ["TF_MEGAKERNEL"] = "1"
import torch
import paper_2407_04991_b200 as P
from paper_2407_04991_b200.pruning import prune_position_embedding
from oracle import tinfer_oracle as O
cfg = P.ModelConfig(40000, 768, 12, 12, 64, 3072, 1024, P.DType.F16, 1, 2)
m = prune_position_embedding(P.init_random(cfg, 42), 512)
prompts = O.synthetic_prompts(40000, 32, 128)
for _ in range(2):
    P.batched_greedy_decode(m, prompts, 64)
torch.cuda.synchronize()
print("done")
