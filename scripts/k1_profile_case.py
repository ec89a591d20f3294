"""One K1 (copris_logprob_gather) workload for ncu: `rows` rows at vocabulary V,
5 launches (the first ones are warm-up for `ncu -s`)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from paper_2511_05589_b200 import Copris
from paper_2511_05589_b200.workload import make_logits

V = int(sys.argv[1]) if len(sys.argv) > 1 else 32000
rows = max(1024, min(65536, (8 << 30) // (2 * V)))
ctx = Copris(0)
tgt = torch.randint(0, V, (rows,), dtype=torch.int32, device="cuda")
logits = make_logits(rows, V, tgt, 1, device="cuda")
for _ in range(5):
    ctx.sequence_logprobs(logits, tgt)
torch.cuda.synchronize()
ctx.check()
print("k1 rows", rows, "V", V, ctx.last_launch())
