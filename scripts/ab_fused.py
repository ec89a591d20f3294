"""A/B of fused-kernel selections on one chunk of the bench workload, in
alternation on the same box: each measurement runs `reps` back-to-back
launches (long enough to reach the power cap) and reports the algorithmic
GB/s (4V + 16 bytes per row) and the SM clock sampled meanwhile.

  python scripts/ab_fused.py [V] [rows] [reps] [rounds] opt=val[,opt=val] ...
each positional `name:opt=val,...` is one arm (context options, e.g.
`pair:fused_impl=3` `ring:fused_impl=1`)."""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05589_b200 import ClipConfig, Copris
from paper_2511_05589_b200.packing import upload
from paper_2511_05589_b200.workload import make_host_batch, make_logits

V, rows, reps, rounds = (int(a) for a in sys.argv[1:5])
arms = []
for a in sys.argv[5:]:
    name, _, opts = a.partition(":")
    arms.append((name, dict((k, int(v)) for k, v in (o.split("=") for o in opts.split(",") if o))))
ctx = Copris(0)
hb = make_host_batch(1, max(1, rows // 4096), 8, V, fixed_len=min(rows, 512))
T = hb.n_tok
logits = make_logits(T, V, torch.from_numpy(hb.target).cuda(), 1, device="cuda")
blp = np.zeros(T, np.float32)
batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage,
               reward=hb.reward)
outs = ctx.alloc_outputs(T, logits.device)
dl = torch.empty_like(logits)
defaults = {k: ctx.get_option(k) for a in arms for k in a[1]}


def clocks():
    q = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                        "-i", "0"], capture_output=True, text=True).stdout.strip().split(",")
    return q


res = {n: [] for n, _ in arms}
for rnd in range(rounds):
    for name, opts in arms:
        for k, v in defaults.items():
            ctx.set_option(k, v)
        for k, v in opts.items():
            ctx.set_option(k, v)
        for _ in range(3):
            ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T)
        e1.record()
        time.sleep(0.5)
        ck = clocks()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        gbs = T * (4 * V + 16) / ms / 1e6
        res[name].append(gbs)
        print(f"round {rnd} {name:10s} {ctx.last_launch()['kernel']:34s} {ms:8.3f} ms/launch "
              f"{gbs:7.0f} GB/s  sm/power {ck}", flush=True)
ctx.check()
for name, v in res.items():
    print(f"{name:10s} mean {np.mean(v):7.0f} GB/s  ({', '.join(f'{x:.0f}' for x in v)})")
