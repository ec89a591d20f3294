"""Fixed per-step cost of a small fused loss step (config #5's one-group case):
CUDA-graph replay of ONE fused launch (loss + in-kernel reduction) over n rows at
V = 32,000, n = 8 .. 4,096; prints ms/step and the algorithmic fraction of the
measured HBM peak. usage: python scripts/small_step_sweep.py [impl ...]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from bench import measured_peaks
from paper_2511_05589_b200 import ClipConfig, Copris
from paper_2511_05589_b200.packing import upload
from paper_2511_05589_b200.workload import make_host_batch, make_logits, stale_logprobs

V = 32000
args = sys.argv[1:]
noreduce = "--no-reduce" in args
impls = [a for a in args if not a.startswith("--")] or ["auto"]
peak, _ = measured_peaks()
for impl in impls:
    ctx = Copris(0)
    ctx.set_option("fused_impl", {"auto": 0, "tma": 2, "pair": 3, "solo": 4}[impl])
    for n in ((8, 2048) if noreduce else (8, 148, 444, 1024, 2048, 4096)):
        L = max(1, n // 8)
        hb = make_host_batch(1, 1, 8, V, fixed_len=L)
        T = hb.n_tok
        tgt = torch.from_numpy(hb.target).cuda()
        logits = make_logits(T, V, tgt, 1, device="cuda")
        cur, _ = ctx.sequence_logprobs(logits, tgt)
        blp = stale_logprobs(cur.cpu().numpy(), hb.stage, hb.cur_stage, 1)
        batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage,
                       reward=hb.reward)
        outs = ctx.alloc_outputs(T, logits.device)
        dl = torch.empty_like(logits)
        out4 = torch.zeros(4, dtype=torch.float64, device="cuda")
        run = lambda: ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T,
                                           out4=None if noreduce else out4)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            run()
        torch.cuda.current_stream().wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            run()
        for _ in range(20):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        reps = 500
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        info = ctx.last_launch()
        print(json.dumps({"impl": impl, "kernel": info["kernel"], "fused_reduce": info.get("fused_reduce"), "out4": not noreduce,
                          "rows": T, "us_per_step": ms * 1e3,
                          "frac": T * (4 * V + 16) / (ms / 1e3) / 1e9 / peak}), flush=True)
    ctx.check()
