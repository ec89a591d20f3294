"""K1 (copris_logprob_gather, the reference's sequence_logprobs,
policy.hpp:160-173) at the HBM roofline: the fused kernels in gather-only mode
(one read of each bf16 logit, online log-sum-exp, cur_lp + lse out).

Algorithmic bytes per token: 2V (logits) + 4 (target) + 8 (cur_lp, lse).
Each measurement: `reps` launches over a chunk of `rows` rows captured in one
CUDA graph (device time per launch), clocks sampled meanwhile.

usage: python scripts/bench_k1.py [V ...]   (default: 32000 151936 256000)
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

from bench import ClockSampler, measured_peaks
from paper_2511_05589_b200 import Copris
from paper_2511_05589_b200.workload import make_logits


def main():
    vocabs = [int(a) for a in sys.argv[1:]] or [32000, 151936, 256000]
    ctx = Copris(0)
    peak, src = measured_peaks()
    for V in vocabs:
        rows = max(1024, min(65536, (8 << 30) // (2 * V)))  # ~8 GB of logits
        tgt = torch.randint(0, V, (rows,), dtype=torch.int32, device="cuda")
        logits = make_logits(rows, V, tgt, 1, device="cuda")
        lp = torch.empty(rows, dtype=torch.float32, device="cuda")
        lse = torch.empty(rows, dtype=torch.float32, device="cuda")
        run = lambda: ctx.sequence_logprobs(logits, tgt, out_lp=lp, out_lse=lse)
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            run()
        torch.cuda.current_stream().wait_stream(side)
        reps = 20
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(reps):
                run()
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        sampler = ClockSampler(None)
        sampler.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        clocks = sampler.stop()
        ctx.check()
        s = e0.elapsed_time(e1) / 1e3 / (5 * reps)
        byt = rows * (2 * V + 12)
        print(json.dumps({"kernel": "K1 copris_logprob_gather", "vocab": V, "rows": rows,
                          "us_per_launch": s * 1e6, "rows_per_s": rows / s, "GBps": byt / s / 1e9,
                          "frac": byt / s / 1e9 / peak, "peak": peak, "peak_source": src,
                          "clocks": clocks}), flush=True)


if __name__ == "__main__":
    main()
