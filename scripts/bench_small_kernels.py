"""HBM roofline of the O(T) kernels of the path at BASELINE sizes (CUDA events,
inputs resident, each launch timed over `reps` back-to-back launches):

  behaviour_kernel   concat_segments select + stale flags  (17 B/token)
  expand_u32_kernel  stage[t] from segment (offset, version) (4 B/token + segments)
  token_traj         trajectory id per token                (4 B/token + trajectories)
  reduce_kernel      loss / token / stale / clipped sums     (9 B/token)
  group_advantages   per-group mean / std, fp64             (16 B/trajectory)

usage: python scripts/bench_small_kernels.py [config ...]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05589_b200 import Copris
from paper_2511_05589_b200.workload import CONFIGS, make_host_batch


def peak():
    try:
        with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                               "MEASURED_PEAKS.json")) as f:
            return float(json.load(f)["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


def timed(fn, reps=20):
    """Device time per launch: `reps` launches captured in one CUDA graph, so
    the host-side launch cost (Python + ctypes, ~10 us) is not measured."""
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
    torch.cuda.current_stream().wait_stream(side)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(reps):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e-3


def main():
    names = sys.argv[1:] or ["grpo_128x8_v151936", "grpo_512x16_v151936"]
    ctx = Copris(0)
    pk = peak()
    dev = torch.device("cuda", 0)
    for name in names:
        c = dict(CONFIGS[name])
        P, G, V = c.pop("P"), c.pop("G"), c.pop("vocab")
        c.pop("strong", None)
        hb = make_host_batch(1, P, G, V, **c)
        T, n = hb.n_tok, hb.n_traj
        stage = torch.from_numpy(hb.stage.view(np.int32)).to(dev)
        blp = torch.randn(T, device=dev)
        cur = torch.randn(T, device=dev)
        seg_off = torch.from_numpy(hb.seg_off).to(dev)
        seg_ver = torch.from_numpy(hb.seg_ver.view(np.int32)).to(dev)
        tok_off = torch.from_numpy(hb.tok_off).to(dev)
        rew = torch.from_numpy(hb.reward).to(dev)
        goff = torch.from_numpy(hb.group_off).to(dev)
        goff_host = hb.group_off.tolist()
        outs = {"obj": torch.randn(T, dtype=torch.float64, device=dev),
                "flags": torch.randint(0, 4, (T,), dtype=torch.uint8, device=dev)}
        out4 = torch.empty(4, dtype=torch.float64, device=dev)
        n_seg = len(hb.seg_ver)
        rows = [
            ("behaviour_kernel (K2 concat)", 17 * T,
             lambda: ctx.concat_segments(stage, hb.cur_stage, blp, cur)),
            ("expand_u32_kernel (stage)", 4 * T + 12 * n_seg,
             lambda: ctx.expand_segments(seg_off, seg_ver, T)),
            ("expand_u32_kernel (token_traj)", 4 * T + 8 * n,
             lambda: ctx.token_traj(tok_off, T)),
            ("reduce_kernel", 9 * T, lambda: ctx.reduce(outs, T, out4)),
            ("group_advantages_kernel", 16 * n + 8 * (P + 1),
             lambda: ctx.compute_advantages(rew, goff, group_off_host=goff_host)),
        ]
        print(f"{name}: T = {T:,} tokens, {n:,} trajectories, {n_seg:,} segments")
        for label, nbytes, fn in rows:
            s = timed(fn)
            gbs = nbytes / s / 1e9
            print(f"  {label:32s} {s * 1e6:9.1f} us  {gbs:8.1f} GB/s  {gbs / pk:6.3f} of {pk:.0f}")


if __name__ == "__main__":
    main()
