"""Tail of one fused-loss launch: per-CTA entry and end times (COPRIS_TRACE,
pair family) against the launch's device time. If CTAs end far apart, static
row striding leaves SMs idle at the end of every chunk launch.

usage: python scripts/cta_tail.py V rows [reps]"""
import ctypes as C
import os
import sys

os.environ.setdefault("COPRIS_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_2511_05589_b200 import ClipConfig, Copris
from paper_2511_05589_b200.packing import upload
from paper_2511_05589_b200.workload import make_host_batch, make_logits

V = int(sys.argv[1]) if len(sys.argv) > 1 else 151936
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 32768
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
ctx = Copris(0)
hb = make_host_batch(1, max(1, rows // 512), 8, V, fixed_len=64)
T = hb.n_tok
logits = make_logits(T, V, torch.from_numpy(hb.target).cuda(), 1, device="cuda")
batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, np.zeros(T, np.float32), hb.cur_stage,
               stage=hb.stage, reward=hb.reward)
outs = ctx.alloc_outputs(T, logits.device)
dl = torch.empty_like(logits)
buf = (C.c_longlong * (2048 * 10))()
run = lambda: ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T)
for _ in range(5):
    run()
torch.cuda.synchronize()
for rep in range(reps):
    ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    ctx._call(ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10))
    a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 10)
    info = ctx.last_launch()
    g = info["grid"]
    ent = a[:g, 6].astype(np.float64)
    t0 = ent.min()
    end = (ent + a[:g, 8] - t0) / 1e3
    st = (ent - t0) / 1e3
    rows_cta = a[:g, 5]
    ms = e0.elapsed_time(e1)
    q = np.percentile(end, [0, 10, 50, 90, 100])
    print(f"V={V} T={T} {info['kernel']} grid={g} launch {ms * 1e3:.0f} us; entry max {st.max():.1f} us; "
          f"CTA end us p0/p10/p50/p90/max {q[0]:.0f}/{q[1]:.0f}/{q[2]:.0f}/{q[3]:.0f}/{q[4]:.0f}; "
          f"mean end {end.mean():.0f}; idle SM-time after each CTA's end {100 * (q[4] - end).mean() / q[4]:.1f}%; "
          f"rows/CTA {rows_cta.min()}-{rows_cta.max()}", flush=True)
