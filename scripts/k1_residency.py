"""Do the K1 (gather-only) CTAs of the solo kernel co-reside two per SM?
COPRIS_TRACE lifetimes per CTA vs the launch duration, for K1, the forward-only
loss and the loss with bf16 dlogits at the same shape."""
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

V = int(sys.argv[1]) if len(sys.argv) > 1 else 32000
ctx = Copris(0)
hb = make_host_batch(1, 128, 8, V, fixed_len=64)
T = hb.n_tok
tgt = torch.from_numpy(hb.target).cuda()
logits = make_logits(T, V, tgt, 1, device="cuda")
batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, np.zeros(T, np.float32), hb.cur_stage,
               stage=hb.stage, reward=hb.reward)
outs = ctx.alloc_outputs(T, logits.device)
dl = torch.empty_like(logits)
buf = (C.c_longlong * (2048 * 10))()
runs = {
    "k1": lambda: ctx.sequence_logprobs(logits, tgt),
    "fwd_only": lambda: ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=None, total_tokens=T),
    "loss_bf16": lambda: ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T),
}
for name, fn in runs.items():
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    e1.record()
    torch.cuda.synchronize()
    ctx._call(ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10))
    a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 10)
    info = ctx.last_launch()
    ms = e0.elapsed_time(e1)
    g = info.get("grid") or int((a[:, 9] > 0).sum())
    if name == "k1" or g == 0:  # K1 records no trace: time only
        print(f"{name:10s} V={V} T={T} {ms * 1e3:.0f} us", flush=True)
        continue
    life = a[:g, 8] / 1e3
    rows = a[:g, 5]
    print(f"{name:10s} V={V} T={T} {info['kernel']} grid={g} {ms * 1e3:.0f} us; CTA lifetime us: "
          f"first half mean {life[:g // 2].mean():.0f} (min {life[:g // 2].min():.0f}), "
          f"second half mean {life[g // 2:].mean():.0f} (min {life[g // 2:].min():.0f}); rows/CTA {rows.mean():.1f}",
          flush=True)
    if a[0, 6] > 0:  # pair family: start time and SM of every CTA
        t0 = a[:g, 6].min()
        st = (a[:g, 6] - t0) / 1e3
        sm = a[:g, 7]
        late = st > 0.25 * ms * 1e3
        print(f"           start us: CTAs starting after 25% of the launch: {int(late.sum())}; "
              f"distinct SMs {len(np.unique(sm))}; max CTAs per SM {np.bincount(sm).max()}; "
              f"first CTA of the late ones {int(np.argmax(late)) if late.any() else -1}", flush=True)
