"""Per-row phase breakdown of the fused kernel (COPRIS_TRACE): run one chunk of
the bench workload and print mean cycles per row in each phase."""
import os, sys, ctypes as C
os.environ.setdefault("COPRIS_TRACE", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2511_05589_b200 import ClipConfig, Copris
from paper_2511_05589_b200.packing import upload
from paper_2511_05589_b200.workload import make_host_batch, make_logits

V = int(sys.argv[1]) if len(sys.argv) > 1 else 151936
rows = int(sys.argv[2]) if len(sys.argv) > 2 else 16384
ctx = Copris(0)
hb = make_host_batch(1, 64, 8, V, fixed_len=rows // 512)
T = hb.n_tok
logits = make_logits(T, V, torch.from_numpy(hb.target).cuda(), 1, device="cuda")
blp = np.zeros(T, np.float32)
batch = upload(ctx, hb.tok_off, hb.group_off, hb.target, blp, hb.cur_stage, stage=hb.stage, reward=hb.reward)
outs = ctx.alloc_outputs(T, logits.device)
dl = torch.empty_like(logits)
# TRACE_WARMUP launches first (e.g. a few thousand to reach the power cap)
for rep in range(int(os.environ.get("TRACE_WARMUP", "3"))):
    ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T)
torch.cuda.synchronize()
buf = (C.c_longlong * (2048 * 10))()
ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10)  # reset after warmup
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl, total_tokens=T)
e1.record(); torch.cuda.synchronize()
ctx._call(ctx.lib.copris_ctx_trace_read(ctx.h, buf, 2048 * 10))
a = np.frombuffer(buf, dtype=np.int64).reshape(2048, 10)
a = a[a[:, 5] > 0]
info = ctx.last_launch()
per = a[:, :5].sum(0) / a[:, 5].sum()
waits = a[:, 6:8].sum(0) / a[:, 5].sum()
ms = e0.elapsed_time(e1)
print(f"V={V} rows={T} kernel={info} {ms:.3f} ms, {T * (4*V+16) / ms / 1e6:.0f} GB/s")
for name, v in zip(["passB", "waitA", "scalar", "waitB", "passC"], per):
    print(f"  {name:8s} {v:9.0f} cycles/row ({100*v/per.sum():.1f}%)")
print(f"  total    {per.sum():9.0f} cycles/row; CTAs traced {len(a)}")
if info["kernel"].startswith("fused_stream"):  # the pair family keeps entry time / SM id in slots 6/7
    print(f"  of which waiting for ring data: passB {waits[0]:.0f}, passC {waits[1]:.0f} cycles/row")
life_ns, life_cyc = a[:, 8], a[:, 9]
print(f"  CTA lifetime: {life_cyc.mean():.0f} cycles, {life_ns.mean() / 1e3:.1f} us "
      f"(min {life_ns.min() / 1e3:.1f}, max {life_ns.max() / 1e3:.1f}) -> "
      f"{(life_cyc / life_ns).mean():.3f} GHz; rows/CTA {a[:, 5].mean():.1f} "
      f"(min {a[:, 5].min()}, max {a[:, 5].max()})")
