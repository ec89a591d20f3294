"""LM-head forward (tcgen05 + fused LSE partials) vs cuBLAS, and the chunked
LM-head IS-loss step in its variants: step_default (cuBLAS forward -> one-pass
fused loss in place -> cuBLAS backward), step_fused_loss (the same with the
tcgen05 forward, logits only), step_lse (tcgen05 forward with LSE partials ->
merge -> K2 -> K3), step_tcgen05_* (backward GEMMs on the tcgen05 kernels);
composed = the default written out by hand. Every timing is a loop of >= 1.5 s
with its own nvidia-smi clock record (sustained, at the power cap)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402
from paper_2511_05589_b200 import ClipConfig, Copris
from paper_2511_05589_b200.lmhead import lmhead_grpo_step_loss
from paper_2511_05589_b200.packing import upload


CLOCKS = {}


def timeit(fn, iters=10, warm=3, name=None, seconds=1.5):
    """Mean ms per call over a timed loop of at least `seconds` (so the clock
    sampler sees it under load); nvidia-smi clocks of the loop in CLOCKS[name]."""
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    reps = max(iters, int(seconds * 1e3 / max(ms, 1e-3)))
    sampler = ClockSampler(None)
    sampler.start()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    CLOCKS[name or getattr(fn, "__name__", "?")] = sampler.stop()
    return s.elapsed_time(e) / reps


def peaks():
    try:
        with open("MEASURED_PEAKS.json") as f:
            p = json.load(f)
        return p["bf16_tflops"], p["bf16_tflops_sustained"], "MEASURED_PEAKS.json"
    except (OSError, KeyError, ValueError):
        return 2250.0, 2250.0, "nominal dense bf16"


def main():
    sampler = ClockSampler(None)
    sampler.start()
    T = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
    H = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
    V = int(sys.argv[3]) if len(sys.argv) > 3 else 151936
    ctx = Copris(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    x = torch.randn(T, H, device="cuda", generator=g).to(torch.bfloat16)
    w = (torch.randn(V, H, device="cuda", generator=g) / H ** 0.5).to(torch.bfloat16)
    tgt = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32, generator=g)
    ldv = (V + 7) // 8 * 8
    buf = torch.empty((T, ldv), dtype=torch.bfloat16, device="cuda")[:, :V]
    part = torch.empty((T, ctx.lib.copris_lmhead_num_vtiles(V), 2), dtype=torch.float32, device="cuda")
    flops = 2.0 * T * H * V
    t_ours = timeit(lambda: ctx.lmhead_logits(x, w, tgt, logits=buf, partials=part), name="lmhead_fwd")
    t_cublas = timeit(lambda: torch.mm(x, w.t(), out=buf), name="cublas_fwd")
    out = {"T": T, "H": H, "V": V,
           "lmhead_fwd_ms": t_ours, "lmhead_fwd_tflops": flops / t_ours / 1e9,
           "cublas_fwd_ms": t_cublas, "cublas_fwd_tflops": flops / t_cublas / 1e9}
    # full step
    n_traj = T // 512
    tok_off = np.arange(0, T + 1, 512, dtype=np.int64)
    group_off = np.arange(0, n_traj + 1, 8, dtype=np.int64)
    stage = (np.arange(T) % 2).astype(np.uint32) + 1
    blp = np.full(T, -10.0, np.float32)
    reward = (np.arange(n_traj) % 2).astype(np.float64)
    batch = upload(ctx, tok_off, group_off, tgt.cpu().numpy(), blp, 2, stage=stage, reward=reward)
    dW = torch.zeros((V, H), dtype=torch.float32, device="cuda")
    chunk = int(sys.argv[4]) if len(sys.argv) > 4 else 8192
    t_step = timeit(lambda: lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk,
                                                  dweight=dW, loss_impl="lse", fwd_impl="tcgen05"),
                    iters=3, warm=1, name="step_lse")
    wt = w.t().contiguous()
    t_step_tc = timeit(lambda: lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk,
                                                     dweight=dW, dhidden_impl="tcgen05", weight_t=wt,
                                                     dweight_impl="tcgen05", fwd_impl="tcgen05"),
                       iters=3, warm=1,
                       name="step_tcgen05_bwd")
    t_step_dh = timeit(lambda: lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk,
                                                     dweight=dW, dhidden_impl="tcgen05", weight_t=wt,
                                                     fwd_impl="tcgen05"),
                       iters=3, warm=1, name="step_tcgen05_dhidden")
    t_step_fused = timeit(lambda: lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk,
                                                        dweight=dW, loss_impl="fused", fwd_impl="tcgen05"),
                          iters=3, warm=1, name="step_fused_loss")
    t_step_default = timeit(lambda: lmhead_grpo_step_loss(ctx, x, w, batch, ClipConfig(), chunk_rows=chunk,
                                                          dweight=dW),
                            iters=3, warm=1, name="step_default")
    dh = torch.empty_like(x)
    outs = ctx.alloc_outputs(T, x.device)
    out4 = torch.empty(4, dtype=torch.float64, device="cuda")

    def composed():
        for a in range(0, T, chunk):
            n = min(chunk, T - a)
            lg = buf[:n]
            torch.mm(x[a:a + n], w.t(), out=lg)
            ctx.loss_chunk_fused(lg, batch, ClipConfig(), outs, dlogits=lg, row_base=a, total_tokens=T)
            torch.mm(lg, w, out=dh[a:a + n])
            torch.addmm(dW, lg.t(), x[a:a + n], out_dtype=torch.float32, out=dW)
        ctx.reduce(outs, T, out4)
        ctx.check()
        return out4.cpu()

    t_comp = timeit(composed, iters=3, warm=1, name="composed_step")
    burst, sustained, src = peaks()
    step_tf = 6 * T * H * V / t_step_default / 1e9  # the default step (cuBLAS GEMMs + one-pass loss)
    out.update({"step_lse_ms": t_step, "step_fused_loss_ms": t_step_fused, "step_default_ms": t_step_default, "step_tcgen05_bwd_ms": t_step_tc, "step_tcgen05_dhidden_ms": t_step_dh,
                "composed_step_ms": t_comp, "chunk": chunk, "step_tflops": step_tf,
                "step_frac_of_sustained_bf16": step_tf / sustained,
                "fwd_frac_of_burst_bf16": out["lmhead_fwd_tflops"] / burst,
                "cublas_fwd_frac_of_burst_bf16": out["cublas_fwd_tflops"] / burst,
                "peaks": {"bf16_tflops": burst, "bf16_tflops_sustained": sustained, "source": src},
                "clocks_per_measurement": CLOCKS, "clocks_whole_script": sampler.stop()})
    print(json.dumps(out))


if __name__ == "__main__":
    main()
