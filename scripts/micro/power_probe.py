"""Power/clock probe: sustained device copy vs the fused loss kernel (3 s each),
nvidia-smi sampled every 100 ms. Tells whether the loss kernel is power-capped
because of HBM traffic (a plain copy caps too) or because of SM work."""
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))


def sample(fn, seconds=3.0):
    p = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks_event_reasons.sw_power_cap",
                          "--format=csv,noheader,nounits", "-lms", "100"], stdout=subprocess.PIPE, text=True)
    rows = []
    th = threading.Thread(target=lambda: [rows.append(l.strip().split(", ")) for l in p.stdout], daemon=True)
    th.start()
    time.sleep(0.5)
    n0 = len(rows)
    t0 = time.time()
    it = 0
    while time.time() - t0 < seconds:
        fn()
        it += 1
        if it % 4 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    el = time.time() - t0
    n1 = len(rows)
    p.terminate()
    sm = [float(r[0]) for r in rows[n0:n1]]
    pw = [float(r[1]) for r in rows[n0:n1]]
    cap = sum(1 for r in rows[n0:n1] if r[2].startswith("Active"))
    return {"iters_per_s": it / el, "sm_mhz": statistics.median(sm), "power_w": statistics.median(pw),
            "power_cap_frac": cap / max(1, n1 - n0)}


def main():
    from paper_2511_05589_b200 import ClipConfig, Copris
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.workload import make_logits
    import numpy as np
    V, T = 151936, 16384
    src = torch.empty(T * V, dtype=torch.bfloat16, device="cuda")
    dst = torch.empty_like(src)
    out = {}
    r = sample(lambda: dst.copy_(src))
    r["GBs"] = r["iters_per_s"] * src.numel() * 4 / 1e9
    out["copy"] = r
    ctx = Copris(0)
    tgt = torch.randint(0, V, (T,), device="cuda", dtype=torch.int32)
    logits = make_logits(T, V, tgt, 3, device="cuda")
    tok_off = np.arange(0, T + 1, 512, dtype=np.int64)
    n = len(tok_off) - 1
    batch = upload(ctx, tok_off, np.arange(0, n + 1, 8, dtype=np.int64), tgt.cpu().numpy(),
                   np.full(T, -5, np.float32), 2, stage=(np.arange(T) % 2 + 1).astype(np.uint32),
                   reward=(np.arange(n) % 2).astype(np.float64))
    outs = ctx.alloc_outputs(T, logits.device)
    dl = torch.empty_like(logits)
    variants = os.environ.get("PROBE_VARIANTS", "stream:2,stream:0").split(",")
    for v in variants:
        impl, la = v.split(":")
        os.environ["COPRIS_FUSED_IMPL"] = impl
        os.environ["COPRIS_TUNE_LOOKAHEAD"] = la
        r = sample(lambda: ctx.loss_chunk_fused(logits, batch, ClipConfig(), outs, dlogits=dl))
        r["GBs"] = r["iters_per_s"] * T * (4 * V + 16) / 1e9
        r["kernel"] = ctx.last_launch()["kernel"]
        out[v] = r
    print(json.dumps(out))


if __name__ == "__main__":
    main()
