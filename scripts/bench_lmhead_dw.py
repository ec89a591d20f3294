"""LM-head backward weight gradient dW [V x H] += dlogits^T @ hidden:
copris_lmhead_dweight (tcgen05 CTA pair, MN-major operands) vs cuBLAS addmm
(fp32 out); --dhidden also times dhidden = dlogits @ W (copris_lmhead_dhidden vs
torch.mm). Usage: python scripts/bench_lmhead_dw.py [--dhidden] [T ...] (H=4096, V=151,936)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2511_05589_b200 import Copris


def timeit(fn, iters=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    flags = [a for a in sys.argv[1:] if a.startswith("--")]
    Ts = [int(a) for a in sys.argv[1:] if not a.startswith("--")] or [4096, 8192]
    H, V = 4096, 151936
    ctx = Copris(0)
    g = torch.Generator(device="cuda").manual_seed(0)
    w_ld = (V + 7) // 8 * 8
    dW = torch.zeros((V, H), dtype=torch.float32, device="cuda")
    dW2 = torch.zeros_like(dW)
    print(f"# dW += dlogits^T @ hidden, H={H}, V={V}, fp32 dW, 1 B200")
    for T in Ts:
        dl = (torch.randn((T, w_ld), device="cuda", generator=g) * 1e-3).to(torch.bfloat16)[:, :V]
        x = torch.randn((T, H), device="cuda", generator=g).to(torch.bfloat16)
        flops = 2.0 * T * H * V
        if "--only-dhidden" not in flags:
            t_ours = timeit(lambda: ctx.lmhead_dweight(dl, x, out=dW))
            t_cub = timeit(lambda: torch.addmm(dW2, dl.t(), x, out_dtype=torch.float32, out=dW2))
            print(f"T={T} tcgen05 pair MN-major  {t_ours:.3f} ms  {flops / t_ours / 1e9:.0f} TFLOP/s  "
                  f"[{ctx.last_launch()}]")
            print(f"T={T} cuBLAS addmm fp32-out  {t_cub:.3f} ms  {flops / t_cub / 1e9:.0f} TFLOP/s")
            dW.zero_()
            dW2.zero_()
            ctx.lmhead_dweight(dl, x, out=dW)
            torch.addmm(dW2, dl.t(), x, out_dtype=torch.float32, out=dW2)
            torch.cuda.synchronize()
            print(f"max |diff| vs cuBLAS: {float((dW - dW2).abs().max()):.3e} "
                  f"max |ref| {float(dW2.abs().max()):.3e}")
            dW.zero_()
            dW2.zero_()
        if "--dhidden" in flags or "--only-dhidden" in flags:
            w = (torch.randn((V, H), device="cuda", generator=g) * 0.02).to(torch.bfloat16)
            wt = torch.nn.functional.pad(w.t().contiguous(), (0, w_ld - V))[:, :V]
            dh = torch.empty((T, H), dtype=torch.bfloat16, device="cuda")
            t_dh = timeit(lambda: ctx.lmhead_dhidden(dl, wt, out=dh))
            t_dhc = timeit(lambda: torch.mm(dl, w, out=dh))
            print(f"T={T} dhidden tcgen05 pair    {t_dh:.3f} ms  {flops / t_dh / 1e9:.0f} TFLOP/s")
            print(f"T={T} dhidden cuBLAS mm       {t_dhc:.3f} ms  {flops / t_dhc / 1e9:.0f} TFLOP/s")
            del w, wt, dh


if __name__ == "__main__":
    main()
