#!/usr/bin/env python
"""bench.py — BASELINE.json metric: "IS-corrected loss fwd+bwd tokens/sec & %
HBM roofline at 1/2/4/8 B200 vs CPU".

One step = one pass of the hot path over one synthetic GRPO batch
(BASELINE.json configs[1]: 128 prompts x 8 responses, lognormal lengths up to
8k, vocab 151,936, 2 rollout stages): for every chunk of packed rows the fused
kernel (log-softmax + gather, cross-stage behaviour select, ratio/clip, token
mean, dlogits) and then the deterministic reduction (+ NCCL allreduce of four
fp64 scalars when sharded). Inputs are resident in HBM when the timed region
starts; the logits chunk buffer (chunk_rows x V bf16, ~10 GB) is far larger
than L2. Weak scaling: each rank holds 128 x 8 prompts' worth of whole groups
(LPT over token counts), T_global is known on the host.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--impl reference runs the reference's own CPU path (oracle/_ref/libcopris_ref.so,
compiled from /root/reference's headers) on the host cores, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "IS-corrected loss fwd+bwd tokens/sec & % HBM roofline at 1/2/4/8 B200 vs CPU"
UNIT = "tokens/s"


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="grpo_128x8_v151936")
    ap.add_argument("--chunk-rows", type=int, default=32768)
    ap.add_argument("--unfused", action="store_true", help="K1 -> K2 -> K3 instead of the fused kernel")
    ap.add_argument("--vocab", type=int, default=None,
                    help="override the config's vocabulary (a vocabulary sweep; not a BASELINE config)")
    ap.add_argument("--dlogits", choices=["bf16", "f32"], default="bf16",
                    help="f32: the parity mode (dlogits within 1e-5; 6V+16 B/token)")
    ap.add_argument("--entropy-coeff", type=float, default=0.0,
                    help="grpo.entropy_coeff (grpo.hpp:168-181); the headline configs use 0 (desk.json)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--e2e-tokens", type=int, default=16384, help="per-rank sample for the host round trip")
    ap.add_argument("--e2e-chunk", type=int, default=512)
    ap.add_argument("--cpu-tokens-per-thread", type=int, default=256)
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--graph-steps", type=int, default=1,
                    help="with --graph: steps captured back to back in one graph (a training loop's "
                         "consecutive small steps; N=1 only); --steps must be a multiple")
    ap.add_argument("--graph", action="store_true",
                    help="capture one step (all chunk launches + the reduction) in a CUDA graph "
                         "and replay it; the allreduce stays outside the graph")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md recipe)
# ---------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("pci.bus_id,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
    LOAD_W = 400.0  # a sample counts as "under load" at or above this board power

    def __init__(self, bus_id: str | None):
        self.bus = (bus_id or "").upper()
        self.rows = []
        self.proc = None
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (OSError, ValueError):
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()
        time.sleep(0.3)

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != 8:
                continue
            if self.bus and not parts[0].upper().endswith(self.bus[-12:]):
                continue
            self.rows.append(parts)

    def stop(self):
        if not self.proc:
            return None
        time.sleep(0.3)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if r[4 + i].lower().startswith("active")})
        pw = [float(r[3]) for r in self.rows if r[3].replace(".", "").isdigit()]
        out = {"sm_mhz": statistics.median(sm) if sm else None,
               "sm_max_mhz": max(mx) if mx else None, "reasons": reasons, "samples": len(self.rows),
               "power_w": statistics.median(pw) if pw else None}
        # samples under load only (a sampler that also covers setup phases)
        load = [(float(r[1]), float(r[3])) for r in self.rows
                if r[1].replace(".", "").isdigit() and r[3].replace(".", "").isdigit()
                and float(r[3]) >= self.LOAD_W]
        if load and len(load) < len(self.rows):
            out["under_load"] = {"samples": len(load), "sm_mhz": statistics.median(a for a, _ in load),
                                 "power_w": statistics.median(b for _, b in load)}
        return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback (B200_PROFILING.md)"


def traffic_per_row(config, unfused, kernel, dlogits="bf16"):
    """dram bytes per row of the top kernel from the committed ncu capture
    (profiles/ncu_traffic.json, written from an `ncu --set full` run); None
    unless that capture is of the kernel this run launched."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            t = json.load(f)
        key = ("unfused:" if unfused else "") + config + (":f32" if dlogits == "f32" else "")
        rec = t[key]
        if not unfused and kernel not in rec["kernel"]:
            return None
        return float(rec["dram_bytes_per_row"])
    except (OSError, KeyError, ValueError):
        return None


# ---------------------------------------------------------------------------
# CPU: the reference's own path (oracle/_ref) on the host cores
# ---------------------------------------------------------------------------
def pcie_probe(h_src, h_dst, d_dst, d_src, reps=3):
    """Pinned host<->device copy rates on this box (GB/s): H2D alone, D2H alone,
    and both at once on two streams (the e2e pipeline's situation). Wall clock
    around synchronised copies of ~GBs, so launch overhead is negligible."""
    import torch
    n = min(h_src.shape[0], h_dst.shape[0], d_dst.shape[0], d_src.shape[0])
    nb = n * h_src.shape[1] * h_src.element_size()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def timed(h2d, d2h):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            if h2d:
                with torch.cuda.stream(s1):
                    d_dst[:n].copy_(h_src[:n], non_blocking=True)
            if d2h:
                with torch.cuda.stream(s2):
                    h_dst[:n].copy_(d_src[:n], non_blocking=True)
        torch.cuda.synchronize()
        return reps * nb / (time.perf_counter() - t0) / 1e9

    timed(True, True)
    return {"h2d_gbs": timed(True, False), "d2h_gbs": timed(False, True),
            "duplex_gbs_each_way": timed(True, True), "bytes_per_copy": nb}


def cpu_reference(V, tokens_per_thread, seconds, seed, threads=None, min_rounds=1, max_rounds=None):
    """Times the UNMODIFIED reference hot path (sequence_logprobs ->
    concat_segments -> grpo_step_loss, compiled from /root/reference) with one
    independent batch per host thread, like the reference CLI's
    --parallel-seeds (copris_cli.cpp:98-115). Returns (tok/s, details)."""
    import numpy as np
    from oracle.oracle import Oracle, Reference

    kind = "reference" if Reference.available else "port"
    impl = Reference() if Reference.available else Oracle()
    threads = threads or os.cpu_count() or 1
    rng = np.random.default_rng(seed)
    L = tokens_per_thread
    target = rng.integers(0, V, L).astype(np.int32)
    z = rng.standard_normal((L, V)).astype(np.float32).astype(np.float64) * 2.0
    z[np.arange(L), target] += 4.0
    tok_off = np.array([0, L // 2, L], np.int64)          # one group of two trajectories
    stage = np.full(L, 7, np.uint32)
    stage[: L // 4] = 6                                   # a stale first segment
    cur = Oracle().logprob_gather(z[: L // 4], target[: L // 4]) if kind == "port" else None
    blp = np.zeros(L, np.float64)
    blp[: L // 4] = (cur if cur is not None else -12.0) + rng.uniform(-0.3, 0.3, L // 4)
    adv = np.array([1.0, -1.0])
    tokens = 0
    rounds = 0
    ref_time = 0.0  # sum over rounds of the slowest thread's time inside the reference path
    t_start = time.perf_counter()

    while True:
        secs = [0.0] * threads

        def work(i):
            secs[i] = impl.is_loss(z, tok_off, target, stage, 7, blp, adv, want_dlogits=True).seconds

        ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        rounds += 1
        tokens += threads * L
        ref_time += max(secs)
        if (time.perf_counter() - t_start >= seconds and rounds >= min_rounds) or \
                (max_rounds and rounds >= max_rounds):
            break
    wall = ref_time
    try:
        model = open("/proc/cpuinfo").read().split("model name")[1].split(":")[1].split("\n")[0].strip()
    except (OSError, IndexError):
        model = "unknown"
    return tokens / wall, {
        "kind": kind, "cores": threads, "cpu_model": model,
        "sample": f"{rounds} rounds x {threads} threads x {L} tokens (1 group of 2 trajectories, "
                  f"2 stages) at V={V}; {wall:.2f}s inside the reference path (slowest thread "
                  f"per round; table construction excluded)",
    }


def run_reference(args):
    """--impl reference: rank 0 alone times the reference CPU path."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2511_05589_b200.workload import CONFIGS, describe
    cfg = CONFIGS[args.config]
    V = cfg["vocab"]
    # warmup + steps: each step one bounded sample (all threads once)
    per_step = []
    det = None
    for i in range(args.warmup + args.steps):
        tps, det = cpu_reference(V, args.cpu_tokens_per_thread, 0.0, args.seed + i, max_rounds=1)
        if i >= args.warmup:
            per_step.append(tps)
    value = statistics.mean(per_step)
    tok_step = det["cores"] * args.cpu_tokens_per_thread
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1000.0 * tok_step / value, "higher_is_better": True,
        "scaling": "strong" if cfg.get("strong") else "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{describe(args.config)} — bounded CPU sample",
                   "vocab": V, "tokens_per_step": tok_step},
        "cpu_baseline": {"value": value, "unit": UNIT, **det},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# ours
# ---------------------------------------------------------------------------
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2511_05589_b200 import ClipConfig, Copris
    from paper_2511_05589_b200.grpo import HostWorkspace
    from paper_2511_05589_b200.packing import upload
    from paper_2511_05589_b200.sharding import allreduce_scalars, lpt_shard, shard_arrays
    from paper_2511_05589_b200.workload import (CONFIGS, describe, make_host_batch, make_logits,
                                                 stale_logprobs)

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        # never print a line whose n_gpus differs from the requested N
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    # control-flow rehearsal of the multi-rank path on a single GPU (not a
    # measurement): COPRIS_BENCH_ONE_GPU=1 puts every rank on cuda:0 and
    # COPRIS_BENCH_BACKEND=gloo replaces NCCL (which refuses shared devices)
    if os.environ.get("COPRIS_BENCH_ONE_GPU"):
        local = 0
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    comm = {"backend": None, "world_size": 1}
    if world > 1:
        backend = os.environ.get("COPRIS_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
        # the communicator's own rank count (what the allreduce runs over)
        probe = torch.ones(1, dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(probe)
        comm = {"backend": dist.get_backend(), "world_size": dist.get_world_size(),
                "ranks_in_allreduce": int(probe.item())}
        if comm["world_size"] != args.gpus or comm["ranks_in_allreduce"] != args.gpus:
            raise SystemExit(f"bench.py: communicator has {comm} ranks, --gpus {args.gpus}")

    cfgd = dict(CONFIGS[args.config])
    if args.vocab:
        cfgd["vocab"] = args.vocab
    V = cfgd["vocab"]
    strong = cfgd.pop("strong", False)
    P_cfg = cfgd.pop("P")
    P_global = P_cfg if strong else P_cfg * world   # strong: one global batch, sharded
    G = cfgd.pop("G")
    cfgd.pop("vocab")
    hb = make_host_batch(args.seed, P_global, G, V, **cfgd)
    shards = lpt_shard(hb.group_tokens(), world)
    tok_off, group_off, pt, pj, _ = shard_arrays(hb.tok_off, hb.group_off, {"stage": hb.stage},
                                                 {"reward": hb.reward}, shards[rank])
    stage, reward = pt["stage"], pj["reward"]
    T_global, T = hb.n_tok, int(tok_off[-1])
    chunk = min(args.chunk_rows, T)
    nchunks = (T + chunk - 1) // chunk

    ctx = Copris(local)
    clip = ClipConfig(entropy_coeff=args.entropy_coeff)
    # resident logits chunk buffer; token t of the local batch reads buffer row
    # t % chunk, whose target column is the boosted one.
    g = torch.Generator(device="cpu")
    g.manual_seed(args.seed + rank)
    tbuf = torch.randint(0, V, (chunk,), generator=g, dtype=torch.int64).to(torch.int32)
    logits = make_logits(chunk, V, tbuf.to(dev), args.seed + rank, device=dev, dtype=torch.bfloat16)
    target = tbuf.numpy()[np.arange(T) % chunk]
    cur_buf, _ = ctx.sequence_logprobs(logits, tbuf.to(dev))
    torch.cuda.synchronize()
    cur = cur_buf.cpu().numpy()[np.arange(T) % chunk]
    blp = stale_logprobs(cur, stage, hb.cur_stage, args.seed + rank)
    del cur
    batch = upload(ctx, tok_off, group_off, target, blp, hb.cur_stage, stage=stage, reward=reward)
    outs = ctx.alloc_outputs(T, dev, lse=args.unfused, behav=args.unfused)
    dl = torch.empty((chunk, V), dtype=torch.float32 if args.dlogits == "f32" else torch.bfloat16,
                     device=dev)
    out4 = torch.zeros(4, dtype=torch.float64, device=dev)
    run_chunk = ctx.loss_chunk_unfused if args.unfused else ctx.loss_chunk_fused

    def launches(evs=None):
        for c in range(nchunks):
            r0 = c * chunk
            n = min(chunk, T - r0)
            if evs is not None:
                evs[c][0].record()
            # the last chunk carries out4: the reduction rides along (inside
            # the loss launch when the step is small, else right behind it)
            run_chunk(logits[:n], batch, clip, outs, dlogits=dl[:n], row_base=r0,
                      total_tokens=T_global, out4=out4 if c == nchunks - 1 else None)
            if evs is not None:
                evs[c][1].record()

    graph = None

    gsteps = max(1, args.graph_steps) if args.graph else 1
    if gsteps > 1 and (world > 1 or args.steps % gsteps):
        raise SystemExit("bench.py: --graph-steps needs N=1 and --steps a multiple of it")

    def step(evs=None):
        torch.cuda.nvtx.range_push("copris step")
        if graph is not None:
            graph.replay()
        else:
            launches(evs)
        allreduce_scalars(out4)
        torch.cuda.nvtx.range_pop()

    for _ in range(max(args.warmup, 1)):
        step()
    ctx.check()
    info = ctx.last_launch()
    fused_reduce = bool(info.get("fused_reduce")) and not args.unfused
    if args.graph:
        # CUDA graph of one step: the per-launch host cost (Python + C-ABI)
        # leaves the loop; replays are bitwise identical to eager steps
        graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(side):
            launches()
        torch.cuda.current_stream().wait_stream(side)
        with torch.cuda.graph(graph):
            for _ in range(gsteps):  # whole steps back to back (each ends with its reduction)
                launches()
        for _ in range(max(args.warmup, 1)):
            step()
        ctx.check()

    evs = [[[torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)]
            for _ in range(nchunks)] for _ in range(args.steps)]
    bus = None
    try:
        p = torch.cuda.get_device_properties(local)
        bus = f"{p.pci_bus_id:02X}:{p.pci_device_id:02X}.0"
    except Exception:
        pass
    sampler = ClockSampler(bus)
    sampler.start()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for k in range(args.steps // gsteps):
        step(evs[k])
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = sampler.stop()
    if world > 1:
        # every rank sampled its own GPU over the same timed region: rank 0
        # reports all of them (reasons are the union; sm_mhz the lowest rank's
        # median, the clock the max-over-ranks time was set by)
        per_rank = [None] * world
        dist.all_gather_object(per_rank, clocks)
        ok = [c for c in per_rank if c and c.get("sm_mhz") is not None]
        if ok:
            clocks = dict(min(ok, key=lambda c: c["sm_mhz"]))
            clocks["reasons"] = sorted({x for c in ok for x in c["reasons"]})
            clocks["per_rank"] = [{k: c.get(k) for k in ("sm_mhz", "reasons", "power_w", "samples")}
                                  if c else None for c in per_rank]
            clocks["busy_gpus"] = sum(1 for c in ok if (c.get("under_load") or {}).get("samples", 0) > 0
                                      or (c.get("power_w") or 0.0) >= ClockSampler.LOAD_W)
    ctx.check()
    ms = e0.elapsed_time(e1) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = t.item()
    loss = -out4[0].item() * (1.0 / T_global)

    # kernel-level roofline (dominant kernel: the fused pass); under --graph
    # the per-chunk events are not recorded and the whole step is charged
    if graph is None:
        kern_ms = sum(evs[k][c][0].elapsed_time(evs[k][c][1]) for k in range(args.steps)
                      for c in range(nchunks))
    else:
        kern_ms = ms * args.steps
    rows_timed = args.steps * T
    bytes_per_tok = (6 if args.dlogits == "f32" else 4) * V + 16
    achieved = rows_timed * bytes_per_tok / (kern_ms / 1e3) / 1e9
    peak, peak_src = measured_peaks()
    tr = None if args.vocab or args.entropy_coeff else traffic_per_row(args.config, args.unfused, info.get("kernel", ""), args.dlogits)

    line = None
    if rank == 0:
        value = T_global / (ms_max / 1e3)
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
            "scaling": "strong" if strong else "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic",
            "config": {
                "workload": describe(args.config) + (f" [vocab overridden: {V}]" if args.vocab else ""),
                "prompts": P_global, "responses": G, "vocab": V, "tokens_global": T_global,
                "tokens_rank0": T, "chunk_rows": chunk, "chunks_per_step": nchunks,
                "parallelism": f"dp{world} (whole prompt groups, LPT by tokens)",
                "path": ("unfused K1->K2->K3" if args.unfused else "fused single pass")
                        + ((" (CUDA graph replay" + (f", {gsteps} steps per graph)" if gsteps > 1 else ")"))
                           if graph is not None else ""),
                "kernel": info, "l2": (f"inputs larger than L2: each step streams {T * V * 2 / 1e6:.0f} MB "
                                       f"of logits and writes as much dlogits (chunk buffer "
                                       f"{chunk * V * 2 / 1e6:.0f} MB; L2 126 MB); no flush"),
                "loss": loss,
                **({"entropy_coeff": args.entropy_coeff} if args.entropy_coeff else {}),
                "offpolicy_fraction": out4[2].item() / out4[1].item() if out4[1].item() else 0.0,
                "clipped_tokens": int(out4[3].item()),
                "dlogits": ("f32 (parity mode: within 1e-5; 6V+16 B/token)" if args.dlogits == "f32"
                            else "bf16 (within 2^-7 relative; 4V+16 B/token)"),
            },
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_source": peak_src,
                         "traffic": (tr * T / nchunks) if tr else None,
                         "algorithmic_bytes_per_token": bytes_per_tok,
                         "kernel_ms_per_step": kern_ms / args.steps,
                         "frac_of_8TBs_nominal": achieved / 8000.0},
            "comm": comm,
            "gpu_launches": args.steps * (nchunks * (3 if args.unfused else 1)
                                          + (0 if fused_reduce else 1)),
            "clocks": clocks,
        }

    # e2e: the host-buffer drop-in (copris_grpo_step_loss_host) on a bounded
    # sample of this rank's batch: pinned host logits + metadata in, host
    # dlogits + loss out, host<->device copies inside the timed region.
    if not args.no_e2e:
        # whole trajectories from the front of the batch, at least e2e_tokens;
        # the pinned host buffers (logits in, dlogits out: 4V bytes per token)
        # of all ranks together stay under ~48 GB of host memory
        e2e_tokens = min(args.e2e_tokens, max(2048, int(48e9 // (4 * V)) // world))
        n_tr = int(np.searchsorted(tok_off, min(e2e_tokens, T), side="left"))
        n_tr = min(max(1, n_tr), len(tok_off) - 1)
        Ts = int(tok_off[n_tr])
        s_tok_off = torch.from_numpy(tok_off[: n_tr + 1].copy()).pin_memory()
        s_target = torch.from_numpy(target[:Ts].copy()).pin_memory()
        s_stage = torch.from_numpy(stage[:Ts].view(np.int32).copy()).pin_memory()
        s_blp = torch.from_numpy(blp[:Ts].copy()).pin_memory()
        # group advantages of the full batch (a sample may cut a group)
        s_adv = batch.adv[:n_tr].cpu().pin_memory()
        h_logits = torch.empty((Ts, V), dtype=torch.bfloat16).pin_memory()
        for a in range(0, Ts, chunk):
            b = min(Ts, a + chunk)
            h_logits[a:b].copy_(logits[: b - a])
        h_dl = torch.empty((Ts, V), dtype=torch.bfloat16).pin_memory()
        ws = HostWorkspace(ctx, min(args.e2e_chunk, Ts), V, Ts, n_tr)
        call = lambda: ws.grpo_step_loss(h_logits, s_tok_off, s_target, s_stage, s_blp,
                                         hb.cur_stage, adv=s_adv, cfg=clip, total_tokens=0,
                                         dlogits=h_dl)
        call()
        e2e_steps = max(1, min(args.steps, 5))
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            res = call()
        el = (time.perf_counter() - t0) / e2e_steps
        te = torch.tensor([el, Ts], dtype=torch.float64, device=dev)
        if world > 1:
            tmax = te[:1].clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            tsum = te[1:].clone()
            dist.all_reduce(tsum)
            el, Ts_all = tmax.item(), tsum.item()
        else:
            Ts_all = Ts
        h2d = Ts * V * 2 + Ts * 12 + (n_tr + 1) * 8 + n_tr * 8
        d2h = Ts * V * 2 + 32
        if line is not None:
            line["e2e"] = {"value": Ts_all / el, "unit": UNIT, "h2d_bytes_per_step": h2d,
                           "d2h_bytes_per_step": d2h,
                           "api": "copris_grpo_step_loss_host (host pinned buffers, 3-stream chunked pipeline)",
                           "sample": f"first {n_tr} trajectories ({Ts} tokens) of each rank's batch, "
                                     f"{e2e_steps} timed calls", "loss": res["loss"],
                           "bound": (f"PCIe: host bf16 logits in and host dlogits out, {2 * V} B per token "
                                     f"each way; the per-token cost does not depend on the sample size, "
                                     f"so the sample's tok/s is the config's")}
            if world == 1 and args.dlogits == "bf16":
                pc = pcie_probe(h_logits, h_dl, dl, logits)
                e2e_gbs = Ts_all / el * 2 * V / 1e9
                line["e2e"]["pcie"] = {**pc, "e2e_gbs_each_way": e2e_gbs,
                                       "frac_of_duplex": e2e_gbs / pc["duplex_gbs_each_way"]}
        ws.close()
        del h_logits, h_dl

    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        tps, det = cpu_reference(V, args.cpu_tokens_per_thread, args.cpu_seconds, args.seed)
        line["cpu_baseline"] = {"value": tps, "unit": UNIT, **det}
        # the reference as it runs in its own trainer: ONE thread (grpo.hpp:113-115,
        # SURVEY.md §8(d) CPU baseline (i)); the full-batch step time is extrapolated
        tps1, det1 = cpu_reference(V, args.cpu_tokens_per_thread, min(4.0, args.cpu_seconds), args.seed,
                                   threads=1, min_rounds=2)
        line["cpu_baseline"]["single_thread"] = {
            "value": tps1, "unit": UNIT, "sample": det1["sample"],
            "extrapolated_step_s": T_global / tps1,
            "extrapolated_step": f"{T_global} tokens / {tps1:.0f} tok/s = {T_global / tps1 / 3600:.2f} h "
                                 f"for one {args.config} step on one core"}
    if line is not None:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()


def relaunch_under_torchrun(args) -> int:
    """`python bench.py --gpus N` (N > 1) outside torchrun: start the N ranks
    here, one process per GPU, exactly as the driver's torchrun launch would
    (127.0.0.1 rendezvous on a free port); rank 0 prints the line."""
    import socket
    import torch
    n_dev = torch.cuda.device_count()
    if args.impl == "ours" and n_dev < args.gpus and not os.environ.get("COPRIS_BENCH_ONE_GPU"):
        print(f"bench.py: --gpus {args.gpus} needs {args.gpus} visible GPUs, found {n_dev}",
              file=sys.stderr)
        return 2
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    args = parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_under_torchrun(args))
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
