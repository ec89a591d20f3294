"""Summarise a profiling run (profiles/run_profile.sh output in gpurun_out/)
into committed, reviewable files under profiles/:

  <tag>_launches.csv     kernel, launches, total/avg device time, share of the
                         bench command (ncu --metrics gpu__time_duration.sum)
  <tag>_ncu_<kernel>.txt key metrics + stall breakdown of one `ncu --set full`
                         capture per kernel
  ncu_traffic.json       dram bytes per row of the top kernel (read by bench.py
                         for roofline.traffic)

usage: python profiles/summarize.py <tag> [gpurun_out] [dest_dir]
(dest_dir defaults to profiles/; round_check.sh summarises on the GPU box into
gpurun_out/profiles_<tag>/ because the raw .ncu-rep files are too large to ship back)
"""
import collections
import csv
import json
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))

KEYS = ["gpu__time_duration.sum", "sm__cycles_active.avg",
        "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__bytes.sum.per_second", "launch__grid_size", "launch__block_size",
        "launch__registers_per_thread", "launch__cluster_dim_x", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "lts__t_sector_hit_rate.pct", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]


def launches(src, dst):
    rows = list(csv.reader(open(src)))
    start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
    hdr = rows[start]
    ix = {h: j for j, h in enumerate(hdr)}
    tot, cnt = collections.defaultdict(float), collections.Counter()
    for r in rows[start + 1:]:
        if len(r) < len(hdr):
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("void ", "")
        tot[name] += float(r[ix["Metric Value"]].replace(",", ""))
        cnt[name] += 1
    s = sum(tot.values())
    with open(dst, "w") as f:
        f.write("kernel,launches,total_ns,avg_ns,share\n")
        for k, v in sorted(tot.items(), key=lambda x: -x[1]):
            f.write(f"\"{k}\",{cnt[k]},{v:.0f},{v / cnt[k]:.0f},{v / s:.4f}\n")


def ncu_summary(rep, dst_prefix, rows_per_launch):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    hdr, units = rows[0], rows[1]
    out = {}
    for r in rows[2:]:
        name = r[hdr.index("Kernel Name")]
        short = name.replace("(anonymous namespace)::", "").split("(")[0].split("<")[0]
        short = short.split("::")[-1].replace("void ", "").strip()
        if short == "fused_pair_kernel" and "<" in name:
            # fused_pair_kernel<F32, CL, BST, PW>: CL = 1 is the solo kernel
            targs = [a.strip() for a in name.split("<", 1)[1].split(">")[0].split(",")]
            if len(targs) >= 2 and targs[1] == "1":
                short = "fused_solo_kernel"
            elif len(targs) >= 2 and targs[1] == "4":
                short = "fused_quad_kernel"
        lines = [f"kernel: {name}"]
        for k in KEYS:
            if k in hdr:
                lines.append(f"{k:70s} {r[hdr.index(k)]} {units[hdr.index(k)]}")
        stalls = []
        for i, h in enumerate(hdr):
            if "warps_issue_stalled" in h and "not_issued" not in h:
                try:
                    stalls.append((float(r[i].replace(",", "")), h.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(v for v, _ in stalls) or 1.0
        lines.append("stall samples: " + ", ".join(f"{h}={100 * v / tot:.1f}%" for v, h in
                                                   sorted(stalls, reverse=True)[:10]))
        rd = float(r[hdr.index("dram__bytes_read.sum")].replace(",", ""))
        wr = float(r[hdr.index("dram__bytes_write.sum")].replace(",", ""))
        scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
        rd *= scale.get(units[hdr.index("dram__bytes_read.sum")], 1.0)
        wr *= scale.get(units[hdr.index("dram__bytes_write.sum")], 1.0)
        lines.append(f"dram bytes per row (read+write) over {rows_per_launch} rows: "
                     f"{(rd + wr) / rows_per_launch:.0f}")
        out[short] = (rd + wr) / rows_per_launch
        with open(f"{dst_prefix}_{short}.txt", "w") as f:
            f.write("\n".join(lines) + "\n")
    return out


def main():
    global HERE
    tag = sys.argv[1]
    src = sys.argv[2] if len(sys.argv) > 2 else os.path.join(os.path.dirname(HERE), "gpurun_out")
    if len(sys.argv) > 3:
        HERE = sys.argv[3]
        os.makedirs(HERE, exist_ok=True)
    if os.path.exists(os.path.join(src, "launches.csv")):
        launches(os.path.join(src, "launches.csv"), os.path.join(HERE, f"{tag}_launches.csv"))
    traffic = {}
    rows = 8192  # run_profile.sh captures with --chunk-rows 8192
    if os.path.exists(os.path.join(src, "prof_fused.ncu-rep")):
        t = ncu_summary(os.path.join(src, "prof_fused.ncu-rep"), os.path.join(HERE, f"{tag}_ncu"), rows)
        for k, v in t.items():
            traffic["grpo_128x8_v151936"] = {"dram_bytes_per_row": v, "kernel": k,
                                             "source": f"profiles/{tag}_ncu_{k}.txt"}
    if os.path.exists(os.path.join(src, "prof_fused_f32.ncu-rep")):
        # the same kernel writing f32 dlogits (parity mode, 6V+16 B/token)
        t = ncu_summary(os.path.join(src, "prof_fused_f32.ncu-rep"), os.path.join(HERE, f"{tag}_ncu_f32"), rows)
        for k, v in t.items():
            traffic["grpo_128x8_v151936:f32"] = {"dram_bytes_per_row": v, "kernel": k,
                                                 "source": f"profiles/{tag}_ncu_f32_{k}.txt"}
    if os.path.exists(os.path.join(src, "prof_unfused.ncu-rep")):
        # K1 (the fused kernel in gather-only mode) and K3 of one chunk
        t = ncu_summary(os.path.join(src, "prof_unfused.ncu-rep"), os.path.join(HERE, f"{tag}_ncu_unfused"), rows)
        if t:
            traffic["unfused:grpo_128x8_v151936"] = {"dram_bytes_per_row": sum(t.values()),
                                                     "kernel": "+".join(t),
                                                     "source": "sum of the unfused kernels"}
    if os.path.exists(os.path.join(src, "prof_tma.ncu-rep")):
        # V = 32,000 (configs[4]); run_profile.sh captures with --chunk-rows 16384
        t = ncu_summary(os.path.join(src, "prof_tma.ncu-rep"), os.path.join(HERE, f"{tag}_ncu"), 16384)
        for k, v in t.items():
            for cfg in ("grpo_128x8_v32000_L256", "grpo_128x8_v32000_L512", "grpo_128x8_v32000_L1024",
                        "grpo_128x8_v32000_L2048", "grpo_128x8_v32000_L4096"):
                traffic[cfg] = {"dram_bytes_per_row": v, "kernel": k,
                                "source": f"profiles/{tag}_ncu_{k}.txt (V = 32,000, 16384-row launch)"}
    if os.path.exists(os.path.join(src, "prof_lmhead.ncu-rep")):
        ncu_summary(os.path.join(src, "prof_lmhead.ncu-rep"), os.path.join(HERE, f"{tag}_ncu"), 4096)
    if os.path.exists(os.path.join(src, "prof_lmhead_dw.ncu-rep")):
        # LM-head backward dW (MN-major operands), T = 4096 tokens
        ncu_summary(os.path.join(src, "prof_lmhead_dw.ncu-rep"), os.path.join(HERE, f"{tag}_ncu_dw"), 4096)
    if traffic:
        # merge into the committed table: a partial capture keeps the other entries
        path = os.path.join(HERE, "ncu_traffic.json")
        try:
            with open(path) as f:
                old = json.load(f)
        except (OSError, ValueError):
            old = {}
        old.update(traffic)
        with open(path, "w") as f:
            json.dump(old, f, indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
