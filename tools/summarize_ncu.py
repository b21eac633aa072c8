"""Summarise ncu artefacts from gpurun_out/ into profiles/ (committed).

usage: python tools/summarize_ncu.py <round-tag> <launches.csv> <rep:kernel-label> ...
Writes profiles/<tag>_launches.md, profiles/<tag>_<label>.md and updates
profiles/ncu_traffic.json (per-launch DRAM bytes read+write per kernel,
read by bench.py as roofline.traffic)."""
import csv
import io
import json
import os
import subprocess
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PROF = os.path.join(ROOT, "profiles")

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "lts__t_sector_hit_rate.pct", "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
    "sm__cycles_elapsed.avg.per_second",
    "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    return d


def to_bytes(val, unit):
    x = float(val.replace(",", ""))
    return x * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


def launches(tag, path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(list)
    for r in rows[hi + 1:]:
        if len(r) > vi:
            v = float(r[vi].replace(",", ""))
            if r[ui] in ("nsecond", "ns"):
                v /= 1000.0
            elif r[ui] in ("msecond", "ms"):
                v *= 1000.0
            agg[r[ki].split("(")[0][:70]].append(v)
    tot = sum(sum(v) for v in agg.values())
    lines = [f"# {tag}: ncu launch list (`gpu__time_duration.sum --clock-control none`)", "",
             "Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 400 python bench.py --steps 2 --warmup 3 --no-cpu-baseline`.",
             "Cold-cache, serialised per-launch times (compare shares, not absolutes). The list covers",
             "the config-2 device steps, the e2e steps (whose K1 launches are 64-frame chunks) and the",
             "config-3 sub-record (the 1M x 1M x 128 join: band-plan steps, e2e calls and the dense-screen",
             "pass -- the `k_screen<128, ...>`, `k_band_keys<4>`, `k_prep<1, 4>` rows).", "",
             "| kernel | launches | avg us | total us | share |", "|---|---:|---:|---:|---:|"]
    for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |")
    open(os.path.join(PROF, f"{tag}_launches.md"), "w").write("\n".join(lines) + "\n")


def kernel(tag, rep, label):
    d = raw(rep)
    name = d.get("Kernel Name", ("?", ""))[0] if "Kernel Name" in d else "?"
    lines = [f"# {tag}: `{label}` -- ncu --set full summary", "",
             f"Report: `{os.path.basename(rep)}` (one launch, `--clock-control none`).", "",
             "| metric | value | unit |", "|---|---:|---|"]
    for k in KEYS:
        if k in d:
            lines.append(f"| {k} | {d[k][0]} | {d[k][1]} |")
    stalls = {k: float(v[0].replace(",", "") or 0) for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled") and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1
    lines += ["", "Top warp-stall reasons (pc sampling):", ""]
    for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:8]:
        lines.append(f"- {k.replace('smsp__pcsamp_warps_issue_stalled_', '')}: {100*v/tot:.1f}%")
    open(os.path.join(PROF, f"{tag}_{label}.md"), "w").write("\n".join(lines) + "\n")
    rd = to_bytes(*d["dram__bytes_read.sum"]) if "dram__bytes_read.sum" in d else None
    wr = to_bytes(*d["dram__bytes_write.sum"]) if "dram__bytes_write.sum" in d else None
    return (rd or 0) + (wr or 0), name


def main():
    tag, lcsv = sys.argv[1], sys.argv[2]
    os.makedirs(PROF, exist_ok=True)
    launches(tag, lcsv)
    tpath = os.path.join(PROF, "ncu_traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    for spec in sys.argv[3:]:
        rep, label = spec.split(":")
        b, _ = kernel(tag, rep, label)
        traffic[label] = b
    traffic["_source"] = f"{tag}: dram__bytes_read.sum + dram__bytes_write.sum, one ncu --set full launch"
    json.dump(traffic, open(tpath, "w"), indent=1)


if __name__ == "__main__":
    main()
