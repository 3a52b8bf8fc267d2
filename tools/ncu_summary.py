"""Summarise an ncu launch list + a --set full k_stats capture into profiles/ (committed evidence).

  python tools/ncu_summary.py r01            (reads gpurun_out/r01_launches.csv, gpurun_out/r01_kstats.ncu-rep)
"""
import collections
import csv
import json
import os
import subprocess
import sys

tag = sys.argv[1] if len(sys.argv) > 1 else "r01"
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
g = os.path.join(root, "gpurun_out")
out_dir = os.environ.get("NCU_SUMMARY_OUT", os.path.join(root, "profiles"))
os.makedirs(out_dir, exist_ok=True)

# ---- launch list: per-kernel share of device time (cold-cache, serialised: shares, not absolutes)
rows = list(csv.reader(open(os.path.join(g, f"{tag}_launches.csv"))))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
per = collections.defaultdict(list)
order = []
for r in rows[start + 1:]:
    name = r[ki].split("(")[0]
    val = float(r[vi].replace(",", ""))
    val = val * {"ns": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "ms": 1e3}.get(r[ui], 1.0)
    per[name].append(val)
    order.append((name, val))
tot = sum(sum(v) for v in per.values())
with open(os.path.join(out_dir, f"{tag}_launch_list.md"), "w") as f:
    f.write(f"# {tag}: ncu launch list (gpu__time_duration.sum, --clock-control none)\n\n")
    f.write("Command: `ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv "
            "python bench.py --steps 3 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0` "
            "(C4: 4096 frames x 5000 descriptors, K=256, D=64, tau=1e-6).  Serialised and cold-cache: compare shares.\n\n")
    f.write("| kernel | launches | mean us | total us | share |\n|---|---|---|---|---|\n")
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        f.write(f"| {k} | {len(v)} | {sum(v)/len(v):.1f} | {sum(v):.1f} | {100*sum(v)/tot:.1f}% |\n")
    f.write("\nLaunch order:\n\n")
    for name, val in order:
        f.write(f"- {name}: {val:.1f} us\n")

# ---- full captures: headline metrics, pipe shares, stall reasons
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "smsp__mem_tensor_reads_op_ldt.sum.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__cluster_size", "sm__cycles_elapsed.avg", "sm__warps_active.avg.pct_of_peak_sustained_active"]


def capture(name, title, cmd):
    rep = os.path.join(g, f"{tag}_{name}.ncu-rep")
    if not os.path.exists(rep):
        return None
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, u, v = r[0], r[1], r[2]
    vals = {w: (v[h.index(w)], u[h.index(w)]) for w in WANT if w in h}
    stalls = []
    for i, nm in enumerate(h):
        if nm.startswith("smsp__pcsamp_warps_issue_stalled_") and not nm.endswith("not_issued"):
            try:
                stalls.append((float(v[i]), nm[len("smsp__pcsamp_warps_issue_stalled_"):]))
            except ValueError:
                pass
    tot = sum(x for x, _ in stalls) or 1.0

    def tobytes(val, unit):
        return float(val.replace(",", "")) * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
    dram = None
    if "dram__bytes_read.sum" in vals and "dram__bytes_write.sum" in vals:
        dram = tobytes(*vals["dram__bytes_read.sum"]) + tobytes(*vals["dram__bytes_write.sum"])
    with open(os.path.join(out_dir, f"{tag}_{name}_ncu.md"), "w") as f:
        f.write(f"# {tag}: {title}, ncu --set full --clock-control none (one launch)\n\nCommand: `{cmd}`\n\n")
        f.write("| metric | value | unit |\n|---|---|---|\n")
        for w in WANT:
            if w in vals:
                f.write(f"| {w} | {vals[w][0]} | {vals[w][1]} |\n")
        if dram is not None:
            f.write(f"\nDRAM traffic per launch: {dram/1e9:.3f} GB (read + write).\n")
        f.write("\nWarp stall reasons (share of PC samples):\n\n")
        for x, nm in sorted(stalls, reverse=True)[:10]:
            f.write(f"- {nm}: {100*x/tot:.1f}%\n")
    return dram


NC = "ncu --set full --clock-control none --import-source on"
dram = capture("kstats", "k_stats (narrow, D=64) on C4",
               f"{NC} -k regex:k_stats -s 3 -c 1 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0")
capture("finalize", "k_finalize on C4",
        f"{NC} -k regex:k_finalize -s 3 -c 1 python bench.py --steps 1 --warmup 3 --e2e-steps 0 --no-latency --cpu-seconds 0")
capture("kstats_w", "k_stats_w (wide, D=128, K=512) on a 2M-row C5 set",
        f"{NC} -k regex:k_stats_w -s 3 -c 1 python bench.py --workload c5 --c5-n 2000000 --steps 1 --warmup 3 --e2e-steps 0")
capture("embed", "k_embed (PCA m=80 + xy, 256 frames x 5000 raw descriptors)",
        f"{NC} -k regex:k_embed -s 3 -c 1 python bench.py --workload embed --frames 256 --steps 1 --warmup 3")
n_total = 4096 * 5000
with open(os.path.join(out_dir, "kstats_traffic.json"), "w") as f:
    json.dump({"tag": tag, "n_total": n_total, "dram_bytes_per_launch": dram,
               "source": f"profiles/{tag}_kstats_ncu.md"}, f, indent=1)
print(open(os.path.join(out_dir, f"{tag}_launch_list.md")).read()[:1500])
for nm in ("kstats", "finalize", "kstats_w", "embed"):
    pth = os.path.join(out_dir, f"{tag}_{nm}_ncu.md")
    if os.path.exists(pth):
        print(open(pth).read())
