"""Summarise ncu outputs into profiles/ (markdown): launch-list shares and key
metrics of --set full captures."""
import collections, csv, subprocess, sys, os

def launches(path, steps_hint=None):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h, data = rows[hi], rows[hi + 1:]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    gi = h.index("Grid Size") if "Grid Size" in h else None
    agg = collections.defaultdict(list)
    for r in data:
        agg[(r[ki][:70], r[gi] if gi is not None else "")].append(float(r[vi].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    out = [f"launches: {sum(len(v) for v in agg.values())}, total {tot/1e3:.1f} us (ncu: cold cache, serialised)", "",
           "| share | n | avg us | grid | kernel |", "|---|---|---|---|---|"]
    for (name, grid), v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        out.append(f"| {sum(v)/tot*100:.1f}% | {len(v)} | {sum(v)/len(v)/1e3:.2f} | {grid} | `{name}` |")
    return "\n".join(out)

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
        "smsp__average_warp_latency_issue_stalled_long_scoreboard"]

def full(rep):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        name = r[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        out.append(f"### `{name[:90]}`")
        for k in KEYS:
            if k in h:
                out.append(f"- {k} = {r[h.index(k)]} {units[h.index(k)]}")
    return "\n".join(out)

if __name__ == "__main__":
    tag, dest = sys.argv[1], sys.argv[2]
    parts = [f"# ncu summary ({tag})", ""]
    if os.path.exists("gpurun_out/launches.csv"):
        parts += ["## Launch list of one bench step (`ncu --metrics gpu__time_duration.sum --clock-control none`)", "",
                  launches("gpurun_out/launches.csv"), ""]
    for rep in sorted(p for p in os.listdir("gpurun_out") if p.startswith("prof_") and p.endswith(".ncu-rep")):
        parts += [f"## `ncu --set full` {rep}", "", full(os.path.join("gpurun_out", rep)), ""]
    open(dest, "w").write("\n".join(parts))
    print(dest)
