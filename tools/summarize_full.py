"""Key metrics + warp-stall breakdown of every kernel in `ncu --set full`
captures, as markdown (for profiles/). Usage: python tools/summarize_full.py rep..."""
import collections
import csv
import io
import subprocess
import sys

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "dram read"),
        ("dram__bytes_write.sum", "dram write"),
        ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "dram % of peak"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % of peak"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "tensor pipe %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__grid_size", "grid"), ("launch__registers_per_thread", "regs")]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return [(dict(zip(hdr, r)), dict(zip(hdr, units))) for r in data]


def stalls(rep, i):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                          "--launch-skip", str(i), "--launch-count", "1"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hi = [k for k, r in enumerate(rows) if r and r[0] == "Address"]
    if not hi:
        return "", 0
    hdr = rows[hi[0]]
    cols = [(k, h[6:]) for k, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
    agg = collections.Counter()
    n = 0
    for r in rows[hi[0] + 1:]:
        if len(r) < len(hdr):
            continue
        n += 1
        for k, h in cols:
            try:
                agg[h] += float(r[k] or 0)
            except ValueError:
                pass
    tot = sum(agg.values()) or 1
    return ", ".join(f"{k} {v / tot:.0%}" for k, v in agg.most_common(4)), n


def main():
    for rep in sys.argv[1:]:
        print(f"### `{rep.split('/')[-1]}`\n")
        for i, (m, u) in enumerate(raw(rep)):
            name = m.get("Kernel Name", "?")
            print(f"**{name[:90]}**\n")
            for k, label in KEYS:
                if k in m:
                    print(f"- {label}: {m[k]} {u.get(k, '')}".rstrip())
            st, n = stalls(rep, i)
            print(f"- SASS instructions: {n}; top warp-stall reasons (sampled): {st}\n")


if __name__ == "__main__":
    main()
