"""Summarise an ncu per-launch CSV of one decode step (tools/one_step.py under
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum)
into per-kernel-type rows + step totals; writes JSON next to the CSV.
Usage: python tools/step_profile.py profiles/r1_ncu_step_c2.csv"""
import csv
import json
import sys
from collections import OrderedDict

UNITS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0,
         "ms": 1e3, "msecond": 1e3}


def load(path):
    rows = [r for r in csv.reader(open(path)) if r]
    hdr_i = next(i for i, r in enumerate(rows) if "Metric Name" in r)
    hdr = rows[hdr_i]
    ix = {k: hdr.index(k) for k in ("ID", "Kernel Name", "Grid Size", "Metric Name", "Metric Unit", "Metric Value")}
    launches = OrderedDict()
    for r in rows[hdr_i + 1:]:
        if len(r) < len(hdr):
            continue
        d = launches.setdefault(r[ix["ID"]], {"kernel": r[ix["Kernel Name"]], "grid": r[ix["Grid Size"]]})
        v = float(r[ix["Metric Value"]].replace(",", "")) * UNITS.get(r[ix["Metric Unit"]], 1)
        d[r[ix["Metric Name"]]] = v
    return list(launches.values())


def main():
    path = sys.argv[1]
    ls = load(path)
    tot_us = sum(l.get("gpu__time_duration.sum", 0) for l in ls)
    tot_b = sum(l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0) for l in ls)
    kinds = OrderedDict()
    for l in ls:
        k = kinds.setdefault(l["kernel"].split("(")[0], {"n": 0, "us": 0.0, "bytes": 0.0, "grid": l["grid"]})
        k["n"] += 1
        k["us"] += l.get("gpu__time_duration.sum", 0)
        k["bytes"] += l.get("dram__bytes_read.sum", 0) + l.get("dram__bytes_write.sum", 0)
    out = {"launches": len(ls), "sum_us": tot_us, "dram_bytes": tot_b,
           "kinds": [dict(kernel=k, **v, share=v["us"] / tot_us) for k, v in
                     sorted(kinds.items(), key=lambda kv: -kv[1]["us"])]}
    json.dump(out, open(path.rsplit(".", 1)[0] + ".json", "w"), indent=1)
    print(f"{len(ls)} launches, {tot_us:.1f} us summed (serialised, cold), dram {tot_b / 1e6:.1f} MB")
    for k in out["kinds"]:
        print(f"  {k['share']:6.1%} n={k['n']:3d} {k['us'] / k['n']:7.2f} us  {k['bytes'] / k['n'] / 1e6:7.2f} MB  "
              f"{k['grid']:>12}  {k['kernel'][:70]}")


if __name__ == "__main__":
    main()
