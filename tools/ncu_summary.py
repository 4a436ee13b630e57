"""Summarise an ncu launch list (csv) and a --set full report into profiles/.

    python tools/ncu_summary.py <launches.csv> <report.ncu-rep> <out_prefix>
"""

import collections
import csv
import io
import json
import subprocess
import sys


def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    for d in data:
        name = d["Kernel Name"].split("(")[0].replace("void ", "")
        agg.setdefault(name, []).append(float(d["Metric Value"]) / 1e3)
    return agg


def full(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    want = {
        "time_us": "gpu__time_duration.sum",
        "dram_read_B": "dram__bytes_read.sum",
        "dram_write_B": "dram__bytes_write.sum",
        "dram_pct_peak": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
        "regs": "launch__registers_per_thread",
        "fp64_pipe_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smem_bank_conflicts": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    }
    units = rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k, m in want.items():
            if m in hdr:
                v, u = r[hdr.index(m)], units[hdr.index(m)]
                try:
                    v = float(v)
                except ValueError:
                    pass
                if isinstance(v, float):
                    v = v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "us": 1, "ms": 1e3, "ns": 1e-3}.get(u, 1)
                d[k] = v
        stalls = []
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    stalls.append((float(r[i]), h.split("stalled_")[1].replace("_per_issue_active.ratio", "")))
                except ValueError:
                    pass
        d["top_stalls"] = [f"{n}={v:.2f}" for v, n in sorted(stalls, reverse=True)[:4]]
        res.append(d)
    return res


def main():
    lpath, rpath, prefix = sys.argv[1:4]
    agg = launches(lpath)
    fl = full(rpath)
    with open(prefix + "_summary.md", "w") as fh:
        fh.write(f"# ncu summary ({prefix.split('/')[-1]})\n\n")
        fh.write("Launch list (`--metrics gpu__time_duration.sum --clock-control none`, cold-cache and "
                 "serialised: compare shares, not absolutes):\n\n| kernel | launches | mean us |\n|---|---|---|\n")
        for k, v in agg.items():
            fh.write(f"| `{k[:70]}` | {len(v)} | {sum(v) / len(v):.1f} |\n")
        fh.write("\n`--set full` captures (one launch each, steady-state iteration):\n\n")
        fh.write("| kernel | us | DRAM read GB | DRAM write GB | DRAM % of ncu peak | warps active % | regs | "
                 "fp64 pipe % | top stalls |\n|---|---|---|---|---|---|---|---|---|\n")
        for d in fl:
            fh.write(f"| `{d['kernel'][:40]}` | {d.get('time_us', 0):.1f} | {d.get('dram_read_B', 0) / 1e9:.3f} | "
                     f"{d.get('dram_write_B', 0) / 1e9:.3f} | {d.get('dram_pct_peak', 0):.1f} | "
                     f"{d.get('warps_active_pct', 0):.1f} | {d.get('regs', 0):.0f} | {d.get('fp64_pipe_pct', 0):.1f} | "
                     f"{', '.join(d['top_stalls'])} |\n")
    traffic = {}
    names = {"k_rs<": "RS_rows_local", "k_rs_compact<": "RS_rows_local", "k_pk<": "PK_axis0_spectral",
             "k_maxis<256, 1": "MI_axis1_inverse", "k_maxis<256, 0": "MF_axis1_forward",
             "k_tpk<": "PK_T", "k_trs<": "RS_T", "k_taxis<256, 1>": "MI_T", "k_taxis<256, 0>": "MF_T"}
    for d in fl:
        for key, stage in names.items():
            if key in d["kernel"] and stage not in traffic:
                traffic[stage] = d.get("dram_read_B", 0) + d.get("dram_write_B", 0)
    json.dump(traffic, open(prefix + "_traffic.json", "w"), indent=1)
    print(open(prefix + "_summary.md").read())


if __name__ == "__main__":
    main()
