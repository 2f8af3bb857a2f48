"""Summarise ncu output into profiles/ text files.

    python tools/summarize_ncu.py launches <launches.csv>        # per-kernel launch-time table
    python tools/summarize_ncu.py report <prof.ncu-rep> [regex]   # key metrics + stall reasons per kernel
"""
import collections
import csv
import io
import subprocess
import sys

UNIT = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    hdr = rows[0]
    ix = {h: i for i, h in enumerate(hdr)}
    agg = collections.OrderedDict()
    for r in rows[1:]:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        key = (r[ix["Kernel Name"]].split("(")[0][:70], r[ix["Grid Size"]])
        us = float(r[ix["Metric Value"]].replace(",", "")) * UNIT.get(r[ix["Metric Unit"]], 1.0)
        agg.setdefault(key, []).append(us)
    tot = sum(sum(v) for v in agg.values())
    out = ["kernel | grid | launches | avg us | total us | share of listed device time",
           "---|---|---|---|---|---"]
    for (k, grid), v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        out.append(f"{k} | {grid} | {len(v)} | {sum(v) / len(v):.2f} | {sum(v):.1f} | {100 * sum(v) / tot:.1f}%")
    return "\n".join(out)


KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum",
        "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "lts__t_sectors_srcunit_tex_op_red.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size"]


def report(path, regex=None):
    args = ["ncu", "-i", path, "--page", "raw", "--csv"]
    if regex:
        args += ["-k", f"regex:{regex}"]
    raw = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        out.append(f"## {d.get('Kernel Name', '?')[:110]}")
        for k in KEYS:
            if k in d:
                out.append(f"  {k:60s} {d[k]:>16s} {units[hdr.index(k)]}")
        tot = 0.0
        st = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued"):
                try:
                    st[h.replace("smsp__pcsamp_warps_issue_stalled_", "")] = float(r[i])
                    tot += float(r[i])
                except ValueError:
                    pass
        if tot:
            top = sorted(st.items(), key=lambda x: -x[1])[:6]
            out.append("  stall samples: " + ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in top))
    return "\n".join(out)


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        print(launches(sys.argv[2]))
    else:
        print(report(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None))
