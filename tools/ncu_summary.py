"""Summarise an ncu report: duration, pipes, stall reasons, hottest SASS."""
import csv
import io
import subprocess
import sys
from collections import Counter


FILTER = []


def page(rep, name, extra=()):
    out = subprocess.run(["ncu", "-i", rep, *FILTER, "--page", name, "--csv", *extra],
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main(rep, top=30):
    rows = page(rep, "raw")
    h, v = rows[0], rows[2]
    kv = dict(zip(h, v))
    for k in ("gpu__time_duration.sum", "sm__cycles_elapsed.avg", "sm__cycles_active.avg",
              "launch__grid_size", "launch__registers_per_thread",
              "dram__bytes_read.sum", "dram__bytes_write.sum"):
        print(k, kv.get(k))
    for k in sorted(kv):
        if "inst_executed_pipe" in k and k.endswith("avg.pct_of_peak_sustained_active"):
            try:
                if float(kv[k]) > 1:
                    print("  ", k.split("__")[1].split(".")[0], kv[k])
            except ValueError:
                pass
    st = []
    for k, x in kv.items():
        if "pcsamp_warps_issue_stalled" in k and "not_issued" not in k:
            try:
                st.append((float(x.replace(",", "")), k.split("stalled_")[1]))
            except ValueError:
                pass
    tot = sum(a for a, _ in st) or 1
    print("stalls:", ", ".join("%s %.1f%%" % (k, 100 * a / tot)
                               for a, k in sorted(st, reverse=True)[:8]))
    src = page(rep, "source", ("--print-source", "sass"))
    hh = src[1]
    ia, isrc = hh.index("Address"), hh.index("Source")
    iss, iex = hh.index("Warp Stall Sampling (All Samples)"), hh.index("Instructions Executed")
    data = []
    for r in src[2:]:
        try:
            data.append((int(r[iss]), int(r[iex]), r[ia][-5:], r[isrc].strip()))
        except (ValueError, IndexError):
            pass
    tot = sum(d[0] for d in data) or 1
    hot = sorted(data, key=lambda d: -d[0])[:top]
    for d in sorted(hot, key=lambda d: d[2]):
        print("%5.1f%% %9d %s %s" % (100 * d[0] / tot, d[1], d[2], d[3][:80]))
    c = Counter()
    for s, e, a, srcl in data:
        op = srcl.split()[1] if srcl.startswith("@") else srcl.split()[0]
        c[op.split(".")[0]] += e
    print("executed mix:", c.most_common(16))


if __name__ == "__main__":
    # ncu_summary.py REPORT [TOP] [LAUNCH_INDEX]: one kernel of a multi-kernel report
    if len(sys.argv) > 3:
        FILTER = ["--launch-skip", sys.argv[3], "--launch-count", "1"]
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30)
