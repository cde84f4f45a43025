"""One line per kernel launch of an ncu --set full report: duration, DRAM
bytes and achieved GB/s (vs the measured HBM peak), tensor-pipe activity
(legacy HMMA pipe `tc%` and the tcgen05 datapath `utc%` =
sm__mem_tensor_cycles_active), MUFU (XU) pipe, SM / L2 throughput and the
top warp-stall reasons.

    python tools/ncu_table.py REPORT.ncu-rep [HBM_PEAK_GBs]
"""
import csv
import io
import subprocess
import sys


def main(rep, peak):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name, default="nan"):
        i = col.get(name)
        return r[i] if i is not None and i < len(r) else default

    def num(x):
        try:
            return float(str(x).replace(",", ""))
        except ValueError:
            return float("nan")

    stall_cols = [h for h in hdr if h.startswith("smsp__pcsamp_warps_issue_stalled_")
                  and "not_issued" not in h]
    print("%-44s %8s %9s %8s %6s %6s %6s %6s %6s %6s  %s" % (
        "kernel", "us", "DRAM MB", "GB/s", "%HBM", "tc%", "utc%", "xu%", "SM%", "L2%", "top stalls"))
    for r in rows[2:]:
        name = get(r, "Kernel Name")[:44]
        tu = rows[1][col["gpu__time_duration.sum"]]
        us = num(get(r, "gpu__time_duration.sum")) * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0,
                                                       "usecond": 1.0, "ms": 1e3,
                                                       "msecond": 1e3}.get(tu, 1e-3)
        mbs = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
        mb = sum(num(get(r, k)) * mbs.get(rows[1][col[k]], 1e-6)
                 for k in ("dram__bytes_read.sum", "dram__bytes_write.sum") if k in col)
        gbs = mb / 1e3 / (us / 1e6) if us > 0 else float("nan")
        tc = num(get(r, "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                     get(r, "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed")))
        sm = num(get(r, "sm__throughput.avg.pct_of_peak_sustained_elapsed"))
        # tcgen05 (UTC) datapath activity and the MUFU (XU) pipe
        utc = num(get(r, "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"))
        xu = num(get(r, "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed"))
        l2 = num(get(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"))
        st = sorted(((num(get(r, h)), h.split("stalled_")[1].split(".")[0]) for h in stall_cols),
                    reverse=True)
        tot = sum(a for a, _ in st if a == a) or 1.0
        top = ", ".join("%s %.0f%%" % (k, 100 * a / tot) for a, k in st[:3])
        print("%-44s %8.1f %9.1f %8.0f %6.1f %6.1f %6.1f %6.1f %6.1f %6.1f  %s" % (
            name, us, mb, gbs, 100 * gbs / peak, tc, utc, xu, sm, l2, top))


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 6536.0)
