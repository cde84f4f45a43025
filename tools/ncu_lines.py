"""Aggregate an ncu report's warp-stall samples by CUDA source line.

    python tools/ncu_lines.py REPORT.ncu-rep OBJECT.o [top] [kernel-regex] [sass-function-substring]

OBJECT.o is the -lineinfo object the kernel came from (its SASS offsets carry
the file:line table; they match the report's addresses relative to the
kernel's first instruction)."""
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def main(rep, obj, top=25, kre=None, fsub=None):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, check=True,
                   capture_output=True)
    cubin = [f for f in os.listdir(tmp) if f.endswith(".cubin")][0]
    sass = subprocess.run(["nvdisasm", "-g", os.path.join(tmp, cubin)], capture_output=True,
                          text=True).stdout.splitlines()
    # kernel-regex[@skip]: the skip-th launch matching the regex
    flt = []
    if kre:
        name, _, skip = kre.partition("@")
        flt = ["--kernel-name", "regex:" + name, "--launch-skip", skip or "0", "--launch-count", "1"]
    out = subprocess.run(["ncu", "-i", rep, *flt, "--page", "source", "--csv", "--print-source",
                          "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, data = rows[1], rows[2:]
    ai = hdr.index("Warp Stall Sampling (All Samples)")
    # per-reason columns (stall_*, all samples)
    rcols = [(i, h[6:]) for i, h in enumerate(hdr) if h.startswith("stall_") and "(" not in h]
    # the kernel's own function in the cubin: match by instruction count order
    kname = rows[0][1].split("(")[0].split("::")[-1]
    funcs, cur, cur_fn = {}, None, None
    for line in sass:
        if line.startswith("\t.text.") or line.startswith(".text."):
            cur_fn = line.strip().rstrip(":")
            funcs[cur_fn] = {}
            cur = None
            continue
        m = re.search(r'line (\d+)', line)
        if "## File" in line and m:
            cur = (line.split('"')[1].split("/")[-1], int(m.group(1)))
        m2 = re.match(r'\s+/\*([0-9a-f]{4,})\*/', line)
        if m2 and cur and cur_fn:
            funcs[cur_fn][int(m2.group(1), 16)] = cur
    kname = kname.split("<")[0]
    cands = [f for f in funcs if (fsub in f if fsub else kname in f)] or list(funcs)
    base = int(data[0][0], 16)
    def fl(x):
        try:
            return float(x)
        except ValueError:
            return 0.0
    tot = sum(fl(r[ai]) for r in data if len(r) > ai) or 1.0
    for fn in cands:
        agg, why = {}, {}
        for r in data:
            if len(r) <= ai:
                continue
            try:
                key = funcs[fn].get(int(r[0], 16) - base, ("?", 0))
            except ValueError:
                continue
            agg[key] = agg.get(key, 0.0) + fl(r[ai])
            w = why.setdefault(key, {})
            for i, nm in rcols:
                if i < len(r):
                    w[nm] = w.get(nm, 0.0) + fl(r[i])
        print("==", fn)
        for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
            w = why.get(k, {})
            tw = sum(w.values()) or 1.0
            rs = ", ".join("%s %d%%" % (n, 100 * c / tw) for n, c in
                           sorted(w.items(), key=lambda x: -x[1])[:3] if c > 0)
            print("%5.1f%% %-26s %s" % (100 * v / tot, "%s:%d" % k, rs))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 25,
         sys.argv[4] if len(sys.argv) > 4 else None, sys.argv[5] if len(sys.argv) > 5 else None)
