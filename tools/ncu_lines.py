"""Stall samples per CUDA source line from an ncu report (cuda,sass source view), with
the dominant stall reasons of each line.
usage: python tools/ncu_lines.py report.ncu-rep [top]"""
import csv, io, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg, why = {}, {}
cur = None; fname = None; tot = 0; hdr = None; stall_cols = []
for r in rows:
    if len(r) >= 2 and r[0] == "File Name":
        fname = r[1].split("/")[-1]; continue
    if "Warp Stall Sampling (All Samples)" in r:
        hdr = r; wi = r.index("Warp Stall Sampling (All Samples)")
        stall_cols = [(i, c) for i, c in enumerate(r) if c.startswith("stall_")]
        continue
    if hdr is None or len(r) <= wi:
        continue
    if r[0].isdigit():
        cur = (fname, int(r[0]), r[1].strip()[:90])
    try:
        v = int(r[wi])
    except ValueError:
        continue
    if not r[0].isdigit() and cur is not None:
        agg[cur] = agg.get(cur, 0) + v; tot += v
        d = why.setdefault(cur, {})
        for i, c in stall_cols:
            try:
                d[c] = d.get(c, 0) + int(r[i])
            except ValueError:
                pass
print("total samples", tot)
for k, v in sorted(agg.items(), key=lambda x: -x[1])[:top]:
    reasons = sorted(why.get(k, {}).items(), key=lambda x: -x[1])[:3]
    rs = " ".join("%s=%d%%" % (c[6:], 100 * n // max(v, 1)) for c, n in reasons if n)
    print("%7d %5.1f%%  %s:%d  %-70s  [%s]" % (v, 100.0 * v / tot, k[0], k[1], k[2][:70], rs))
