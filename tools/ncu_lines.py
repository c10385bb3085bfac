"""Aggregate ncu SASS-level stall samples by CUDA source line (via nvdisasm line info)."""
import csv, re, subprocess, sys, collections
rep, func, cubin = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h = rows[1]
ai, si, ni = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
data = [(int(r[ai], 16), float(r[si] or 0), r[ni]) for r in rows[2:] if len(r) > si and r[ai].startswith("0x")]
base = data[0][0]
sass = subprocess.run(["nvdisasm", "--print-line-info", "-fun", func, cubin], capture_output=True, text=True).stdout
if not sass.strip():
    sass = subprocess.run(["nvdisasm", "--print-line-info", cubin], capture_output=True, text=True).stdout
    i = sass.index(".text." + func)
    sass = sass[i:]
    j = sass.find("//--------------------- .text.", 10)
    sass = sass[:j] if j > 0 else sass
line = None
off2line = {}
for l in sass.splitlines():
    m = re.search(r'line (\d+)', l)
    if "//## File" in l and m:
        line = int(m.group(1))
        continue
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/', l)
    if m and line is not None:
        off2line[int(m.group(1), 16)] = line
agg = collections.Counter()
tot = 0.0
for a, v, s in data:
    agg[off2line.get(a - base, -1)] += v
    tot += v
src = open("/root/repo/paper_1908_10169_b200/csrc/bilu_factor.cu").read().splitlines()
for ln, v in agg.most_common(top):
    print("%5.1f%%  %5d  %s" % (100 * v / tot, ln, src[ln - 1].strip()[:100] if 0 < ln <= len(src) else "?"))
