"""Per-source-line dynamic instruction counts of one kernel from an ncu source-page CSV.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    nvdisasm -gi -c kernel.cubin > kernel.sass
    python scripts/sass_lines.py sass.csv kernel.sass <mangled kernel name> <source.cu> <pixels> [lo hi]

Each SASS instruction is attributed to its innermost source line (nvdisasm -gi inline
chains); prints warp-level executed instructions per pixel-warp for lines lo..hi.
"""
import csv
import re
import sys
from collections import defaultdict

sass_csv, dis, kname, src = sys.argv[1:5]
pixels = float(sys.argv[5])
lo = int(sys.argv[6]) if len(sys.argv) > 6 else 0
hi = int(sys.argv[7]) if len(sys.argv) > 7 else 10**9
rows = list(csv.reader(open(sass_csv)))
hdr = rows[1]
ia, iexe, isamp = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(int(r[ia], 16), float(r[iexe] or 0), float(r[isamp] or 0)) for r in rows[2:]
        if len(r) > iexe and r[ia].startswith("0x")]
base = data[0][0]
line_of, cur, inside = {}, None, False
fre = re.compile(r'//## File "([^"]+)", line (\d+)')
for ln in open(dis):
    if ln.startswith(kname + ":"):
        inside = True
        continue
    if not inside:
        continue
    if ln.startswith(".text.") or (ln.startswith("_Z") and ln.rstrip().endswith(":")):
        break
    m = fre.search(ln)
    if m:
        if "inlined at" not in ln.split(m.group(0))[0] and not ln.lstrip().startswith("//## File") :
            pass
        # innermost entry is the first line of a chain block: nvdisasm prints innermost first
        if cur is None or not prev_was_chain:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
        prev_was_chain = True
        continue
    mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
    if mo:
        line_of[int(mo.group(1), 16)] = cur
        prev_was_chain = False
srcl = open(src).read().split("\n")
agg = defaultdict(lambda: [0.0, 0.0])
tot = 0.0
for a, e, s in data:
    k = line_of.get(a - base)
    agg[k][0] += e
    agg[k][1] += s
    tot += e
wp = pixels / 32
print(f"total warp-inst per pixel-warp {tot / wp:.1f}")
sel = 0.0
for k, (e, s) in sorted(agg.items(), key=lambda x: (x[0] is None, x[0])):
    if k is None or not k[0].endswith(src.split("/")[-1]) or not (lo <= k[1] <= hi):
        continue
    sel += e
    print(f"{k[1]:5d} {e / wp:7.1f}  {srcl[k[1] - 1].strip()[:100]}")
print(f"selected lines: {sel / wp:.1f} per pixel-warp")
