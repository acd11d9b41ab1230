"""Attribute ncu per-SASS-instruction counters to source functions of a kernel.

    ncu -i rep.ncu-rep --page source --csv --print-source sass > sass.csv
    nvdisasm -gi -c kernel.cubin > kernel.sass
    python scripts/sass_hotspots.py sass.csv kernel.sass <mangled kernel name> <source.cu>

For each instruction the inline chain from nvdisasm -gi ("line X inlined at line Y ...")
is resolved to the innermost enclosing function of <source.cu> (function extents are
found by a brace scan of the source) and to the call-site line in the kernel body.
Prints warp-stall samples and executed instructions per function and per kernel line.
"""
import csv
import re
import sys
from collections import defaultdict


def function_ranges(src):
    """(start, end, name) for every top-level or namespace-level function body."""
    lines = open(src).read().split("\n")
    out, depth, cur, start = [], 0, None, 0
    sig = re.compile(r"^\s*(?:template\s*<.*>\s*)?(?:__\w+__\s+)*(?:[\w:<>,\s\*&]+?)\s+(\w+)\s*\(")
    pending = None
    for i, ln in enumerate(lines, 1):
        s = ln.split("//")[0]
        if cur is None:
            m = sig.match(s)
            if m and m.group(1) not in ("if", "for", "while", "switch", "return"):
                pending = (m.group(1), i)
        for ch in s:
            if ch == "{":
                if cur is None and pending and depth <= 2:
                    cur, start, base = pending[0], pending[1], depth
                depth += 1
            elif ch == "}":
                depth -= 1
                if cur is not None and depth == base:
                    out.append((start, i, cur))
                    cur, pending = None, None
        if s.strip().endswith(";") and cur is None:
            pending = None
    return out


def main():
    sass_csv, dis, kname, src = sys.argv[1:5]
    rows = list(csv.reader(open(sass_csv)))
    hdr = rows[1]
    ia, isamp, iexe = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), \
        hdr.index("Instructions Executed")
    stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_")]
    data = []
    for r in rows[2:]:
        if len(r) <= iexe or not r[ia].startswith("0x"):
            continue
        data.append((int(r[ia], 16), float(r[isamp] or 0), float(r[iexe] or 0),
                     {hdr[i]: float(r[i] or 0) for i in stall_cols}))
    base = data[0][0]
    # offset -> chain of (file, line)
    chain_of, chain, inside = {}, [], False
    fre = re.compile(r'//## File "([^"]+)", line (\d+)(?: inlined at "([^"]+)", line (\d+))?')
    for ln in open(dis):
        if ln.startswith(kname + ":"):
            inside = True
            continue
        if not inside:
            continue
        if ln.startswith(".L_x") or ln.strip().startswith("//##") or "/*" in ln:
            pass
        if ln.startswith(".text.") or (ln.startswith("_Z") and ln.rstrip().endswith(":")):
            break
        m = fre.search(ln)
        if m:
            if "inlined at" not in ln and chain and chain[-1][2] is None:
                chain = []
            if not chain or chain[-1][2] is None:
                chain = []
            chain.append((m.group(1), int(m.group(2)), m.group(3)))
            continue
        mo = re.match(r"\s*/\*([0-9a-f]{4,})\*/", ln)
        if mo:
            chain_of[int(mo.group(1), 16)] = [(f, l) for f, l, _ in chain]
    fr = function_ranges(src)

    def fname(line):
        best = None
        for s, e, n in fr:
            if s <= line <= e and (best is None or e - s < best[1] - best[0]):
                best = (s, e, n)
        return best[2] if best else "?"

    by_path = defaultdict(lambda: [0.0, 0.0])
    by_fn, by_line = defaultdict(lambda: [0.0, 0.0]), defaultdict(lambda: [0.0, 0.0])
    stall_fn = defaultdict(lambda: defaultdict(float))
    tot_s = tot_e = 0.0
    for addr, samp, exe, st in data:
        ch = chain_of.get(addr - base, [])
        ours = [l for f, l in ch if f.endswith(src.split("/")[-1])]
        inner = fname(ours[0]) if ours else "(other)"
        if ch and not ch[0][0].endswith(src.split("/")[-1]):
            inner = f"{inner}<{ch[0][0].split('/')[-1]}>"
        outer = ours[-1] if ours else -1
        for d in range(1, 5):
            key = tuple(reversed(ours))[:d]
            if len(key) == d:
                by_path[key][0] += samp
                by_path[key][1] += exe
        by_fn[inner][0] += samp
        by_fn[inner][1] += exe
        by_line[outer][0] += samp
        by_line[outer][1] += exe
        for k, v in st.items():
            stall_fn[inner][k] += v
        tot_s += samp
        tot_e += exe
    print(f"total stall samples {tot_s:.0f}, warp instructions executed {tot_e:.0f}")
    print(f"{'function':40s} {'samples%':>9s} {'inst%':>7s}  top stalls")
    for k, (s, e) in sorted(by_fn.items(), key=lambda x: -x[1][0]):
        if s / tot_s < 0.003:
            continue
        top = sorted(stall_fn[k].items(), key=lambda x: -x[1])[:4]
        tops = " ".join(f"{n[6:]}:{100 * v / max(s, 1):.0f}%" for n, v in top if v > 0)
        print(f"{k:40s} {100 * s / tot_s:9.1f} {100 * e / tot_e:7.1f}  {tops}")
    print("\ncall paths (outermost line first, depth <= 4), >= 1% of samples:")
    for k, (s, e) in sorted(by_path.items()):
        if s / tot_s >= 0.01:
            print(f"  {'  ' * (len(k) - 1)}{'>'.join(map(str, k)):24s} [{fname(k[-1])}] "
                  f"samples {100 * s / tot_s:5.1f}%  inst {100 * e / tot_e:5.1f}%")
    print("\nkernel-body call-site lines:")
    for k, (s, e) in sorted(by_line.items(), key=lambda x: -x[1][0])[:25]:
        print(f"  line {k:5d}  samples {100 * s / tot_s:5.1f}%  inst {100 * e / tot_e:5.1f}%")


if __name__ == "__main__":
    main()
