"""Stall samples of one kernel by source line.

Joins an ncu SASS source page (`ncu -i rep --page source --csv --print-source
sass -k regex:NAME`) with the line table of the same kernel's cubin
(`nvdisasm -gi`): every SASS instruction is charged to its innermost source
line and to the outermost line of the kernel's own file (the call site in
the kernel body).

usage: python sass_hotspots.py page.csv cubin.sass mangled_name [kernel_file]
"""
import collections
import csv
import re
import sys


def line_table(sass_path: str, mangled: str):
    txt = open(sass_path).read().split("\n")
    start = next(i for i, l in enumerate(txt) if ".section" in l and f".text.{mangled}," in l)
    loc, table, prev_comment = [], {}, False
    for l in txt[start + 1:]:
        if ".section" in l and ".text." in l:
            break
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', l)
        if m:
            chain = [(m.group(1).split("/")[-1], int(m.group(2)))]
            for f, n in re.findall(r'inlined at "([^"]+)", line (\d+)', m.group(3)):
                chain.append((f.split("/")[-1], int(n)))
            # consecutive comments: the first carries the whole inline chain
            if not prev_comment:
                loc = chain
            prev_comment = True
            continue
        prev_comment = False
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            table[int(m.group(1), 16)] = (loc, m.group(2).strip())
    return table


def main():
    page, sass, mangled = sys.argv[1:4]
    kfile = sys.argv[4] if len(sys.argv) > 4 else None
    rows = list(csv.reader(open(page)))
    h = rows[1]
    ia, isamp, iexe = h.index("Address"), h.index("Warp Stall Sampling (All Samples)"), \
        h.index("Instructions Executed")
    data = [(int(r[ia], 16), int(r[isamp] or 0), int(r[iexe] or 0)) for r in rows[2:] if r[ia].startswith("0x")]
    base = data[0][0]
    table = line_table(sass, mangled)
    inner, outer = collections.Counter(), collections.Counter()
    exe_inner = collections.Counter()
    total = sum(s for _, s, _ in data)
    for a, s, e in data:
        loc, ins = table.get(a - base, ([("?", 0)], "?"))
        key = f"{loc[0][0]}:{loc[0][1]}" if loc else "?"
        inner[key] += s
        exe_inner[key] += e
        if kfile:
            top = [x for x in loc if x[0] == kfile]
            outer[f"{kfile}:{top[-1][1]}" if top else "?"] += s
    print(f"total samples {total}")
    print("innermost source lines (share of samples, warp instructions executed):")
    for k, v in inner.most_common(30):
        print(f"  {100 * v / total:5.1f}%  {exe_inner[k]:>10d}  {k}")
    if kfile:
        print(f"call sites in {kfile}:")
        for k, v in outer.most_common(25):
            print(f"  {100 * v / total:5.1f}%  {k}")


if __name__ == "__main__":
    main()
