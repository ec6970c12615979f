"""Attribute ncu warp-stall samples (SASS source page) to CUDA source lines.

usage: python tools/ncu_lines.py REPORT.ncu-rep OBJ_OR_CUBIN KERNEL_MANGLED_SUBSTR [top]

Runs `ncu -i --page source --csv` (SASS view), `cuobjdump -xelf` + `nvdisasm -g`
for line info, maps instruction offsets (runtime address - function start) to
(file, line), and prints the top lines by stall samples.  Dev tooling only.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile


def main():
    rep, obj, kern = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hi = next(i for i, r in enumerate(rows) if "Address" in r and "Source" in r)
    hdr = rows[hi]
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    i_x = hdr.index("Instructions Executed")
    data = [r for r in rows[hi + 1:] if len(r) > i_s and r[0].startswith("0x")]
    base = min(int(r[0], 16) for r in data)
    tmp = tempfile.mkdtemp()
    if obj.endswith(".cubin"):
        cub = obj
    else:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=tmp, capture_output=True)
        cub = glob.glob(os.path.join(tmp, "*.cubin"))[0]
    sass = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
    # locate function
    lines = sass.splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith(".text.") and kern in l)
    off2line = {}
    cur = ("?", 0)
    for l in lines[start + 1:]:
        if l.startswith(".text."):
            break
        m = re.search(r'//## File "([^"]+)", line (\d+)', l)
        if m:
            cur = (os.path.basename(m.group(1)), int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", l)
        if m:
            off2line[int(m.group(1), 16)] = cur
    agg = collections.Counter()
    ex = collections.Counter()
    tot = 0.0
    for r in data:
        off = int(r[0], 16) - base
        key = off2line.get(off, ("?", 0))
        s = float(r[i_s] or 0)
        agg[key] += s
        ex[key] += float(r[i_x] or 0)
        tot += s
    srcfiles = {}
    order = agg.most_common(top) if os.environ.get("SORT") != "inst" else [(k2, agg[k2]) for k2, _ in ex.most_common(top)]
    for (f, ln), s in order:
        text = ""
        for cand in glob.glob(os.path.join(os.path.dirname(__file__), "..", "paper_2506_02572_b200", "csrc", f)):
            srcfiles.setdefault(cand, open(cand).read().splitlines())
            if 0 < ln <= len(srcfiles[cand]):
                text = srcfiles[cand][ln - 1].strip()
        print(f"{s / tot * 100:5.1f}%  inst={ex[(f, ln)]:9.0f}  {f}:{ln:<5d} {text[:100]}")


if __name__ == "__main__":
    main()
