"""Per-source-line instruction counts and stall samples of one kernel: the ncu
SASS page (--page source --csv --print-source sass, per-instruction metrics)
joined by code offset with `nvdisasm -gi` of the same build's cubin (line
info with the inlining chain; compile with -lineinfo).

usage: python tools/sass_lines.py build/wide_kernels.o MANGLED_KERNEL ncu_sass.csv [top]
Prints the top lines by executed instructions, attributing each instruction to
its innermost source line and to the outermost line of the kernel's own file."""
import collections
import csv
import os
import re
import subprocess
import sys
import tempfile


def disasm(obj, kernel):
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, check=True,
                       stdout=subprocess.DEVNULL)
        cub = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
        out = subprocess.run(["nvdisasm", "-c", "-gi", os.path.join(d, cub)], capture_output=True,
                             text=True, check=True).stdout
    sec = out.split(f".text.{kernel}:")[1].split("\n.section")[0].split("//---------------------")[0]
    cur, chain, grp, rows = None, [], [], {}
    for ln in sec.splitlines():
        m = re.match(r'\s*//## File "([^"]+)", line (\d+)', ln)
        if m:  # a group of these precedes an instruction: innermost first, outermost last
            grp.append((os.path.basename(m.group(1)), int(m.group(2))))
            continue
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
        if m:
            if grp:
                cur, chain, grp = grp[0], grp[1:], []
            if cur:
                rows[int(m.group(1), 16)] = (cur, chain, m.group(2).strip())
    return rows


def main():
    obj, kernel, csvp = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    rows = disasm(obj, kernel)
    R = list(csv.reader(open(csvp)))
    h = R[1]
    ia, isamp = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    data = [r for r in R[2:] if r and r[0].startswith("0x")]
    base = int(data[0][0], 16)
    inner, outer = collections.Counter(), collections.Counter()
    sin, sout = collections.Counter(), collections.Counter()
    tot = ts = 0
    miss = 0
    for r in data:
        off = int(r[0], 16) - base
        n = int(r[ia] or 0)
        s = int(r[isamp] or 0) if r[isamp].isdigit() else 0
        tot += n
        ts += s
        if off not in rows:
            miss += n
            continue
        cur, inl, _ = rows[off]
        kfile = os.path.basename(obj).replace(".o", ".cu")
        chain = [cur] + inl
        out = next((c for c in reversed(chain) if c[0] == kfile), chain[-1])
        inner[cur] += n
        sin[cur] += s
        outer[out] += n
        sout[out] += s
    print(f"total {tot} instructions, {ts} samples, unmapped {miss}")
    print("\n-- innermost line: inst%  samples%")
    for k, n in inner.most_common(top):
        print(f"{k[0]}:{k[1]:<5d} {100 * n / tot:5.1f}%  {100 * sin[k] / max(ts, 1):5.1f}%")
    print("\n-- kernel-file line (outermost): inst%  samples%")
    for k, n in outer.most_common(top):
        print(f"{k[0]}:{k[1]:<5d} {100 * n / tot:5.1f}%  {100 * sout[k] / max(ts, 1):5.1f}%")


if __name__ == "__main__":
    main()
