"""Attribute ncu per-SASS-instruction samples to CUDA source lines.

    python scripts/sass_lines.py <ncu source-page csv> <cubin> <kernel mangled name> [top]

The ncu csv comes from `ncu -i rep --page source --csv`; the cubin from
`cuobjdump -xelf all build/obj/<tu>.o`.  Needs -lineinfo builds.
"""
import collections
import csv
import re
import subprocess
import sys


def line_map(cubin, kernel):
    out = subprocess.run(["nvdisasm", "-g", "-c", "-fun", kernel, cubin], capture_output=True, text=True).stdout
    if not out.strip():
        out = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
        s = out.find(f".text.{kernel}")
        out = out[s:]
        e = out.find("//--------------------- .text.", 10)
        out = out[:e] if e > 0 else out
    cur = None
    mp = {}
    for ln in out.splitlines():
        m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
        if m:
            cur = (m.group(1).split("/")[-1], int(m.group(2)))
            continue
        m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", ln)
        if m and cur:
            mp[int(m.group(1), 16)] = cur
    return mp


def main():
    csvf, cubin, kernel = sys.argv[1:4]
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 40
    mp = line_map(cubin, kernel)
    rows = list(csv.reader(open(csvf)))
    h = rows[1]
    ai, ie, st = h.index("Address"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    base = None
    inst, samp = collections.Counter(), collections.Counter()
    for r in rows[2:]:
        if len(r) <= st:
            continue
        a = int(r[ai], 16)
        base = a if base is None else base
        key = mp.get(a - base, ("?", 0))
        inst[key] += int(r[ie] or 0)
        samp[key] += int(r[st] or 0)
    T, S = sum(inst.values()), sum(samp.values())
    print(f"{'file:line':34s} {'inst%':>6s} {'stall%':>7s}")
    for k, v in sorted(samp.items(), key=lambda x: -x[1])[:top]:
        print(f"{k[0] + ':' + str(k[1]):34s} {100 * inst[k] / T:6.1f} {100 * v / S:7.1f}")


if __name__ == "__main__":
    main()
