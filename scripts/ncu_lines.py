#!/usr/bin/env python
"""Attribute ncu per-SASS-instruction metrics to CUDA source lines.

    python scripts/ncu_lines.py <report.ncu-rep> <libbbwadg.so> <kernel-substring> [--top 40]

ncu's source page (``--page source --csv``) gives instructions executed and stall samples per
SASS address; ``nvdisasm --print-line-info`` on the kernel's cubin gives the source line of each
SASS offset.  Offsets are matched relative to the function start.
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile


def ncu_rows(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ia, ie, isr = hdr.index("Address"), hdr.index("Instructions Executed"), hdr.index("Source")
    iss = hdr.index("Warp Stall Sampling (All Samples)")
    res = []
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        try:
            res.append((int(r[ia], 16), float(r[ie] or 0), float(r[iss] or 0), r[isr].strip()))
        except ValueError:
            continue
    return res


def line_map(so, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "--print-line-info", "-c", cb], capture_output=True, text=True).stdout
        fname = None
        mp = {}
        cur = None
        for ln in dis.splitlines():
            t = ln.strip()
            if t.startswith(".text.") and t.endswith(":"):
                if fname and kernel_sub in fname and mp:
                    return fname, mp
                fname = t[len(".text."):-1]
                mp = {}
                cur = None
                continue
            if fname is None or kernel_sub not in fname:
                continue
            if "//## File" in t:
                m = re.search(r'line (\d+)', t)
                fm = re.search(r'File "([^"]+)"', t)
                if m:
                    cur = (os.path.basename(fm.group(1)) if fm else "?", int(m.group(1)))
                continue
            m2 = re.match(r"/\*([0-9a-f]{4,})\*/", t)
            if m2 and cur:
                mp[int(m2.group(1), 16)] = cur
        if fname and kernel_sub in fname and mp:
            return fname, mp
    return None, {}


def main():
    rep, so, sub = sys.argv[1:4]
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    rows = ncu_rows(rep)
    name, mp = line_map(so, sub)
    if not mp:
        print("no line info found for", sub)
        return
    base = rows[0][0]
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    tot_i = sum(r[1] for r in rows)
    tot_s = sum(r[2] for r in rows)
    for addr, n, s, src in rows:
        key = mp.get(addr - base, ("?", 0))
        agg[key][0] += n
        agg[key][1] += s
    print(f"kernel {name[:100]}  total warp instr {tot_i:.4g}, stall samples {tot_s:.4g}")
    for (f, l), (n, s) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{s / tot_s * 100:6.1f}% stall {n / tot_i * 100:6.1f}% inst  {f}:{l}")


if __name__ == "__main__":
    main()
