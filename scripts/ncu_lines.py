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
    iw, iwi = hdr.index("L1 Wavefronts Shared"), hdr.index("L1 Wavefronts Shared Ideal")
    res = []
    for r in rows[2:]:
        if len(r) <= ie:
            continue
        try:
            res.append((int(r[ia], 16), float(r[ie] or 0), float(r[iss] or 0), r[isr].strip(),
                        float(r[iw] or 0), float(r[iwi] or 0)))
        except ValueError:
            continue
    return res


_HELPERS = {}


def helper_lines(src):
    """Lines of the tiny helpers (ld/st/static_for/cp_async) in the compiled copy of the source."""
    src = os.environ.get("BBW_SRC") or src  # the copy the library was compiled from, if it moved on
    if src not in _HELPERS:
        out = set()
        try:
            for i, ln in enumerate(open(src).read().splitlines(), 1):
                if re.search(r"__forceinline__ (R ld|void st|void static_for|void cp_async|void prefetch_l2|void ld_shared_vec_pred)\(", ln):
                    out.update(range(i, i + 6))
        except OSError:
            pass
        _HELPERS[src] = out
    return _HELPERS[src]


def line_map(so, kernel_sub):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    cubins = [os.path.join(tmp, f) for f in os.listdir(tmp) if f.endswith(".cubin")]
    for cb in cubins:
        dis = subprocess.run(["nvdisasm", "-gi", "-c", cb], capture_output=True, text=True).stdout
        fname = None
        mp = {}
        cur = None
        pending, pending_open = [], False
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
                # consecutive File lines list the inlining chain, innermost first; take the
                # innermost location outside the tiny helpers (ld/st/static_for/intrinsics)
                locs = re.findall(r'"([^"]+)", line (\d+)', t)
                if not pending_open:
                    pending = []
                    pending_open = True
                pending.extend(locs)
                pick = None
                for f, l in pending:
                    if os.path.basename(f) == "stage_kernel.cuh" and int(l) not in helper_lines(f):
                        pick = (os.path.basename(f), int(l))
                        break
                if pick is None and pending:
                    pick = (os.path.basename(pending[0][0]), int(pending[0][1]))
                cur = pick
                continue
            pending_open = False
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
    agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0, 0.0])
    tot_i = sum(r[1] for r in rows)
    tot_s = sum(r[2] for r in rows)
    tot_w = sum(r[4] for r in rows) or 1.0
    for addr, n, s, src, w, wi in rows:
        key = mp.get(addr - base, ("?", 0))
        a = agg[key]
        a[0] += n
        a[1] += s
        a[2] += w
        a[3] += wi
    print(f"kernel {name[:100]}  total warp instr {tot_i:.4g}, stall samples {tot_s:.4g}, smem wavefronts {tot_w:.4g}")
    if "--dump" in sys.argv:  # machine-readable: file line inst stall wavefronts ideal
        with open(sys.argv[sys.argv.index("--dump") + 1], "w") as fh:
            for (f, l), (n, s, w, wi) in sorted(agg.items()):
                fh.write(f"{f} {l} {n} {s} {w} {wi}\n")
    for (f, l), (n, s, w, wi) in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
        print(f"{s / tot_s * 100:6.1f}% stall {n / tot_i * 100:6.1f}% inst {w / tot_w * 100:6.1f}% smem-wf "
              f"(ideal {wi / max(w, 1) * 100:4.0f}%)  {f}:{l}")


if __name__ == "__main__":
    main()
