#!/usr/bin/env python
"""Per-phase totals (instructions, stall samples, shared-memory wavefronts) of the stage kernel.

    python scripts/ncu_phases.py <report.ncu-rep> <libbbwadg.so> <kernel-substring> <elements>

Uses scripts/ncu_lines.py's SASS -> source-line attribution, then maps lines of the compiled
stage_kernel.cuh to phases by its marker comments ("// ---- X:", "// F:", "// G:", ...).
"""
import os
import re
import sys
import tempfile

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
import ncu_lines  # noqa: E402

MARK = [(r"__forceinline__ void sum4_phase", "sum4 (G,H)"), (r"__forceinline__ void face_sum3", "face_sum3 (C2,D)"),
        (r"__forceinline__ void zero_pad_rows", "zero_pad_rows"), (r"// F: h'_g", "F product"), (r"// F \(v5\)", "F product"),
        (r"auto reduce = \[&\]", "G/H tri reduce"), (r"// I: upward, in place", "I upward"),
        (r"// G: M reductions", "G call"), (r"// H: downward", "H call"), (r"// I: upward", "I upward"),
        (r"void __launch_bounds__", "kernel prologue"), (r"// ---- A:", "A loads"), (r"// ---- B1", "B1 flux"),
        (r"// ---- B2", "B2 grad"), (r"// ---- C1", "C1 vol elev"), (r"// ---- C2", "C2"), (r"// ---- C3", "C3 L0"),
        (r"// ---- D:", "D layers"), (r"// ---- E:", "E gather+LSRK u"), (r"// ---- F-I", "F-I call"),
        (r"// ---- J:", "J out+LSRK p"), (r"void pack_kernel", "pack")]


def phases_of(src):
    marks = []
    for i, ln in enumerate(open(src).read().splitlines(), 1):
        for pat, name in MARK:
            if re.search(pat, ln):
                marks.append((i, name))
    return sorted(marks)


def main():
    rep, so, sub, nel = sys.argv[1], sys.argv[2], sys.argv[3], float(sys.argv[4])
    dump = tempfile.mktemp()
    sys.argv = [sys.argv[0], rep, so, sub, "--top", "0", "--dump", dump]
    ncu_lines.main()
    rows = [ln.split() for ln in open(dump)]
    # the copy of stage_kernel.cuh the library was compiled from (BBW_SRC), default: this repo's
    src = os.environ.get("BBW_SRC") or os.path.join(os.path.dirname(HERE), "paper_1808_08645_b200", "csrc",
                                                     "stage_kernel.cuh")
    marks = phases_of(src)
    agg = {}
    T = [0.0] * 4
    for f, l, n, s, w, wi in rows:
        l = int(l)
        vals = list(map(float, (n, s, w, wi)))
        name = "other"
        if f == "stage_kernel.cuh":
            for ml, nm in marks:
                if ml <= l:
                    name = nm
        a = agg.setdefault(name, [0.0] * 4)
        for i, x in enumerate(vals):
            a[i] += x
            T[i] += x
    print(f"{'phase':20s} {'inst/el':>8s} {'stall%':>7s} {'smemwf/el':>10s} {'ideal/el':>9s}")
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"{k:20s} {v[0] / nel:8.0f} {v[1] / T[1] * 100:7.1f} {v[2] / nel:10.0f} {v[3] / nel:9.0f}")
    print(f"{'total':20s} {T[0] / nel:8.0f} {100:7.1f} {T[2] / nel:10.0f} {T[3] / nel:9.0f}")


if __name__ == "__main__":
    main()
