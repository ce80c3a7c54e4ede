#!/usr/bin/env python
"""profiles/traffic.json from the ncu CSVs of scripts/gpu_traffic.sh (DRAM bytes per stage-kernel
launch, read by bench.py for roofline.traffic; scaled by K_local when the bench mesh differs)."""
import csv
import json
import os
import re
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
K = {"N7M4": 4088832, "N5M3": 1053696, "N9M9": 511104}


def parse(path):
    rows = list(csv.reader(open(path)))
    hdr = next(i for i, r in enumerate(rows) if r and r[0] in ("ID", "\"ID\"") or (r and "Metric Name" in r) or
               (r and "dram__bytes_read.sum" in r))
    h = rows[hdr]
    out = {}
    if "Metric Name" in h:  # --metrics --csv (long format)
        im, iv, iu = h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
        for r in rows[hdr + 1:]:
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                     "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(r[iu], 1)
            out[r[im]] = float(r[iv].replace(",", "")) * scale
    else:  # --page raw --csv (wide format; second row holds units)
        units, vals = rows[hdr + 1], rows[hdr + 2]
        for name in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                     "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
                     "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"):
            i = h.index(name)
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "ms": 1e-3,
                     "usecond": 1e-6, "msecond": 1e-3, "nsecond": 1e-9}.get(units[i], 1)
            out[name] = float(vals[i].replace(",", "")) * scale
    return out


def main(src_dir):
    res = {}
    for f in sorted(os.listdir(src_dir)):
        m = re.match(r"traffic_(N\dM\d)(f32|f64)\.csv$", f)
        if not m:
            continue
        d = parse(os.path.join(src_dir, f))
        key = m.group(1) + m.group(2)
        e = {"K_local": K[m.group(1)],
             "dram_bytes_per_launch": d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"],
             "dram_read_bytes": d["dram__bytes_read.sum"], "dram_write_bytes": d["dram__bytes_write.sum"],
             "ncu_duration_s": d["gpu__time_duration.sum"],
             "source": f"ncu --clock-control none, one stage_kernel launch ({f})"}
        if "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed" in d:
            e["l1_data_pipe_pct_of_peak"] = d["l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed"]
            e["smem_wavefronts_per_element"] = d["l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"] / e["K_local"]
            e["warp_instructions_per_element"] = d["smsp__inst_executed.sum"] / e["K_local"]
        res[key] = e
    out = os.path.join(ROOT, "profiles", "traffic.json")
    with open(out, "w") as fh:
        json.dump(res, fh, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out"))
