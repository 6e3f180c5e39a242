"""Condense an ncu `--page raw --csv` export (optionally .gz) into a small JSON
summary: duration, SM clock, DRAM bytes per launch, tensor-pipe activity.

    python tools/ncu_summary.py gpurun_out/k3_fixed11_r02a_raw.csv.gz > profiles/x.json
"""
import csv
import gzip
import json
import sys

SCALE = {"ms": 1e-3, "us": 1e-6, "ns": 1e-9, "s": 1, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "nsecond": 1e-9, "usecond": 1e-6,
         "msecond": 1e-3, "second": 1, "hz": 1, "Khz": 1e3, "Mhz": 1e6, "Ghz": 1e9, "cycle/nsecond": 1e9,
         "cycle/usecond": 1e6, "cycle/second": 1}
KEYS = {
    "duration_s": "gpu__time_duration.sum",
    "sm_hz": "sm__cycles_elapsed.avg.per_second",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "l2_bytes": "lts__t_bytes.sum",
    "tensor_pipe_active_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "tensor_mem_active_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
}


def main(path):
    op = gzip.open if path.endswith(".gz") else open
    rows = list(csv.reader(op(path, "rt")))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        d = {"kernel": vals[hdr.index("Kernel Name")][:120] if "Kernel Name" in hdr else None}
        for k, m in KEYS.items():
            if m in hdr:
                i = hdr.index(m)
                try:
                    v = float(vals[i].replace(",", ""))
                except ValueError:  # "no data" (e.g. no tensor pipe in a split kernel)
                    continue
                d[k] = v * SCALE.get(units[i], 1) if "pct" not in k else v
        if "dram_read_bytes" in d:
            d["traffic_bytes_per_launch"] = d["dram_read_bytes"] + d.get("dram_write_bytes", 0)
        out.append(d)
    print(json.dumps(out if len(out) > 1 else out[0], indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
