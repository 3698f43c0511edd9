"""Per-launch summary of an exported ncu raw CSV (ncu -i X.ncu-rep --page raw --csv):
duration, DRAM read/write bytes (unit-normalised) and achieved DRAM GB/s.
Usage: python scripts/ncu_summary.py profiles/r2/s2/ncu_attn_c5_raw.csv [...]"""
import csv
import json
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
         "nsecond": 1e-9}


def summary(path: str) -> dict:
    rows = list(csv.reader(open(path)))
    h, units = rows[0], rows[1]
    out = []
    for v in rows[2:]:
        d = dict(zip(h, v))

        def val(k):
            i = h.index(k)
            return float(v[i].replace(",", "")) * SCALE.get(units[i], 1.0)
        t = val("gpu__time_duration.sum")
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        out.append({"kernel": d.get("Kernel Name", ""), "duration_s": t, "dram_read_bytes": rd,
                    "dram_write_bytes": wr, "dram_gbs": (rd + wr) / t / 1e9})
    return out[0] if len(out) == 1 else out


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(p, json.dumps(summary(p)))
