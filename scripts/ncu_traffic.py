"""profiles/ncu_traffic_cfg<N>.json from an ncu report of the filter-degree kernel (family
"gram": profiles/ncu_traffic_gram_cfg<N>.json, the DMMA Gram kernels of one ARR): DRAM
bytes per launch (read + write), read by bench.py as roofline.traffic when the kernel
family matches the launched kernel.

    python scripts/ncu_traffic.py gpurun_out/prof.ncu-rep <N> <kernel_family> [source]
"""
import csv
import io
import json
import subprocess
import sys

SCALE = {"byte": 1, "kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "tbyte": 1e12}
TSCALE = {"ms": 1, "us": 1e-3, "usecond": 1e-3, "msecond": 1, "ns": 1e-6, "nsecond": 1e-6, "s": 1e3, "second": 1e3}


def main(rep, cid, family, source=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        def val(k):
            return float(r[h.index(k)]) * SCALE.get(units[h.index(k)].lower(), 1)
        tk = "gpu__time_duration.sum"
        out.append({"kernel": r[h.index("Kernel Name")][:120], "dram_read": val("dram__bytes_read.sum"),
                    "dram_write": val("dram__bytes_write.sum"),
                    "time_ms": float(r[h.index(tk)]) * TSCALE.get(units[h.index(tk)].lower(), 1)})
    per = sum(o["dram_read"] + o["dram_write"] for o in out) / len(out)
    doc = {"kernel_family": family, "dram_bytes_per_launch": per, "launches_profiled": out,
           "source": source or rep, "how": "ncu --set full --clock-control none: dram__bytes_read.sum + dram__bytes_write.sum"}
    name = (f"profiles/ncu_traffic_{family}_cfg{cid}.json" if family in ("gram", "gemm")
            else f"profiles/ncu_traffic_cfg{cid}.json")
    with open(name, "w") as f:
        json.dump(doc, f, indent=1)
    print(json.dumps({"cfg": cid, "dram_bytes_per_launch": per}))


if __name__ == "__main__":
    main(*sys.argv[1:])
