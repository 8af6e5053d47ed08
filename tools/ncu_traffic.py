#!/usr/bin/env python
"""Record the DRAM traffic and L2 hit rates of one row-kernel launch from an ncu --set full report into
profiles/ncu_traffic.json, keyed by workload and stamped with the row-kernel source hash bench.py
checks (a capture is only quoted for the kernel source it measured).

python tools/ncu_traffic.py REPORT.ncu-rep KEY [SOURCE-DESCRIPTION]     e.g. KEY = x2_n262144_m256
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from bench import kernel_src_sha  # noqa: E402

rep, key = sys.argv[1], sys.argv[2]
src = sys.argv[3] if len(sys.argv) > 3 else os.path.basename(rep)
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))


def num(k):
    v = float(d[k].replace(",", ""))
    u = units.get(k, "")
    return v * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)


entry = {"dram_bytes": num("dram__bytes_read.sum") + num("dram__bytes_write.sum"),
         "dram_read_bytes": num("dram__bytes_read.sum"), "dram_write_bytes": num("dram__bytes_write.sum"),
         "l2_hit_pct": {"all_sectors": float(d["lts__t_sector_hit_rate.pct"]),
                        "reads": float(d["lts__t_sector_op_read_hit_rate.pct"])},
         "duration_ms": float(d["gpu__time_duration.sum"]) * (1e-3 if units.get("gpu__time_duration.sum") == "usecond" else 1.0),
         "kernel": d.get("Kernel Name", ""), "src_sha": kernel_src_sha(), "source": src}
p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
db = json.load(open(p)) if os.path.exists(p) else {}
db = {k: v for k, v in db.items() if isinstance(v, dict) or k == "_doc"}
db["_doc"] = ("per launch of the fused row kernel: dram__bytes_read.sum + dram__bytes_write.sum, L2 hit rates "
              "(lts__t_sector_hit_rate.pct all sectors; lts__t_sector_op_read_hit_rate.pct the B gathers) from one "
              "ncu --set full capture; src_sha = hash of csrc/{spgemm,split}.cu + {internal,devutil}.cuh at capture time (bench.py "
              "quotes the traffic only while the kernel source is unchanged)")
db[key] = entry
json.dump(db, open(p, "w"), indent=1)
print(json.dumps(entry))
