"""Record the DRAM traffic of one PCG product from an `ncu --set full` report into
profiles/ncu_traffic.json, keyed by (config, k, vertex order, source hash of the CUDA build), so
bench.py attaches roofline.traffic only for the build that was profiled.
A product may be several launches (the rows path: chunks + two slab passes); the report must hold
exactly the launches of ONE product, whose DRAM bytes and durations are summed.
Usage: python tools/record_traffic.py <report.ncu-rep> <config> <k> <order> [summary.json]"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2101_08143_b200 import build as B  # noqa: E402

rep, cfg, k, order = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
u = dict(zip(hdr, units))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = [dict(zip(hdr, vals)) for vals in rows[2:] if len(vals) == len(hdr)]
tot = sum(float(d[m].replace(",", "")) * scale[u[m]] for d in launches
          for m in ["dram__bytes_read.sum", "dram__bytes_write.sum"])
tunit = {"ns": 1e-3, "nsecond": 1e-3, "us": 1, "usecond": 1, "ms": 1e3, "msecond": 1e3, "s": 1e6, "second": 1e6}[
    u["gpu__time_duration.sum"]]   # -> microseconds
dur = sum(float(d["gpu__time_duration.sum"].replace(",", "")) * tunit for d in launches)
d = launches[0]
path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
key = f"{cfg}/k{k}/{order}/{B.source_hash()}"
db[key] = {"spmv_dram_bytes_per_launch": int(tot), "kernel": " + ".join(x.get("Kernel Name", "?") for x in launches),
           "launches": len(launches), "duration_us": dur,
           "source": sys.argv[5] if len(sys.argv) > 5 else os.path.basename(rep)}
json.dump(db, open(path, "w"), indent=1)
print(key, db[key])
