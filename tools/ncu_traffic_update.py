"""Store the DRAM bytes of the bench's own decode launch (an ncu
--metrics dram__bytes_read.sum,dram__bytes_write.sum csv) in
profiles/ncu_traffic.json, which bench.py reports as roofline.traffic:
    python tools/ncu_traffic_update.py profiles/r02_dram_c5.csv "<command that produced it>"
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

path, cmd = sys.argv[1], sys.argv[2]
vals = {}
for r in csv.reader(open(path)):
    if len(r) > 14 and r[12] in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum"):
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1, "usecond": 1e3, "msecond": 1e6}
        vals[r[12]] = float(r[14].replace(",", "")) * scale.get(r[13], 1)
rd, wr = vals["dram__bytes_read.sum"], vals["dram__bytes_write.sum"]
m, N = 6, 8726282760  # C5: (63,57), 2^39 coded bits
alg = (63 * N + 7) // 8 + (57 * N + 7) // 8 + N + 8
out = {"c5_m6_syn": {"m": m, "n_codewords": N, "syndromes": True, "dram_bytes_read": int(rd), "dram_bytes_write": int(wr),
                     "alg_bytes": alg, "source": f"{os.path.relpath(path, ROOT)}: {cmd} (the bench launch itself, one B200)",
                     "traffic": int(rd + wr), "traffic_per_alg_byte": (rd + wr) / alg,
                     "kernel_ns_under_ncu": vals.get("gpu__time_duration.sum")}}
json.dump(out, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print(json.dumps(out, indent=1))
