"""Per-launch DRAM traffic of the K4 kernels from an ncu --set full capture.

    python tools/traffic_json.py gpurun_out/ncu_k4.ncu-rep 22 profiles/r01_traffic.json

Rows: {"kernel": "k_bmv_bbb_stream<4>", "scale": 22, "tile_dim": 4,
"dram_bytes": read + write, "gpu_time_us": ...}; bench.py reports dram_bytes
as roofline.traffic."""
import csv
import io
import json
import re
import subprocess
import sys

rep, scale, out = sys.argv[1], int(sys.argv[2]), sys.argv[3]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]


def val(r, k):
    i = hdr.index(k)
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-3, "usecond": 1, "msecond": 1e3}
    return float(r[i].replace(",", "")) * mult.get(units[i], 1)


res = []
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    m = re.search(r"k_bmv_bbb_stream<(\d+)", name)
    if not m:
        continue
    d = int(m.group(1))
    res.append({"kernel": f"k_bmv_bbb_stream<{d}>", "scale": scale, "tile_dim": d,
                "dram_bytes": int(val(r, "dram__bytes_read.sum") + val(r, "dram__bytes_write.sum")),
                "gpu_time_us": round(val(r, "gpu__time_duration.sum"), 1)})
json.dump(res, open(out, "w"), indent=1)
print(json.dumps(res))
