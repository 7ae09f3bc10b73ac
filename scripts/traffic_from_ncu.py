"""profiles/k2_traffic.json from one `ncu --set full` capture of the bench step's K2 launch.

    python scripts/traffic_from_ncu.py <capture.ncu-rep> <kernel name> [n batch mode]
"""
import csv
import io
import json
import subprocess
import sys

rep, kernel = sys.argv[1], sys.argv[2]
n, batch, mode = (int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]) if len(sys.argv) > 5 else (1024, 16, "MIXED_EMULATED")
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, units, vals = rows[0], rows[1], rows[2]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "sector": 1, "": 1}


def get(name):
    i = hdr.index(name)
    return float(vals[i]) * scale[units[i]]


rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
json.dump({"n": n, "batch": batch, "mode": mode, "layers": 30, "kernel": kernel,
           "dram_bytes_per_launch": rd + wr, "dram_read_bytes": rd, "dram_write_bytes": wr,
           "lts_sectors": get("lts__t_sectors.sum") if "lts__t_sectors.sum" in hdr else None,
           "source": f"ncu --set full --clock-control none, {rep.split('/')[-1]} (dram__bytes_read.sum + "
                     f"dram__bytes_write.sum) of one {kernel} launch (all 30 layers of the bench step)"},
          open("profiles/k2_traffic.json", "w"), indent=1)
print(open("profiles/k2_traffic.json").read())
