"""Write one profiles/traffic.json entry from an `ncu --set full` report of a fill kernel:
python tools/traffic_record.py REPORT.ncu-rep CFG VARIATES_PER_LAUNCH SOURCE_NOTE"""
import csv
import io
import json
import os
import subprocess
import sys

rep, cfg, nv, note = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
d = dict(zip(hdr, rows[2]))


def val(key, unit_to=1):
    u = units[hdr.index(key)]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "inst": 1, "ns": 1e-9, "us": 1e-6, "ms": 1e-3}
    return float(d[key].replace(",", "")) * scale.get(u, 1)


rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
rec = json.load(open(path)) if os.path.exists(path) else {}
rec[cfg] = {"bytes_per_launch": int(rd + wr), "dram_read_bytes": int(rd), "dram_write_bytes": int(wr),
            "kernel": d["Kernel Name"].replace("<unnamed>::", "").split("(")[0].replace("void ", ""),
            "source": note, "algorithmic_bytes": nv * 8,
            "warp_instructions_per_launch": int(val("smsp__inst_executed.sum")),
            "variates_per_launch": nv, "gpu_time_s": val("gpu__time_duration.sum")}
json.dump(rec, open(path, "w"), indent=1)
print(json.dumps(rec[cfg], indent=1))
