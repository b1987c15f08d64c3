"""DRAM traffic per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the SRWCR
kernels in an `ncu --set full` report -> profiles/ncu_traffic.json[config][kernel].
usage: python tools/ncu_traffic.py REPORT CONFIG"""
import csv, io, json, os, subprocess, sys
rep, cfgname = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics",
                      "dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
units = rows[1]
out = {}
for r in rows[2:]:
    d = dict(zip(h, r))
    u = dict(zip(h, units))
    name = d["Kernel Name"].split("(")[0].split("<")[0].replace("srwcr::", "").replace("void ", "").strip()
    def val(k):
        v = float(d[k].replace(",", ""))
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6,
                 "msecond": 1e-3, "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(u[k], 1)
        return v * scale
    b = val("dram__bytes_read.sum") + val("dram__bytes_write.sum")
    out.setdefault(name, []).append((b, val("gpu__time_duration.sum")))
res = {k: {"bytes": sum(x[0] for x in v) / len(v), "ncu_ms": 1e3 * sum(x[1] for x in v) / len(v), "launches": len(v)}
       for k, v in out.items()}
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "ncu_traffic.json")
db = json.load(open(path)) if os.path.exists(path) else {}
db[cfgname] = {k: v["bytes"] for k, v in res.items()}
db.setdefault("_detail", {})[cfgname] = res
json.dump(db, open(path, "w"), indent=1)
print(json.dumps(res, indent=1))
