"""profiles/traffic.json from an ncu --set full report of the rotation's
traverse_kernel launches (tools/evidence.sh): mean DRAM bytes (read +
write) per launch, and per launch. usage: traffic.py REPORT OUT.json"""
import csv, io, json, subprocess, sys
rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, vals = rows[0], rows[1], rows[2:]
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
per = []
for v in vals:
    b = 0.0
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = h.index(name)
        b += float(v[i].replace(",", "")) * scale.get(u[i], 1)
    per.append(round(b))
d = {"c2": sum(per) / len(per), "per_launch": per, "kernel": "traverse_kernel",
     "source": rep, "note": "mean over the 8-source rotation's launches (the tail kernel's "
     "bytes are in ncu_full_tail.txt)"}
json.dump(d, open(out, "w"), indent=1)
print(json.dumps(d))
