"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo).
usage: ncu_lines.py REPORT [TOP]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
per_line = []
cur = None
for r in rows:
    if len(r) > 4 and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 6:
        if r and r[0] == "File Path":
            fname = r[1]
        continue
    if r[0]:
        nm = len(hdr) - 4
        met = r[-nm:]
        mh = hdr[4:]
        src = ",".join(r[1:len(r) - nm - 2])
        cur = [r[0], src, 0.0, collections.Counter(), 0.0, fname]
        per_line.append(cur)
        val = lambda x: float(x) if x not in ("-", "") else 0.0
        cur[2] = val(met[0])
        cur[4] = val(met[3])
        for h, x in zip(mh, met):
            if h.startswith("stall_") and "Not Issued" not in h:
                cur[3][h[6:]] += val(x)
tot = sum(x[2] for x in per_line) or 1
for ln, src, samp, st, inst, fn in sorted(per_line, key=lambda x: -x[2])[:top]:
    reasons = ", ".join(f"{k} {v/samp*100:.0f}%" for k, v in st.most_common(2)) if samp else ""
    print(f"{fn.split('/')[-1]}:{ln:>4} {samp/tot*100:5.1f}%  inst={inst:>11.0f}  {src.strip()[:70]:70s} {reasons}")
