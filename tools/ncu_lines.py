"""Per-CUDA-source-line stall samples from an ncu report (needs -lineinfo).
usage: ncu_lines.py REPORT [TOP] [MINUS_REPORT]
With MINUS_REPORT the samples of that report are subtracted line by line
(captures of the round kernel stopped after rounds k and k-1: round k alone)."""
import csv, io, subprocess, sys, collections


def parse(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = None
    fname = ""
    lines = {}
    val = lambda x: float(x) if x not in ("-", "") else 0.0
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
            st = collections.Counter()
            for h, x in zip(mh, met):
                if h.startswith("stall_") and "Not Issued" not in h:
                    st[h[6:]] += val(x)
            lines[(fname.split("/")[-1], r[0])] = [src, val(met[0]), st, val(met[3])]
    return lines


rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cur = parse(rep)
if len(sys.argv) > 3:
    for k, (src, samp, st, inst) in parse(sys.argv[3]).items():
        if k in cur:
            cur[k][1] -= samp
            cur[k][3] -= inst
            cur[k][2].subtract(st)
tot = sum(x[1] for x in cur.values()) or 1
for (fn, ln), (src, samp, st, inst) in sorted(cur.items(), key=lambda kv: -kv[1][1])[:top]:
    reasons = ", ".join(f"{k} {v/samp*100:.0f}%" for k, v in st.most_common(2)) if samp > 0 else ""
    print(f"{fn}:{ln:>4} {samp/tot*100:5.1f}%  inst={inst:>11.0f}  {src.strip()[:70]:70s} {reasons}")
