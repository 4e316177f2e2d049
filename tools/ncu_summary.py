"""Summarise an ncu report: key metrics + top stall SASS + opcode mix."""
import csv, collections, subprocess, sys, io
rep = sys.argv[1]
def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout
raw = run("--page", "raw", "--csv")
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, vals = rows[0], rows[1], rows[2:]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "smsp__inst_executed.sum", "lts__t_bytes.sum",
        "l1tex__t_bytes.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
for v in vals:
    print("kernel:", v[hdr.index("Kernel Name")][:80])
    for w in want:
        if w in hdr:
            i = hdr.index(w)
            print(f"  {w:60s} {v[i]:>20s} {units[i]}")
src = run("--page", "source", "--csv", "--print-source", "sass")
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]; data = rows[2:]
ix = {k: i for i, k in enumerate(h)}
S = "Warp Stall Sampling (All Samples)"
tot = sum(float(r[ix[S]] or 0) for r in data) or 1
agg = collections.Counter()
for r in data:
    for k in h:
        if k.startswith("stall_") and "Not Issued" not in k:
            agg[k] += float(r[ix[k]] or 0)
t2 = sum(agg.values()) or 1
print("stalls:", ", ".join(f"{k[6:]} {v/t2*100:.1f}%" for k, v in agg.most_common(8)))
ops = collections.Counter()
for r in data:
    toks = r[1].split()
    op = toks[1] if toks and toks[0].startswith("@") else (toks[0] if toks else "?")
    ops[op] += float(r[ix["Instructions Executed"]] or 0)
print("inst:", sum(ops.values()), ops.most_common(14))
top = sorted(data, key=lambda r: -float(r[ix[S]] or 0))[:int(sys.argv[2]) if len(sys.argv) > 2 else 15]
for r in top:
    s = float(r[ix[S]] or 0)
    rs = sorted([(float(r[ix[k]] or 0), k[6:]) for k in h if k.startswith("stall_") and "Not Issued" not in k], reverse=True)[:2]
    print(f"  {r[0][-5:]} {s/tot*100:5.1f}% n={r[ix['Instructions Executed']]:>9} {r[1][:58]:58s} {rs}")
