"""Per-round metrics from tools/phase_profile.sh captures: round k's share
is capture(stop k) - capture(stop k-1). usage: phase_delta.py DIR"""
import csv, glob, io, os, re, subprocess, sys
d = sys.argv[1]
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_sectors.sum", "lts__t_requests_srcunit_tex.sum",
        "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
        "lts__t_requests_srcunit_tex_op_atom_dot_alu.sum",
        "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum", "smsp__inst_executed.sum",
        "l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__t_sectors_op_atom.sum",
        "lts__t_sectors_op_red.sum"]
STALL = re.compile(r"smsp__pcsamp_warps_issue_stalled_(\w+)$")


def load(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    m = {}
    for i, name in enumerate(h):
        try:
            x = float(v[i].replace(",", ""))
        except ValueError:
            continue
        if name in WANT:
            scale = {"us": 1e3, "ms": 1e6, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9,
                     "byte": 1}.get(u[i], 1)
            m[name] = x * scale
        s = STALL.match(name)
        if s and not s.group(1).endswith("not_issued"):
            m["stall_" + s.group(1)] = x
    return m


caps = {}
for p in glob.glob(os.path.join(d, "stop_*.ncu-rep")):
    k = int(re.search(r"stop_(\d+)", p).group(1))
    caps[k] = load(p)
ks = sorted(caps)
prev = None
for k in ks:
    m = caps[k]
    if prev is not None:
        dm = {n: m.get(n, 0) - caps[prev].get(n, 0) for n in m}
        t = dm["gpu__time_duration.sum"] / 1e3
        dram = (dm.get("dram__bytes_read.sum", 0) + dm.get("dram__bytes_write.sum", 0))
        req = dm.get("lts__t_requests_srcunit_tex.sum", 0)
        rd = dm.get("lts__t_sectors_srcunit_tex_op_read.sum", 0)
        hit = dm.get("lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", 0)
        st = {n[6:]: x for n, x in dm.items() if n.startswith("stall_") and x > 0}
        tot = sum(st.values()) or 1
        top = sorted(st.items(), key=lambda kv: -kv[1])[:5]
        label = f"rounds {prev + 1}..{k}" if k - prev > 1 else f"round {k}"
        print(f"{label:14s} {t:8.1f} us  DRAM {dram / 1e6:8.1f} MB ({dram / max(t, 1e-9) / 1e3:6.0f} GB/s)"
              f"  L2 req {req / 1e6:6.2f} M ({req / max(t, 1e-9) / 1e3:6.1f} G/s)"
              f"  L2 rd sectors {rd / 1e6:6.2f} M hit {100 * hit / max(rd, 1):4.1f}%"
              f"  atom {dm.get('lts__t_requests_srcunit_tex_op_atom_dot_alu.sum', 0) / 1e6:5.2f} M"
              f"  L1 ld sectors {dm.get('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 0) / 1e6:6.2f} M"
              f" hit {100 * dm.get('l1tex__t_sectors_pipe_lsu_mem_global_op_ld_lookup_hit.sum', 0) / max(dm.get('l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum', 0), 1):4.1f}%"
              f"  smem wavefronts {dm.get('l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 0) / 1e6:6.2f} M"
              f"  L2 atom+red sectors {(dm.get('lts__t_sectors_op_atom.sum', 0) + dm.get('lts__t_sectors_op_red.sum', 0)) / 1e6:5.2f} M"
              f"  stalls " + ", ".join(f"{n} {100 * x / tot:.0f}%" for n, x in top))
    else:
        print(f"rounds 0..{k}: {m['gpu__time_duration.sum'] / 1e3:.1f} us")
    prev = k
