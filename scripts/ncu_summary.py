"""Summarise an ncu report: key throughput metrics, stall reasons, SASS opcode mix."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
npairs = float(sys.argv[2]) if len(sys.argv) > 2 else 0
json_out = sys.argv[3] if len(sys.argv) > 3 else None  # profiles/ncu_<config>.json
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, vals = rows[0], rows[2]
want = ['gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum', 'lts__t_bytes.sum',
        'lts__t_sector_hit_rate.pct', 'lts__throughput.avg.pct_of_peak_sustained_elapsed',
        'l1tex__throughput.avg.pct_of_peak_sustained_active', 'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread', 'launch__grid_size',
        'launch__block_size', 'smsp__issue_active.avg.pct_of_peak_sustained_active', 'smsp__inst_executed.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed', 'launch__shared_mem_per_block_dynamic',
        'l1tex__data_pipe_lsu_wavefronts_mem_shared.sum', 'smsp__sass_inst_executed_op_ldgsts.sum',
        'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum']
units = {h: rows[1][i] for i, h in enumerate(hdr)}
for i, h in enumerate(hdr):
    if h in want:
        print(f"{h:60s} {vals[i]:>18s} {units.get(h,'')}")
if json_out:
    import json
    g = {h: vals[i] for i, h in enumerate(hdr)}
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    rd = float(g["dram__bytes_read.sum"]) * scale[units["dram__bytes_read.sum"]]
    wr = float(g["dram__bytes_write.sum"]) * scale[units["dram__bytes_write.sum"]]
    with open(json_out, "w") as f:
        json.dump({"source": rep.split("/")[-1] + " (ncu --set full, 1 launch = 1 epoch)",
                   "kernel_ms": float(g["gpu__time_duration.sum"]),
                   "dram_bytes_per_launch": rd + wr,
                   "l2_hit_rate_pct": float(g["lts__t_sector_hit_rate.pct"]),
                   "lts_throughput_pct": float(g["lts__throughput.avg.pct_of_peak_sustained_elapsed"]),
                   "issue_active_pct": float(g["smsp__issue_active.avg.pct_of_peak_sustained_active"]),
                   "registers": int(float(g["launch__registers_per_thread"])),
                   "grid": int(float(g["launch__grid_size"])),
                   "block": int(float(g["launch__block_size"]))}, f, indent=1)
stalls = [(h, float(vals[i])) for i, h in enumerate(hdr)
          if h.startswith('smsp__pcsamp_warps_issue_stalled') and not h.endswith('not_issued') and vals[i]]
tot = sum(v for _, v in stalls) or 1
print("stall samples:")
for h, v in sorted(stalls, key=lambda x: -x[1])[:10]:
    print(f"  {h.replace('smsp__pcsamp_warps_issue_stalled_',''):28s} {100*v/tot:5.1f}%")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(src.splitlines()))
hdr = rows[1]; data = rows[2:]
iS = hdr.index("Source"); iE = hdr.index("Instructions Executed")
c = Counter()
for r in data:
    toks = r[iS].split()
    if not toks: continue
    op = toks[1] if toks[0].startswith('@') else toks[0]
    c[op.split('.')[0]] += float(r[iE] or 0)
tot = sum(c.values())
print(f"instructions executed: {tot:.4g}" + (f" = {tot/npairs:.0f} per pair" if npairs else ""))
print("  " + ", ".join(f"{op} {n/(npairs or 1):.0f}" for op, n in c.most_common(24)))
