"""Summarise an .ncu-rep (raw metrics + stall breakdown + top SASS lines)."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
h, u, v = r[0], r[1], r[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__cycles_elapsed.avg",
        "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.per_cycle_active", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__m_xbar2l1tex_read_bytes.sum",
        "lts__t_bytes.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__memory_throughput.avg.pct_of_peak_sustained_elapsed", "launch__occupancy_limit_shared_mem",
        "launch__occupancy_limit_registers", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_lsu.sum", "smsp__inst_executed_op_shared_ld.sum",
        "dram__bytes_read.sum.per_second", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__t_sector_hit_rate.pct", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active"]
out = {}
for i, name in enumerate(h):
    if name in want:
        out[name] = (v[i], u[i])
for k in want:
    if k in out:
        print(f"{k:70s} {out[k][0]:>16} {out[k][1]}")
print("-- stall samples")
st = []
for i, name in enumerate(h):
    if name.startswith("smsp__pcsamp_warps_issue_stalled_") and not name.endswith("not_issued"):
        try:
            if float(v[i]) > 0:
                st.append((float(v[i]), name.replace("smsp__pcsamp_warps_issue_stalled_", "")))
        except ValueError:
            pass
for n, nm in sorted(st, reverse=True):
    print(f"  {nm:30s} {int(n)}")
if len(sys.argv) > 2:
    src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(src)))
    hdr = rows[1]
    ix = {x: i for i, x in enumerate(hdr)}
    data = rows[2:]
    tot = sum(int(x[ix["Instructions Executed"]] or 0) for x in data)
    print("-- SASS (total warp instrs %d)" % tot)
    thr = float(sys.argv[2])
    for x in data:
        e = int(x[ix["Instructions Executed"]] or 0)
        s = int(x[ix["Warp Stall Sampling (All Samples)"]] or 0)
        if e > tot * thr or s > 200:
            print(f"{x[ix['Address']][-5:]} {e:>10} {s:>6}  {x[ix['Source']].strip()[:90]}")
