"""Summarise an ncu report: key metrics + instruction mix + top stalls per kernel."""
import csv, collections, subprocess, sys, io
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(io.StringIO(raw)))
hdr, units = r[0], r[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        # tensor-core evidence (tcgen05): pipe activity, instructions, TMEM traffic, operand reads
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_tensor.sum", "sm__inst_executed_pipe_tensor_subpipe_hmma.sum",
        "sm__inst_executed_pipe_tensor_subpipe_imma.sum", "sm__inst_executed_pipe_tmem.sum",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum"]
for row in r[2:]:
    print("=====", row[hdr.index("Kernel Name")][:60])
    for k in keys:
        if k in hdr:
            print(f"  {k} = {row[hdr.index(k)]} {units[hdr.index(k)]}")
    # any other tensor-pipe / TMEM metric the capture holds
    for i, h in enumerate(hdr):
        if ("pipe_tensor" in h or "mem_tensor" in h or "pipe_tc" in h or "pipe_tmem" in h) and h not in keys \
                and row[i] not in ("", "0", "0.00"):
            print(f"  {h} = {row[i]} {units[i]}")
    st = [(h.replace("smsp__pcsamp_warps_issue_stalled_", ""), int(row[i] or 0)) for i, h in enumerate(hdr)
          if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("not_issued") and row[i] not in ("", "0")]
    st.sort(key=lambda x: -x[1]); tot = sum(v for _, v in st)
    print("  stalls:", ", ".join(f"{k} {v/tot*100:.0f}%" for k, v in st[:8]))
