"""Dev tool: summarise an ncu --set full capture into a JSON (profiles/)."""
import csv, json, subprocess, sys

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum"]
rep, out, note = sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else ""
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(txt.splitlines()))
h, u = rows[0], rows[1]
res = {"source": f"ncu --set full --clock-control none capture {rep.split('/')[-1]}", "note": note, "kernels": []}
for v in rows[2:]:
    k = {"name": v[h.index("Kernel Name")], "metrics": {}, "stall_samples": {}}
    for i, n in enumerate(h):
        if n in WANT:
            k["metrics"][n] = {"unit": u[i], "value": v[i]}
        if n.startswith("smsp__pcsamp_warps_issue_stalled") and not n.endswith("not_issued") and v[i] not in ("0", ""):
            k["stall_samples"][n.replace("smsp__pcsamp_warps_issue_stalled_", "")] = v[i]
    res["kernels"].append(k)
json.dump(res, open(out, "w"), indent=1)
print(out, [k["name"] for k in res["kernels"]])
