"""Condense an ncu --set full report into profiles/<name>.json (key metrics + stall mix)."""
import csv, io, json, subprocess, sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__cycles_active.avg", "sm__cycles_active.max", "sm__cycles_elapsed.avg",
        "sm__cycles_elapsed.avg.per_second", "launch__registers_per_thread", "launch__grid_size",
        "launch__block_size", "smsp__inst_executed.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum",
        "lts__t_bytes.sum"]


def main(rep, out, kernel_regex=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    kernels = []
    for vals in rows[2:]:
        rec = {"kernel": vals[hdr.index("Kernel Name")][:160]}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                rec[k] = {"value": vals[i], "unit": units[i]}
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio"):
                try:
                    v = float(vals[i])
                except ValueError:
                    continue
                if v > 0.02:
                    stalls[h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", "")] = v
        rec["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
        kernels.append(rec)
    json.dump({"report": rep, "kernels": kernels}, open(out, "w"), indent=1)
    print(json.dumps(kernels[0], indent=1)[:2000])


if __name__ == "__main__":
    main(*sys.argv[1:])
