"""Curated summary of an `ncu --set full` report (raw page) -> JSON on stdout.

    python scripts/ncu_summary.py gpurun_out/x.ncu-rep [kernel-regex]
"""
import csv, io, json, re, subprocess, sys

KEYS = [
    "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "launch__shared_mem_per_block_dynamic", "launch__cluster_dim_x",
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg.per_second",
    "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_tc.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__cycles_active.avg",
]


def summarise(path, kernel=None):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        if kernel and not re.search(kernel, d.get("Kernel Name", "")):
            continue
        s = {"kernel": d.get("Kernel Name", "")[:80]}
        for k in KEYS:
            if k in d:
                v = d[k].replace(",", "")
                try:
                    s[k] = float(v)
                except ValueError:
                    s[k] = v
        stalls = {k.split("smsp__pcsamp_warps_issue_stalled_")[1]: float(v.replace(",", "") or 0)
                  for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("_not_issued")}
        tot = sum(stalls.values()) or 1.0
        s["stall_top"] = {k: round(v / tot, 3) for k, v in sorted(stalls.items(), key=lambda x: -x[1])[:6]}
        res.append(s)
    return res


if __name__ == "__main__":
    print(json.dumps(summarise(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None), indent=1))
