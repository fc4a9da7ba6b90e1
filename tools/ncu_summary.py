"""Key metrics of an `ncu --set full` report as JSON (read here, no GPU needed).

    python tools/ncu_summary.py gpurun_out/r1a/refine_c2_tile.ncu-rep [more.ncu-rep ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "mem_throughput_pct",
    "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active": "dmma_pipe_pct",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": "fma_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "smsp__cycles_active.avg": "smsp_cycles_active",
    "sm__cycles_elapsed.avg.per_second": "sm_hz",
}


def _num(s):
    try:
        return float(s.replace(",", ""))
    except ValueError:
        return s


def summarise(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, data = rows[0], rows[1], rows[2:]
    res = []
    for r in data:
        item = {"kernel": r[head.index("Kernel Name")].split("(")[0]}
        for k, name in KEYS.items():
            if k in head:
                v = _num(r[head.index(k)])
                u = units[head.index(k)]
                if name.startswith("dram_") and isinstance(v, float):
                    v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
                if name == "duration_ns" and isinstance(v, float):
                    v *= {"ns": 1, "us": 1e3, "usecond": 1e3, "ms": 1e6, "msecond": 1e6}.get(u, 1)
                item[name] = v
        if "dram_read" in item and "dram_write" in item:
            item["dram_bytes_per_launch"] = item["dram_read"] + item["dram_write"]
        res.append(item)
    return res


if __name__ == "__main__":
    allr = {p: summarise(p) for p in sys.argv[1:]}
    print(json.dumps(allr, indent=1))
