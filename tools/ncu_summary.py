"""Summarise ncu reports (``ncu -i <rep> --page raw --csv``) into one JSON
object per captured launch: duration, DRAM bytes and % of peak, issue and
FP64-pipe activity, shared-memory wavefronts, registers, occupancy.

    python tools/ncu_summary.py gpurun_out/r02_*.ncu-rep > profiles/r02/ncu_kernels.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "duration_us": ("gpu__time_duration.sum", 1),
    "dram_read_bytes": ("dram__bytes_read.sum", 1),
    "dram_write_bytes": ("dram__bytes_write.sum", 1),
    "dram_pct_of_peak": ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", 1),
    "issue_active_pct": ("sm__inst_issued.avg.pct_of_peak_sustained_active", 1),
    "fp64_pipe_pct": ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", 1),
    "shared_wavefronts": ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", 1),
    "l1tex_throughput_pct": ("l1tex__throughput.avg.pct_of_peak_sustained_active", 1),
    "registers": ("launch__registers_per_thread", 1),
    "warps_active_per_sm": ("sm__warps_active.avg.per_cycle_active", 1),
    "l2_hit_pct": ("lts__t_sector_hit_rate.pct", 1),
    "grid": ("launch__grid_size", 1),
    "block": ("launch__block_size", 1),
    "smem_per_block": ("launch__shared_mem_per_block", 1),
    "sm_clock_mhz": ("smsp__cycles_elapsed.avg.per_second", 1),
    "l2_to_sm_read_bytes": ("l1tex__m_xbar2l1tex_read_bytes.sum", 1),
    "l2_to_sm_tma_read_bytes": ("l1tex__m_xbar2l1tex_read_bytes_mem_global_op_tma_ld.sum", 1),
}
# unit -> factor to the summary's unit (us, bytes, MHz)
UNITS = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3, "second": 1e6,
         "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "KiB": 1024.0, "MiB": 2.0 ** 20,
         "hz": 1e-6, "Khz": 1e-3, "Mhz": 1.0, "Ghz": 1e3, "cycle/nsecond": 1e3, "cycle/usecond": 1.0,
         "cycle/second": 1e-6}


def num(s):
    try:
        return float(s.replace(",", ""))
    except (ValueError, AttributeError):
        return None


def summarise(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    head, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = dict(zip(head, r))
        e = {"report": rep, "kernel": d.get("Kernel Name", "")[:160]}
        for k, (m, scale) in METRICS.items():
            v = num(d.get(m))
            if v is not None:
                u = units[head.index(m)] if m in head else ""
                e[k] = v * scale * UNITS.get(u, 1.0)
        if "dram_read_bytes" in e and "dram_write_bytes" in e:
            e["dram_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
        res.append(e)
    return res


if __name__ == "__main__":
    allr = []
    for rep in sys.argv[1:]:
        allr += summarise(rep)
    print(json.dumps(allr, indent=1))
