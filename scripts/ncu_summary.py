"""Summarise an ncu --set full report (.ncu-rep) into the compact per-launch
JSON kept under profiles/: device time, DRAM bytes, L2 throughput, tensor-pipe
activity and issue activity per kernel launch.

usage: python scripts/ncu_summary.py report.ncu-rep out.json
"""
import csv
import io
import json
import re
import subprocess
import sys

# tcgen05.mma kind::f16 M=128: 8192 bf16 flops per SM cycle (dense), i.e.
# N/2 cycles per 128 x N x 16 instruction; its SS operands are 128 x 16 (A)
# and N x 16 (B) bf16 = 32 + N/4 tensor-pipe SMEM wavefronts of 128 B
def tc_busy_pct(name, wavefronts, cycles):
    """Tensor-pipe busy share of the SM cycles, in the SM clock domain:
    (MMAs per SM x N/2 cycles) / sm__cycles_elapsed.avg, with the MMA count
    recovered from the tensor pipe's SMEM operand wavefronts and the kernel's
    N tile (tc_gemm_kernel<BN, ...>)."""
    m = re.search(r"tc_gemm_kernel<(\d+)", name)
    if not m or not wavefronts or not cycles:
        return None
    bn = int(m.group(1))
    n_mma = wavefronts / (32 + bn / 4)
    return round(100.0 * n_mma * (bn / 2) / (148 * cycles), 2)


def _f(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return None


def summarise(rep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True,
                         check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    col = {h: i for i, h in enumerate(hdr)}

    def get(r, name):
        i = col.get(name)
        return _f(r[i]) if i is not None and i < len(r) else None

    out = []
    for r in data:
        us = get(r, "gpu__time_duration.sum")
        unit = units[col["gpu__time_duration.sum"]]
        us = us / 1e3 if unit == "nsecond" else (us * 1e3 if unit == "msecond" else us)
        wf = get(r, "l1tex__data_pipe_tc_wavefronts_mem_shared.sum")
        cyc = get(r, "sm__cycles_elapsed.avg")
        name = r[col["Kernel Name"]]
        out.append({
            "kernel": name.split("(")[0][:110],
            "grid": int(get(r, "launch__grid_size") or 0),
            "regs": int(get(r, "launch__registers_per_thread") or 0),
            "us": round(us, 3),
            "dram_read_MB": get(r, "dram__bytes_read.sum"),
            "dram_write_MB": get(r, "dram__bytes_write.sum"),
            "lts_pct": get(r, "lts__throughput.avg.pct_of_peak_sustained_elapsed"),
            "tensor_busy_pct": tc_busy_pct(name, wf, cyc),
            "tc_smem_operand_pct": get(r, "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
            "issue_active_pct": get(r, "smsp__issue_active.avg.pct_of_peak_sustained_active"),
            "sm_clock_ghz": round(cyc / (us * 1e3), 3) if cyc and us else None,
        })
        # dram byte units: ncu reports MB or KB depending on size
        for key, m in (("dram_read_MB", "dram__bytes_read.sum"), ("dram_write_MB", "dram__bytes_write.sum")):
            u = units[col[m]] if m in col else "Mbyte"
            if out[-1][key] is not None:
                out[-1][key] = round(out[-1][key] * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0,
                                                     "Gbyte": 1e3}.get(u, 1.0), 3)
    return out


if __name__ == "__main__":
    res = summarise(sys.argv[1])
    json.dump(res, open(sys.argv[2], "w"), indent=1)
    for k in res:
        print(k)
