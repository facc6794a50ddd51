#!/usr/bin/env python
"""Reads an .ncu-rep (ncu -i ... --page raw --csv) and writes the metrics the round reports:
usage: python tools/ncu_select.py <report.ncu-rep> <out.csv> [<summary key> <summary.json>]"""
import csv
import io
import json
import subprocess
import sys

WANT = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__inst_executed_pipe_tensor.sum", "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_xu_cycles_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "sm__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_issued.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
    "lts__t_bytes.sum", "lts__t_sector_hit_rate.pct", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "sm__cycles_elapsed.avg",
    "sm__cycles_active.avg", "smsp__cycles_active.avg", "gpc__cycles_elapsed.max", "sm__cycles_elapsed.avg.per_second",
]


def main():
    rep, out_csv = sys.argv[1], sys.argv[2]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    idx = {h: i for i, h in enumerate(hdr)}
    keep = ["Kernel Name"] + [m for m in WANT if m in idx] + [h for h in hdr if "pipe_tensor" in h and h not in WANT]
    with open(out_csv, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(["metric", "unit"] + [f"launch{i}" for i in range(len(data))])
        for m in keep:
            w.writerow([m, units[idx[m]]] + [r[idx[m]] for r in data])
    if len(sys.argv) > 4:
        key, js = sys.argv[3], sys.argv[4]
        try:
            with open(js) as f:
                summ = json.load(f)
        except FileNotFoundError:
            summ = {}

        def val(m, scale_units=True):
            if m not in idx:
                return None
            v = float(data[0][idx[m]].replace(",", ""))
            u = units[idx[m]].lower()
            if scale_units:
                v *= {"kbyte": 1e3, "mbyte": 1e6, "gbyte": 1e9, "ms": 1e3, "ns": 1e-3}.get(u, 1.0)
            return v
        rd, wr = val("dram__bytes_read.sum"), val("dram__bytes_write.sum")
        summ[key] = {
            "source": f"{out_csv} (ncu --set full --clock-control none)",
            "kernel": data[0][idx["Kernel Name"]][:120],
            "dram_read_bytes": rd, "dram_write_bytes": wr,
            "dram_bytes_per_launch": (rd or 0) + (wr or 0),
            "duration_us_under_ncu": val("gpu__time_duration.sum"),
            "tensor_pipe_active_pct": val("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", False),
            "xu_pipe_pct": val("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", False),
            "issue_active_pct": val("sm__inst_issued.avg.pct_of_peak_sustained_active", False),
            "sm_cycles_elapsed": val("sm__cycles_elapsed.avg", False), "sm_cycles_active": val("sm__cycles_active.avg", False),
            "l2_hit_rate_pct": val("lts__t_sector_hit_rate.pct", False),
            "dram_throughput_pct": val("dram__throughput.avg.pct_of_peak_sustained_elapsed", False),
        }
        with open(js, "w") as f:
            json.dump(summ, f, indent=1)
        print(json.dumps(summ[key], indent=1))


if __name__ == "__main__":
    main()
