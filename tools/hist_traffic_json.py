"""profiles/latest_hist_traffic.json from an ncu --set full raw CSV of the C2
hist launch (tools/ncu_hist_capture.sh), which bench.py reads for
roofline.traffic.

    python tools/hist_traffic_json.py gpurun_out/hist_full_raw.csv COMMIT [summary.txt]
"""
import csv
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}


def main():
    rows = list(csv.reader(open(sys.argv[1])))
    names, units, vals = rows[0], rows[1], rows[2]

    def get(name, unit_scale=True):
        i = names.index(name)
        v = float(vals[i].replace(",", ""))
        return v * SCALE.get(units[i], 1) if unit_scale else v

    rd, wr = get("dram__bytes_read.sum"), get("dram__bytes_write.sum")
    out = {
        "kernel": vals[names.index("Kernel Name")].split("(")[0],
        "workload": "bench.py C2, 100 frames x 13 candidates, one launch (timed region)",
        "source": "ncu --set full --clock-control none --import-source on -k regex:judge_hist -s 3 -c 1 "
                  "python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pipeline "
                  f"(tools/ncu_hist_capture.sh at commit {sys.argv[2]}"
                  + (f", {sys.argv[3]}" if len(sys.argv) > 3 else "") + ")",
        "captured_at_commit": sys.argv[2],
        "duration_ms": get("gpu__time_duration.sum"),
        "dram_read_bytes": rd,
        "dram_write_bytes": wr,
        "bytes_per_launch": rd + wr,
        "algorithmic_bytes_per_launch": 100 * 2048 * 2048 * 2,
        "l1tex_lsu_data_pipe_pct_of_peak": get("l1tex__data_pipe_lsu_wavefronts.sum.pct_of_peak_sustained_elapsed"),
        "smem_wavefronts": get("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"),
        "smem_bank_conflict_wavefronts": get("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"),
        "atoms_instructions": get("smsp__inst_executed_op_shared_atom.sum"),
        "lts_throughput_pct": get("lts__throughput.avg.pct_of_peak_sustained_elapsed"),
        "lts_hit_rate_pct": get("lts__t_sector_hit_rate.pct"),
    }
    (ROOT / "profiles" / "latest_hist_traffic.json").write_text(json.dumps(out, indent=1) + "\n")
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
