"""Summarise ncu --set full reports into profiles/ JSON (one object per profiled launch).

    python tools/ncu_summary.py gpurun_out/prof_r1_c2.ncu-rep profiles/ncu_c2_summary.json

The first launch of the scoring kernel also provides `dram_bytes_per_launch` (read + write),
which bench.py reports as roofline.traffic.
"""
import csv
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_ns",
    "dram__bytes_read.sum": "dram_bytes_read",
    "dram__bytes_write.sum": "dram_bytes_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "launch__registers_per_thread": "registers_per_thread",
    "launch__grid_size": "grid_size",
    "launch__block_size": "block_size",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wavefronts",
    "smsp__inst_executed.sum": "warp_instructions",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64_pipe_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active": "xu_pipe_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active": "lsu_pipe_pct",
    "sm__inst_executed_pipe_adu.avg.pct_of_peak_sustained_active": "adu_pipe_pct",
    "sm__cycles_elapsed.avg.per_second": "sm_clock_hz",
}


def main(rep, out):
    txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        if len(r) != len(hdr):
            continue
        d = dict(zip(hdr, r))
        rec = {"kernel": d.get("Kernel Name", "")[:120], "id": d.get("ID")}
        for k, name in KEYS.items():
            if k in d and d[k] != "":
                try:
                    v = float(d[k].replace(",", ""))
                    u = units[hdr.index(k)]
                    scale = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "us": 1e3, "usecond": 1e3,
                             "ms": 1e6, "msecond": 1e6, "Ghz": 1e9, "Mhz": 1e6}
                    v *= scale.get(u, 1.0)
                    rec[name] = v
                except ValueError:
                    pass
        if "dram_bytes_read" in rec:
            rec["dram_bytes_total"] = rec["dram_bytes_read"] + rec.get("dram_bytes_write", 0.0)
        launches.append(rec)
    summary = {"source": rep, "launches": launches}
    names = ("dense_rank_cut", "pq_rank_cut", "dense_score", "pq_scan", "bin_score", "multi_score", "pq_encode_kernel",
             "pq_encode_mma")
    score = [l for l in launches if any(s in l["kernel"] for s in names)]
    if score:
        summary["dram_bytes_per_launch"] = score[0].get("dram_bytes_total")
        summary["score_kernel"] = score[0]["kernel"]
        # the binary scan is one launch per 128-byte slice: one scoring call = one launch of each
        # slice (capture -c <slices + 1> so each slice appears once, in any order)
        if "bin_score_bytes" in score[0]["kernel"]:
            run = [l for l in launches if "bin_score_bytes" in l["kernel"]]
            summary["dram_bytes_per_launch"] = sum(l.get("dram_bytes_total", 0.0) for l in run)
            summary["score_launches_summed"] = len(run)
    with open(out, "w") as f:
        json.dump(summary, f, indent=1)
    print(json.dumps({k: v for k, v in summary.items() if k != "launches"}))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
