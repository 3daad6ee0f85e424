"""Summarise an ncu report (read here, no GPU needed) into a JSON of the metrics we cite.

    python tools/ncu_summary.py gpurun_out/prof_r1.ncu-rep > profiles/r1_ncu_full_summary.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "duration": "gpu__time_duration.sum",
    "dram_read": "dram__bytes_read.sum",
    "dram_write": "dram__bytes_write.sum",
    "dram_pct": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "tensor_pipe_pct": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "bf16_mma_ops_pct": "sm__ops_path_tensor_op_utchmma_src_bf16_dst_fp32_sparsity_off.avg.pct_of_peak_sustained_elapsed",
    "mem_tensor_pct": "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "l1tex_throughput_pct": "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "xu_pipe_pct_active": "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm_throughput_pct": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "shared_pipe_pct": "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_dyn": "launch__shared_mem_per_block_dynamic",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "issue_active_pct": "sm__inst_issued.avg.pct_of_peak_sustained_active",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0, "nsecond": 1e-9}


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")][:120]}
        for k, m in KEYS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(r[i].replace(",", ""))
            except ValueError:
                d[k] = r[i]
                continue
            u = units[i]
            if u in SCALE:
                v *= SCALE[u]
                if k == "duration":
                    d["duration_us"] = round(v * 1e6, 2)
                    continue
            d[k] = v
        # stall breakdown (per-warp average cycles per issued instruction), top 6
        stalls = {}
        for i, h in enumerate(hdr):
            if h.startswith("smsp__pcsamp_warps_issue_stalled_") and not h.endswith("_not_issued"):
                try:
                    stalls[h[len("smsp__pcsamp_warps_issue_stalled_"):]] = float(r[i].replace(",", ""))
                except ValueError:
                    pass
        if stalls:
            tot = sum(stalls.values()) or 1.0
            d["stall_samples_pct"] = {k: round(100 * v / tot, 1) for k, v in
                                      sorted(stalls.items(), key=lambda kv: -kv[1])[:7]}
        res.append(d)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
