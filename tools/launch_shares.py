"""Per-kernel mean duration and share of libtt time from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv`), timed steps only.

    python tools/launch_shares.py gpurun_out/r1b/launches_agentic8k.csv > profiles/r1_launch_shares_agentic8k.json
"""
import csv
import json
import re
import sys
from collections import OrderedDict

OURS = ("pack_fill_kernel", "pack_tiles_kernel", "tree_attn_fwd_sm100", "loss_cluster_kernel", "loss_pipe_kernel", "loss_kernel",
        "loss_sum_kernel", "bwd_pre_tc_kernel", "tree_attn_bwd_sm100", "tree_attn_bwd_flat_sm100", "dq_convert_kernel",
        "sqnorm_partial_kernel", "sum_partials_kernel", "sqnorm_final_kernel", "rope_kernel",
        "restore_grad_kernel", "lm_", "simt_")


def main(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 14 and r[0].isdigit()]
    stats = OrderedDict()
    for r in rows:
        name = r[4]
        m = re.search(r"(\w+)(<[^(]*>)?\(", name)
        short = m.group(1) if m else name[:40]
        if not any(short.startswith(o) for o in OURS):
            continue
        unit, val = r[13], float(r[14])
        us = val / 1e3 if unit == "ns" else val * (1e3 if unit == "ms" else 1.0)
        s = stats.setdefault(short, [0, 0.0])
        s[0] += 1
        s[1] += us
    total = sum(v[1] for v in stats.values())
    out = OrderedDict((k, {"launches": v[0], "mean_us": round(v[1] / v[0], 2),
                           "share_of_libtt_time": round(v[1] / total, 4)}) for k, v in stats.items())
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
