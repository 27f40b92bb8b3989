#!/usr/bin/env python
"""Round-2 ncu summaries read by bench.py (profiles/r02_m2l_ncu.json,
profiles/r02_p2p_pipes.json) from the per-launch metric lists of
tools/gpu/prof_r02.sh (one cfg2 matvec per dtype under ncu).

  python tools/summarise_ncu_r02.py gpurun_out/prof_r02
"""

from __future__ import annotations

import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from ncu_to_json import parse  # noqa: E402

M2L_KERNELS = ("m2l_group_kernel", "m2l_rows_kernel", "m2l_blocked_kernel", "m2l_stage_kernel", "f2l_rows_kernel",
               "m2l_lf")


def main(src: str):
    m2l, pipes = {}, {}
    for dt in ("c64", "c128"):
        path = os.path.join(src, f"metrics_cfg2_{dt}.csv")
        if not os.path.exists(path):
            continue
        res = parse(path)
        ks = {k: v for k, v in res.items() if k.startswith(M2L_KERNELS)}
        tot = lambda m: sum(v.get(m, 0.0) * v["launches"] for v in ks.values())  # noqa: E731
        m2l[f"cfg2:{dt}"] = {
            "kernels": sorted(ks),
            "time_ns": tot("gpu__time_duration.sum"),
            "dram_bytes": tot("dram__bytes_read.sum") + tot("dram__bytes_write.sum"),
            "dram_read_bytes": tot("dram__bytes_read.sum"),
            "dram_write_bytes": tot("dram__bytes_write.sum"),
            "l2_to_l1_bytes": tot("l1tex__m_xbar2l1tex_read_bytes.sum"),
            "source": f"{os.path.basename(path)}: ncu --metrics, one cfg2 matvec, M2L-stage launches summed",
        }
        p = next((v for k, v in res.items() if k.startswith(("p2p_mut", "p2p_kernel", "p2p_f32"))), None)
        if p is not None:
            pipes[dt] = {
                "fma_pipe_pct": p.get("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"),
                "fp64_pipe_pct": p.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                "xu_pipe_pct": p.get("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"),
                "issue_pct": p.get("sm__inst_issued.avg.pct_of_peak_sustained_active"),
                "kernel_ns_ncu": p.get("gpu__time_duration.sum"),
                "source": f"{os.path.basename(path)} (cfg2, one launch)",
            }
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles")
    with open(os.path.join(out, "r02_m2l_ncu.json"), "w") as fh:
        json.dump(m2l, fh, indent=1, sort_keys=True)
    with open(os.path.join(out, "r02_p2p_pipes.json"), "w") as fh:
        json.dump(pipes, fh, indent=1, sort_keys=True)
    print(json.dumps(m2l, indent=1), json.dumps(pipes, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
