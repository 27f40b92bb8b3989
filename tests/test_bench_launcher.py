"""bench.py launch contract on CPU: ``--gpus N`` (N > 1) outside torchrun
re-launches the script as N ranks through torch.distributed.run on 127.0.0.1;
under torchrun the reference arm (CPU only) runs on rank 0 alone and prints
ONE JSON line with the contract's keys."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gpus_n_spawns_ranks_and_rank0_prints_one_reference_line():
    env = dict(os.environ, OMP_NUM_THREADS="1", OPENBLAS_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    env.pop("RANK", None)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--workload", "cfg1",
                          "--gpus", "2", "--steps", "1", "--warmup", "0"], env=env, capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1  # rank 0 only; rank 1 exits 0 without work
    d = lines[0]
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["steps"] == 1 and d["higher_is_better"] is True
    assert d["metric"] == "particles/s per FMM matvec" and d["unit"] == "particles/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["check"]["counts_equal_reference"] is True  # cfg1: the reference's own counts
    assert d["check"]["rel_l2_vs_reference_golden_1000"] <= 1e-12
