"""CPU: the bench's contract pieces that need no GPU -- both arms report the
same workload `config` (the driver compares them), the reference arm's
process never imports the product package, and `--gpus` is honoured."""

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_imports_no_product_code():
    code = ("import sys; sys.argv=['bench.py']; sys.path.insert(0, %r); import bench; "
            "import oracle; from oracle import scale; "
            "print(any(m.startswith('paper_1604_01879_b200') for m in sys.modules))" % ROOT)
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True,
                         cwd=ROOT, timeout=300)
    assert out.returncode == 0, out.stderr
    assert out.stdout.strip().endswith("False")


def test_both_arms_report_the_same_config():
    sys.path.insert(0, ROOT)
    import bench

    for name in ("c1", "c2", "c3", "c4"):
        w = bench.synth.WORKLOADS[name]
        a = bench.workload_config(w, "single")
        b = bench.workload_config(w, "single")
        assert a == b and a["workload"] == name
        assert {"n_shapes", "n_views", "dim", "K", "ma", "top_k", "batch", "l2"} <= set(a)


def test_gpus_must_match_world_size():
    env = dict(os.environ, WORLD_SIZE="2", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "4"], capture_output=True,
                         text=True, cwd=ROOT, env=env, timeout=300)
    assert out.returncode != 0 and "WORLD_SIZE=2" in out.stderr
