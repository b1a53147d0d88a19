"""CPU: bench.py's multi-process plumbing without a GPU (--selftest: gloo and a
CPU stand-in for the kernels). `python bench.py --gpus N` must run N ranks
itself (re-launch under torch.distributed.run) and report n_gpus = N, the C2
chunked gather must assemble the full matrix on rank 0 for even and uneven
row shares, and a --gpus / WORLD_SIZE mismatch must fail loudly. The reference
arm must not load the product libraries (hermetic)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, env=None, timeout=240):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                       env=e, timeout=timeout, cwd=ROOT)
    lines = [json.loads(x) for x in p.stdout.splitlines() if x.startswith("{")]
    return p.returncode, lines, p.stderr


@pytest.mark.parametrize("gpus", [1, 2, 3])
def test_launcher_spawns_ranks(gpus):
    rc, lines, err = run(["--gpus", str(gpus), "--selftest", "--steps", "2", "--warmup", "1"])
    assert rc == 0, err[-2000:]
    assert len(lines) == 1, "rank 0 alone prints the line"
    assert lines[0]["n_gpus"] == gpus
    assert lines[0]["selftest_ok"] is True
    shares = lines[0]["shares"]
    assert shares[0][0] == 0 and shares[-1][1] == 37 and len(shares) == gpus


def test_gpus_world_size_mismatch_fails():
    rc, lines, err = run(["--gpus", "4", "--selftest"], env={"WORLD_SIZE": "2", "RANK": "0", "LOCAL_RANK": "0"})
    assert rc == 2 and not lines and "WORLD_SIZE" in err


def test_reference_arm_is_hermetic():
    sys.path.insert(0, os.path.join(ROOT, "oracle"))
    from pyoracle import reference_available

    if not reference_available():
        pytest.skip("oracle/_ref not built")
    rc, lines, err = run(["--impl", "reference", "--config", "c4", "--steps", "1", "--warmup", "0"], timeout=600)
    assert rc == 0, err[-2000:]
    line = lines[0]
    assert line["impl"] == "reference" and line["value"] > 0
    assert all(p.startswith("oracle/") for p in line["repo_libs_loaded"]), line["repo_libs_loaded"]
