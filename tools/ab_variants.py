"""A/B the fused C1 kernel (AB_CONFIG=c4: the SRV pair kernel) across library variants built by tools/variant.sh.

    python tools/ab_variants.py base jac early ...   (run on the GPU box)

Each variant runs in its own process (CVA_LIB_PATH selects the library): the
C1 batch (seed 1, 4096 pairs) is timed with CUDA events (median of rounds,
interleaved across variants) and its results are compared with the first
variant's (shift equal, theta / energy / aligned within 1e-12 relative).
Development only.
"""
from __future__ import annotations

import json
import os
import subprocess
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(out_path: str, reps: int) -> None:
    sys.path.insert(0, ROOT)
    import torch

    from paper_2501_17779_b200 import _native, synth

    lib = _native.load()
    s = torch.cuda.current_stream().cuda_stream
    if os.environ.get("AB_CONFIG", "c1") == "c4":
        P, N = 8192, 2048
        a, b, _, _, _ = synth.srv_pairs(1, P, N)
        da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
        out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
        al = torch.empty((P, N, 2), dtype=torch.float64, device="cuda")

        def fused():
            _native.check(lib.cva_srv_align_batch(da.data_ptr(), db.data_ptr(), P, N, out.data_ptr(), al.data_ptr(), s))
    else:
        pts, offs, _, _ = synth.ragged_pairs(1, 4096, 1024)
        dp = torch.from_numpy(pts).cuda()
        do = torch.from_numpy(offs).cuda()
        mx = int(np.diff(offs).max())
        P, N = 4096, 1024
        out = torch.empty((P, 48), dtype=torch.uint8, device="cuda")
        al = torch.empty((P, N, 2), dtype=torch.float64, device="cuda")

        def fused():
            _native.check(lib.cva_preprocess_align_batch(dp.data_ptr(), do.data_ptr(), P, mx, N, 1,
                                                         out.data_ptr(), al.data_ptr(), s))

    for _ in range(5):
        fused()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fused()
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1) / 10 * 1e3)
    rec = np.frombuffer(out.cpu().numpy().tobytes(), dtype=_native.ALIGNMENT_DTYPE)
    np.savez(out_path, shift=rec["shift"], theta=rec["theta"], energy=rec["energy"], status=rec["status"],
             aligned=al.cpu().numpy(), times=np.array(times))


def main() -> None:
    if sys.argv[1] == "--child":
        child(sys.argv[2], int(sys.argv[3]))
        return
    names = sys.argv[1:]
    rounds = int(os.environ.get("AB_ROUNDS", "3"))
    times = {n: [] for n in names}
    for r in range(rounds):
        for n in names:
            env = dict(os.environ)
            lib = os.path.join(ROOT, "build", f"var_{n}", "libcurvalign_cuda.so")
            if n != "tree":
                env["CVA_LIB_PATH"] = lib
            path = f"/tmp/ab_{n}.npz"
            subprocess.run([sys.executable, __file__, "--child", path, "8"], env=env, check=True)
            times[n] += list(np.load(path)["times"])
    ref = np.load(f"/tmp/ab_{names[0]}.npz")
    res = {}
    for n in names:
        d = np.load(f"/tmp/ab_{n}.npz")
        ok = d["status"] == 0
        dth = np.abs(np.angle(np.exp(1j * (d["theta"] - ref["theta"]))))[ok]
        de = (np.abs(d["energy"] - ref["energy"]) / np.maximum(np.abs(ref["energy"]), 1e-300))[ok]
        da = np.abs(d["aligned"] - ref["aligned"]).max() / np.abs(ref["aligned"]).max()
        res[n] = {"us_median": float(np.median(times[n])), "us_min": float(np.min(times[n])),
                  "shift_mismatch": int((d["shift"] != ref["shift"]).sum()),
                  "status_mismatch": int((d["status"] != ref["status"]).sum()),
                  "max_dtheta": float(dth.max()) if dth.size else 0.0,
                  "max_rel_denergy": float(de.max()) if de.size else 0.0, "max_rel_daligned": float(da)}
        print(n, json.dumps(res[n]))


if __name__ == "__main__":
    main()
