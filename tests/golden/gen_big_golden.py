"""Golden fixtures at BASELINE sizes, produced by running the REFERENCE itself.

Run here (the container that has /root/reference), ~10 min on one core:
    python tests/golden/gen_big_golden.py
Nothing at test time reads /root/reference; the fixtures travel with the repo.

  config1.json   BASELINE config 1 (n = m = k = 1024, phi = 0.5, fp8e4m3/fp32,
                 reference defaults, hardware FP64): sha256 of the C bits of
                 ozdgemm.oz_gemm, per-block (s_x, s_y), gemm_count, and a few
                 C entries.  Inputs: numpy PCG64 seed 0, drawn
                 rng.random((m,k)), rng.standard_normal((m,k)), then B the same
                 way.
  accept.npz     acceptance criteria 6/7 (pkg/tests/test_acceptance.py:201-250):
                 ref_gemm (exact dot products, one rounding) of
                 1 + 9*rand inputs at 64^3 seeds 1-3 (full C), plus sha256 of
                 ref_gemm's C at 256^3 seed 1 and 512^3 seeds 1-3, and the
                 naive_gemm_fp64 max relative errors the criteria compare with.
"""

from __future__ import annotations

import hashlib
import json
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, "/root/reference/pkg/src")

import ozdgemm as R  # noqa: E402
from ozdgemm.oracle import max_rel_error, naive_gemm_fp64, ref_gemm  # noqa: E402


def sha(C) -> str:
    return hashlib.sha256(np.ascontiguousarray(C, dtype=np.float64).view(np.uint64).tobytes()).hexdigest()


def config1_inputs(n=1024, phi=0.5, seed=0):
    rng = np.random.default_rng(seed)
    A = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    B = (rng.random((n, n)) - 0.5) * np.exp(phi * rng.standard_normal((n, n)))
    return A, B


def gen_config1():
    A, B = config1_inputs()
    cfg = R.GemmConfig(R.get_format("fp8e4m3"), R.get_format("fp32"))
    t0 = time.perf_counter()
    res = R.oz_gemm(A, B, cfg)
    dt = time.perf_counter() - t0
    C = res.C
    idx = [(0, 0), (1, 2), (511, 777), (1023, 1023), (100, 900)]
    out = {"n": 1024, "phi": 0.5, "seed": 0, "type2": "fp8e4m3", "type3": "fp32",
           "sha256_C": sha(C), "sha256_A": sha(A), "sha256_B": sha(B),
           "blocks": [[b.k_lo, b.k_hi, b.s_x, b.s_y] for b in res.stats.blocks],
           "gemm_count": res.stats.gemm_count,
           "samples": [[i, j, int(C.view(np.uint64)[i, j])] for i, j in idx],
           "reference_seconds": dt}
    (HERE / "config1.json").write_text(json.dumps(out, indent=1))
    print("config1", dt, out["blocks"], flush=True)


def gen_accept():
    store, meta = {}, {"hashes": {}, "err_naive": {}}
    for n, seeds in ((64, (1, 2, 3)), (256, (1, 2, 3)), (512, (1, 2, 3))):
        for seed in seeds:
            rng = np.random.default_rng(seed)
            A = 1.0 + 9.0 * rng.random((n, n))
            B = 1.0 + 9.0 * rng.random((n, n))
            t0 = time.perf_counter()
            Cref = ref_gemm(A, B)
            err = max_rel_error(naive_gemm_fp64(A, B), Cref)
            key = f"{n}_{seed}"
            meta["hashes"][key] = sha(Cref)
            meta["err_naive"][key] = err
            if n == 64:
                store[f"ref_{key}"] = Cref.view(np.uint64)
            print("accept", key, time.perf_counter() - t0, err, flush=True)
    np.savez_compressed(HERE / "accept.npz", **store)
    (HERE / "accept.json").write_text(json.dumps(meta, indent=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["accept", "config1"]
    if "accept" in which:
        gen_accept()
    if "config1" in which:
        gen_config1()
