"""K4 — measure the effective accumulator width of tcgen05 FP8 / FP16 MMA.

The reference proves the slice products exact under per-step RNE FP32
accumulation (lpgemm.py:1-9).  Real tensor cores may align/truncate partial
sums internally (Hopper FP8 did), so before the k-block length of the fused
kernel is trusted we measure, on the device, through the same tcgen05 tile
kernel the pipeline uses (oz_lp_gemm):

  A. ladder: D[r, r] = 2^r (sum of 2^r unit products) + 2^-8 (one product of
     two slice-grid minima).  Exact iff the accumulator keeps r + 8 + 1 bits
     while adding a product 2^(r+8) times smaller.  r = 0..16 covers every
     |G| the FP8 pipeline can produce for k <= 65536.
  B. random slice planes (coefficients on the 2^-4 grid, |c| <= 1; FP16: 2^-5
     grid) at k = 1024 .. 65536, compared with the exact float64 product.
  C. all-ones (|G| = k, the worst-case magnitude).
  D. rounding probe past 2^24: 2^24 + 1 + 1 and 2^24 + 3 (informational).

Writes a JSON artefact (default profiles/accwidth_r01.json) that DESIGN.md cites.
"""

from __future__ import annotations

import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from paper_2508_00441_b200 import _lib  # noqa: E402
from paper_2508_00441_b200.lpgemm import _padded_codes, encode_values  # noqa: E402
from paper_2508_00441_b200.formats import get_format  # noqa: E402


def tc_gemm(Avals, Bvals_nk, fmt):
    """D = A @ B^T on the tensor cores (B given K-major as N x K)."""
    f = get_format(fmt)
    ta, lda = _padded_codes(torch, encode_values(Avals, f))
    tb, ldb = _padded_codes(torch, encode_values(Bvals_nk, f))
    m, k = Avals.shape
    n = Bvals_nk.shape[0]
    D = torch.empty((m, n), dtype=torch.float32, device="cuda")
    _lib.call("oz_lp_gemm", ta.data_ptr(), tb.data_ptr(), lda, ldb, m, n, k, _lib.FMT_CODE[fmt],
              D.data_ptr(), n, _lib.stream_ptr(torch))
    torch.cuda.synchronize()
    return D.double().cpu().numpy()


def ladder(fmt, grid_exp, shared_chunk=False):
    """Row r: 2^r unit products then one 2^(2*grid_exp) product.  With
    shared_chunk the small product sits inside the same K=32 MMA instruction as
    31 unit products (tests intra-instruction alignment)."""
    R = 17
    k = (1 << (R - 1)) + 128
    A = np.zeros((R, k))
    for r in range(R):
        A[r, : 1 << r] = 1.0
        pos = (1 << r) - 7 if (shared_chunk and r >= 5) else (1 << r)
        if shared_chunk and r >= 5:
            A[r, pos] = 2.0 ** grid_exp  # replaces one unit product ...
            A[r, 1 << r] = 1.0           # ... which moves to the next chunk
        else:
            A[r, pos] = 2.0 ** grid_exp
    D = tc_gemm(A, A, fmt)
    exact = A @ A.T
    rows = []
    for r in range(R):
        need = r + 1 - 2 * grid_exp  # significand bits of 2^r + 2^(2*grid_exp)
        rows.append({"r": r, "bits_needed": need, "exact": float(exact[r, r]), "got": float(D[r, r]),
                     "ok": bool(D[r, r] == exact[r, r])})
    in_range = [x for x in rows if x["bits_needed"] <= 24]
    return {"k": k, "shared_chunk": shared_chunk, "diag": rows,
            "exact_where_fp32_can_be": all(x["ok"] for x in in_range),
            "max_exact_bits": max((x["bits_needed"] for x in rows if x["ok"]), default=0)}


def random_planes(fmt, grid_exp, ks, rng):
    out = []
    for k in ks:
        m = n = 256
        q = 2.0 ** grid_exp
        lim = int(round(1 / q))
        A = rng.integers(-lim, lim + 1, size=(m, k)) * q
        B = rng.integers(-lim, lim + 1, size=(n, k)) * q
        D = tc_gemm(A, B, fmt)
        exact = A @ B.T  # exact: |sum| <= k, grid 2^(2*grid_exp)
        out.append({"k": k, "mismatches": int(np.sum(D != exact)), "entries": m * n,
                    "max_abs_G": float(np.abs(exact).max())})
    return out


def all_ones(fmt, ks):
    out = []
    for k in ks:
        A = np.ones((128, k))
        D = tc_gemm(A, A[:8], fmt)
        out.append({"k": k, "exact": float(k), "ok": bool(np.all(D == k))})
    return out


def rounding(fmt):
    # 256 products of 2^16 (= 2^24), then +1, +1 ; and 2^24 + 3.
    big = 256.0 if fmt.startswith("fp8") else 256.0
    k = 384
    A = np.zeros((2, k))
    A[:, :256] = big
    A[0, 256] = 1.0
    A[0, 257] = 1.0
    A[1, 256] = 1.0
    A[1, 257] = 2.0
    D = tc_gemm(A, A, fmt)
    # B = A, so D[i,i] includes squares: (256^2)*256 + 1 + 1 (row 0), + 1 + 4 (row 1)
    exact = A @ A.T
    return {"row0_exact": float(exact[0, 0]), "row0_got": float(D[0, 0]),
            "row1_exact": float(exact[1, 1]), "row1_got": float(D[1, 1]),
            "fp32_rne": [float(np.float32(exact[0, 0])), float(np.float32(exact[1, 1]))]}


def main(out_path: str):
    rng = np.random.default_rng(1234)
    res = {"when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime()),
           "device": torch.cuda.get_device_name(0)}
    for fmt, grid in (("fp8e4m3", -4), ("fp16", -5)):
        r = {"ladder": ladder(fmt, grid), "ladder_shared_chunk": ladder(fmt, grid, True),
             "random": random_planes(fmt, grid, [1024, 8192, 16384, 65536], rng),
             "all_ones": all_ones(fmt, [8192, 65536]),
             "rounding_past_2^24": rounding(fmt)}
        lads = (r["ladder"], r["ladder_shared_chunk"])
        r["verdict"] = {
            # the pipeline's partial sums never need more than 24 bits (k * 2^(2(53-rho)) <= 2^24)
            "exact_for_pipeline": bool(all(l["exact_where_fp32_can_be"] for l in lads)
                                       and all(x["mismatches"] == 0 for x in r["random"])
                                       and all(x["ok"] for x in r["all_ones"])),
            "accumulator_bits_at_least": min(l["max_exact_bits"] for l in lads),
        }
        res[fmt] = r
        print(fmt, json.dumps(r["verdict"]), flush=True)
    Path(out_path).parent.mkdir(parents=True, exist_ok=True)
    Path(out_path).write_text(json.dumps(res, indent=1))
    print("wrote", out_path)


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else str(ROOT / "profiles" / "accwidth_r01.json"))
