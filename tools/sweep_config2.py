"""BASELINE config 2: square sweep n = 1024..16384 on one B200 next to native
cuBLAS DGEMM, with accuracy vs slice count.

Per n: cuBLAS DGEMM TFLOP/s (torch.matmul float64) and its max relative error,
then for every Ozaki configuration the device-timed FP64-equivalent TFLOP/s
(full oz_gemm step, split + pair GEMM, graph replay) and the max relative
error, both errors against the double-double GEMM (oz_dd_gemm) on a row sample.
Configurations: reference defaults, max_slices = 6/8/10/12 (accuracy vs slice
count), pair_cutoff = 10/11/12, and the fixed-step grouped mode at cutoff
10/11 (opt-in extensions).  Writes JSON to argv[1] and prints a table.
usage: python tools/sweep_config2.py out.json [n ...]"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from paper_2508_00441_b200 import _lib  # noqa: E402
from bench import gpu_inputs  # noqa: E402

out_path = sys.argv[1]
sizes = [int(v) for v in sys.argv[2:]] or [1024, 2048, 4096, 8192, 16384]
f8, f32 = oz.get_format("fp8e4m3"), oz.get_format("fp32")
CONFIGS = [("defaults", {})] + [(f"max_slices={s}", {"max_slices": s}) for s in (6, 8, 10, 12)] + \
          [(f"pair_cutoff={c}", {"pair_cutoff": c}) for c in (10, 11, 12)] + \
          [(f"fixed cutoff={c}", {"pair_cutoff": c, "slice_exponents": "fixed"}) for c in (10, 11)]


def timed(fn, reps):
    fn()
    torch.cuda.synchronize()
    e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
    e[0].record()
    for _ in range(reps):
        fn()
    e[1].record()
    torch.cuda.synchronize()
    return e[0].elapsed_time(e[1]) / reps


rows = []
for n in sizes:
    A, _ = gpu_inputs(torch, n, n, 8, 0.5, 1000, "cuda")
    _, B = gpu_inputs(torch, 8, n, n, 0.5, 2000, "cuda")
    reps = max(2, min(20, int(2e12 / n ** 3)))
    r = min(n, 256)
    Cdd = torch.empty((r, n), dtype=torch.float64, device="cuda")
    _lib.call("oz_dd_gemm", A[:r].contiguous().data_ptr(), B.data_ptr(), Cdd.data_ptr(), r, n, n,
              _lib.stream_ptr(torch))
    d = Cdd.cpu().numpy()
    mask = np.abs(d) > 0

    def relerr(C):
        return float(np.max(np.abs(C[:r].cpu().numpy()[mask] - d[mask]) / np.abs(d[mask])))

    C64 = torch.empty((n, n), dtype=torch.float64, device="cuda")
    ms = timed(lambda: torch.matmul(A, B, out=C64), reps)
    flops = 2.0 * n ** 3
    row = {"n": n, "cublas_dgemm": {"tflops": flops / ms / 1e9, "ms": ms, "max_rel_err": relerr(C64)}, "ozaki": {}}
    C = torch.empty((n, n), dtype=torch.float64, device="cuda")
    for name, kw in CONFIGS:
        cfg = oz.GemmConfig(f8, f32, **kw)
        st = {}

        def run():
            st["s"] = oz.oz_gemm_device(A, B, cfg, out=C, graph=True)[1]

        ms = timed(run, reps)
        s = st["s"]
        row["ozaki"][name] = {"tflops": flops / ms / 1e9, "ms": ms, "max_rel_err": relerr(C),
                              "pairs": s.gemm_count, "s": [s.blocks[0].s_x, s.blocks[0].s_y],
                              "kernel_ms": s.t_gemm * 1e3, "split_ms": s.t_slice * 1e3}
    rows.append(row)
    print(f"n={n:6d} cuBLAS DGEMM {row['cublas_dgemm']['tflops']:6.2f} TF/s err {row['cublas_dgemm']['max_rel_err']:.2e}",
          flush=True)
    for name, v in row["ozaki"].items():
        print(f"    {name:18s} {v['tflops']:7.2f} TF/s ({v['tflops'] / row['cublas_dgemm']['tflops']:.2f}x) "
              f"err {v['max_rel_err']:.2e} pairs {v['pairs']}", flush=True)
    del A, B, C, C64, Cdd
    torch.cuda.empty_cache()
Path(out_path).write_text(json.dumps({"device": torch.cuda.get_device_name(), "phi": 0.5, "rows_checked": 256,
                                      "oracle": "oz_dd_gemm (double-double)", "sizes": rows}, indent=1))
