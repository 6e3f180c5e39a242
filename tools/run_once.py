"""One Ozaki DGEMM on resident inputs (for ncu / compute-sanitizer runs)."""
import argparse
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

import paper_2508_00441_b200 as oz  # noqa: E402
from bench import gpu_inputs  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=8192)
ap.add_argument("--phi", type=float, default=0.5)
ap.add_argument("--type2", default="fp8e4m3")
ap.add_argument("--emu", action="store_true")
ap.add_argument("--pair-cutoff", type=int, default=None)
ap.add_argument("--reps", type=int, default=1)
ap.add_argument("--fixed", action="store_true", help="slice_exponents='fixed'")
ap.add_argument("--kblock", type=int, default=0)
ap.add_argument("--variant", type=int, nargs=2, default=None, metavar=("CTA", "N"), help="force the pair-GEMM variant")
a = ap.parse_args()
A, _ = gpu_inputs(torch, a.n, a.n, 8, a.phi, 1000, "cuda")
_, B = gpu_inputs(torch, 8, a.n, a.n, a.phi, 2000, "cuda")
cfg = oz.GemmConfig(oz.get_format(a.type2), oz.get_format("fp32"), fp64_emulation=a.emu, pair_cutoff=a.pair_cutoff,
                    k_block=a.kblock, slice_exponents="fixed" if a.fixed else "adaptive")
if a.variant:
    from paper_2508_00441_b200 import _lib

    _lib.set_pair_variant(a.variant[0], a.variant[1], 0)
for _ in range(a.reps):
    C, st = oz.oz_gemm_device(A, B, cfg)
torch.cuda.synchronize()
print("blocks", [(b.s_x, b.s_y) for b in st.blocks], "t_gemm", st.t_gemm, "t_slice", st.t_slice)
