import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2508_00441_b200 as oz
from conftest import spread_matrix, bits
import oracle
rng = np.random.default_rng(1000 + 31)
m, n, k = 230, 379, 444
A = spread_matrix(rng, m, k, 0.5); B = spread_matrix(rng, k, n, 0.5)
for kb in (35, 0, 100, 222, 24):
    for ks in ([k, 70, 35]):
        cfg = oz.GemmConfig(oz.get_format("fp8e4m3"), oz.get_format("fp32"), k_block=kb if kb <= ks else 0)
        Ad = torch.from_numpy(A[:, :ks].copy()).cuda(); Bd = torch.from_numpy(B[:ks].copy()).cuda()
        C1, s1 = oz.oz_gemm_device(Ad, Bd, cfg, deferred=True)
        C2, s2 = oz.oz_gemm_device(Ad, Bd, cfg, deferred=False)
        Cref, info = oracle.oz_gemm(A[:, :ks], B[:ks], "fp8e4m3", "fp32", cfg.k_block)
        d1 = int((bits(C1.cpu().numpy()) != bits(Cref)).sum()); d2 = int((bits(C2.cpu().numpy()) != bits(Cref)).sum())
        print("kb", cfg.k_block, "k", ks, "deferred diff", d1, "sync diff", d2, [(b.s_x, b.s_y) for b in s1.blocks][:3], [(b.s_x, b.s_y) for b in s2.blocks][:3])
