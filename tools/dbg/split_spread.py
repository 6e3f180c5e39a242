import sys; sys.path.insert(0, '.')
import numpy as np, torch, oracle
import paper_2508_00441_b200 as oz
from paper_2508_00441_b200.slicing import split_rows_device
for fmt_name, k in (("fp16", 8), ("fp8e4m3", 8), ("fp16", 1024)):
    fmt = oz.get_format(fmt_name)
    p = oz.compute_params(53, fmt.mant_bits, 24, k)
    rng = np.random.default_rng(1)
    X = 1 + 9 * rng.random((3000, k)); X = np.ldexp(X, rng.integers(-20, 21, size=X.shape))
    ss = oz.slice_matrix(X, "rows", fmt, p)
    coeff, expo, cnt, s, fl = oracle.split_rows(X, p.rho)
    print(fmt_name, k, "s", ss.s, s, fl)
    for q in range(min(s, ss.s)):
        bad = np.nonzero(np.any(ss.coeff[q].view(np.uint64) != coeff[q].view(np.uint64), axis=1) | (ss.expo[q] != expo[q]))[0]
        if len(bad):
            r = bad[0]
            print(" plane", q, "bad rows", len(bad), "row", r, "X", X[r], "gpu", ss.coeff[q][r], ss.expo[q][r], "ora", coeff[q][r], expo[q][r])
            break
    Xt = torch.from_numpy(X).cuda()
    ds, _ = split_rows_device(Xt, fmt, p, False)
    print(" device s", ds.s, "planes shape", tuple(ds.planes.shape), "ld", ds.ld)
