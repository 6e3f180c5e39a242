"""The C-ABI library (no GPU needed): it loads, exports every entry point that
include/oz_b200.h declares, the ctypes signatures cover exactly those, and the
emulated-FP64 kernels contain no FP64 arithmetic in their SASS."""

import re
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
HEADER = ROOT / "include" / "oz_b200.h"


@pytest.fixture(scope="module")
def lib():
    import __graft_entry__

    __graft_entry__.build()
    from paper_2508_00441_b200 import _lib

    return _lib.load()


def declared_functions():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^(?:int|int64_t|const char\*)\s+(oz_\w+)\s*\(", text, flags=re.M)))


def test_header_declares_expected_entry_points():
    names = declared_functions()
    for must in ("oz_split_count", "oz_split_rows", "oz_pair_gemm", "oz_lp_gemm", "oz_transpose"):
        assert must in names


def test_library_exports_every_declared_symbol(lib):
    for name in declared_functions():
        assert hasattr(lib, name), name


def test_ctypes_signatures_cover_header(lib):
    from paper_2508_00441_b200 import _lib

    assert sorted(_lib.SIGNATURES) == declared_functions()


def test_version_and_strerror_without_gpu(lib):
    assert b"sm_100a" in lib.oz_version()
    assert lib.oz_strerror(0) == b"ok"
    assert b"unsupported" in lib.oz_strerror(2)


def test_argument_errors_return_status_without_gpu(lib):
    # null / negative arguments are rejected before any CUDA call
    assert lib.oz_transpose(None, -1, 2, 2, None, 2, None) == 1
    assert lib.oz_split_count(None, 4, 8, 8, 9, 49, 0, None, None, None, None) == 2  # bad type2
    assert lib.oz_pair_gemm(None, None, 16, 16, 1, 1, None, None, None, None, 4, 4, 16, 2, 1, 0, 0, -1, 0, 0,
                            None, 4, None, None, 0, 0, None, 0, None, None, None) == 1


def _sass_of(lib_path, kernel_substr):
    if not shutil.which("cuobjdump") and not Path("/usr/local/cuda/bin/cuobjdump").exists():
        pytest.skip("cuobjdump not available")
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    out = subprocess.run([exe, "-sass", str(lib_path)], check=True, capture_output=True, text=True).stdout
    funcs = {}
    cur = None
    for line in out.splitlines():
        m = re.match(r"\s*Function : (\S+)", line)
        if m:
            cur = m.group(1)
            funcs[cur] = []
        elif cur:
            funcs[cur].append(line)
    sel = {k: v for k, v in funcs.items() if kernel_substr(k)}
    assert sel, "kernel not found in SASS"
    return sel


FP64_OPS = re.compile(r"\b(DFMA|DADD|DMUL|DSETP|DMNMX|DSET|F2F\.F64|F2F\.F32\.F64|I2F\.F64|F2I\.F64|DRCP|DMMA)\b")


# Every kernel an emulated-FP64 oz_gemm launches (fp64_emulation=True): the
# split_fused_kernel<threads, EPT, cluster, elem_bytes, emu=true> instantiations,
# pair_gemm_kernel<emu=true, ...>, and the mode-independent helpers (code table,
# zero padding, transpose, B-exponent prep, tile counts).
EMU_SPLIT = re.compile(r"split_fused_kernelILi\d+ELi\d+ELi\d+ELi\d+ELb1EE")
EMU_COLS = re.compile(r"col_slice_kernelILi\d+ELb1EE")  # fixed-step in-place column split, emulated
EMU_HELPERS = ("build_code_table_kernel", "pad_planes_kernel", "transpose_kernel", "prep_eb_kernel",
               "tile_counts_kernel", "col_stats_kernel", "col_finish_kernel")


def is_emulated_path_kernel(name: str) -> bool:
    return ("pair_gemm_kernelILb1E" in name or EMU_SPLIT.search(name) is not None
            or EMU_COLS.search(name) is not None or any(h in name for h in EMU_HELPERS))


def test_emulated_kernels_have_no_fp64_arithmetic(lib):
    """north_star: the emulated path contains no DFMA/DADD/DMUL (or any other
    FP64 instruction) in its SASS — checked over all 28 emulated split / pair-GEMM
    instantiations (18 row splits, 2 in-place column splits, 8 pair GEMMs) and
    the 7 helpers they run with."""
    from paper_2508_00441_b200 import _lib

    sel = _sass_of(_lib.LIB_PATH, is_emulated_path_kernel)
    n_split = sum(1 for k in sel if EMU_SPLIT.search(k))
    n_cols = sum(1 for k in sel if EMU_COLS.search(k))
    n_pair = sum(1 for k in sel if "pair_gemm_kernelILb1E" in k)
    assert n_split == 18 and n_cols == 2 and n_pair == 8, (n_split, n_cols, n_pair)
    assert all(any(h in k for k in sel) for h in EMU_HELPERS)
    for name, lines in sel.items():
        bad = [ln for ln in lines if FP64_OPS.search(ln)]
        assert not bad, f"{name} contains FP64 arithmetic: {bad[:3]}"


def test_hw_kernels_do_use_fp64_and_tensor_cores(lib):
    from paper_2508_00441_b200 import _lib

    sel = _sass_of(_lib.LIB_PATH, lambda k: "pair_gemm_kernelILb0E" in k)
    body = "\n".join(next(iter(sel.values())))
    assert "DADD" in body
    assert re.search(r"UTC[QH]MMA", body), "tcgen05.mma missing"
    assert "UTMALDG" in body, "TMA load missing"
    assert "LDTM" in body, "tcgen05.ld missing"


def test_pair_gemm_workspace_query_without_gpu(lib):
    # pure host arithmetic: exponent table + pacing counters, 0 when nothing to do
    assert lib.oz_pair_gemm_workspace(0, 128, 256, 0, 3, 3, -1) == 0
    small = lib.oz_pair_gemm_workspace(256, 192, 256, 0, 4, 4, -1)
    assert small > 0 and small % 4 == 0
    assert lib.oz_pair_gemm_workspace(8192, 8192, 8192, 0, 16, 17, -1) > lib.oz_pair_gemm_workspace(8192, 8192, 8192, 0, 16, 17, 11)


def test_pair_plan_emulated_mode_never_gets_a_hardware_kernel(lib):
    """The emulated-FP64 mode must only launch integer-only instantiations (no
    N = 192 kernel exists for it; N = 256 only in grouped mode, first k-block,
    where its Cb lives in C): the host plan never picks others, for any
    size, k-block, grouping or forced variant; the hardware grouped mode gets
    the 256-column tiles at large n."""
    import ctypes

    cta, tn = ctypes.c_int(), ctypes.c_int()

    def plan(m, n, kb, emu, gmax=1, acc=0, t2=0):
        assert lib.oz_pair_plan(m, n, kb, t2, 16, 16, -1, emu, gmax, acc, ctypes.byref(cta), ctypes.byref(tn)) == 0
        return cta.value, tn.value

    try:
        for forced in ((0, 0), (2, 192), (2, 256), (1, 64), (1, 128)):
            assert lib.oz_set_pair_variant(forced[0], forced[1], 0) == 0
            for n in (256, 1024, 2048, 4096, 8192, 16384):
                for kb in (256, 1024, 8192):
                    for gmax, acc in ((1, 0), (8, 0), (8, 1)):
                        c, t = plan(n, n, kb, 1, gmax, acc)
                        assert t in (64, 128) or (t == 256 and gmax > 1 and not acc), (forced, n, kb, gmax, acc, c, t)
    finally:
        lib.oz_set_pair_variant(0, 0, 0)
    assert plan(8192, 8192, 8192, 0, 8, 0) == (2, 256)
    assert plan(8192, 8192, 8192, 0, 1, 0) == (2, 192)
    assert plan(8192, 8192, 8192, 0, 8, 1)[1] != 256  # later k-blocks accumulate into C: no C-resident Cb
    assert plan(1024, 1024, 1024, 0) == (1, 64)
