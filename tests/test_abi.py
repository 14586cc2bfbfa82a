"""The C-ABI library loads, exports every symbol include/sr_fmg.h declares, and validates
descriptors before touching the GPU.  CPU only (no compute calls)."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _header_functions():
    src = open(os.path.join(ROOT, "include", "sr_fmg.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sr_fmg_\w+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1406_7808_b200 import _lib
    declared = _header_functions()
    assert len(declared) >= 15
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(re.findall(r"\b[TW] (sr_fmg_\w+)", out))
    missing = [f for f in declared if f not in exported]
    assert not missing, missing
    assert sorted(declared) == sorted(_lib.EXPORTED)


def test_library_links_no_torch_and_no_oracle():
    from paper_1406_7808_b200 import _lib
    deps = subprocess.run(["ldd", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in deps and "python" not in deps
    syms = subprocess.run(["nm", "-D", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in syms


def test_kernel_names():
    from paper_1406_7808_b200 import kernel_names
    names = kernel_names()
    assert "k_cheb_step" in names and "k_prolong" in names


def _desc(**kw):
    from paper_1406_7808_b200._lib import Desc, lib
    d = Desc()
    lib.sr_fmg_desc_init(ctypes.byref(d))
    base = dict(n=(32, 32, 32), M=4, seg=16, buffer=2, sr_levels=2)
    base.update(kw)
    for i in range(3):
        d.n[i] = base["n"][i]
    for k, v in base.items():
        if k == "n":
            continue
        if k == "pgrid":
            for i in range(3):
                d.pgrid[i] = v[i]
            continue
        setattr(d, k, v)
    return d


@pytest.mark.parametrize("kw", [
    dict(n=(30, 32, 32)),                 # n not divisible by 2^M
    dict(M=-1),
    dict(sr_levels=5),                    # K > M
    dict(seg=12),                         # n % seg != 0
    dict(seg=16, sr_levels=4, M=4, n=(32, 32, 32)) | dict(seg=8, sr_levels=4),  # seg % 2^K
    dict(buffer=-1),
    dict(dtype=7),
    dict(alpha=-1),
    dict(cheb_lo=0.5, cheb_hi=0.25),
    dict(world=2),                        # world != prod(pgrid)
    dict(sched_A=2),                      # sched_B missing
    dict(h=-1.0),
])
def test_invalid_descriptors_rejected_before_allocation(kw):
    from paper_1406_7808_b200._lib import SR_ERR_INVALID_ARGUMENT, lib
    d = _desc(**kw)
    h = ctypes.c_void_p(123)
    st = lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(h))
    assert st == SR_ERR_INVALID_ARGUMENT
    assert h.value is None
    assert len(lib.sr_fmg_last_error(None)) > 0


def test_unsupported_configs():
    from paper_1406_7808_b200._lib import SR_ERR_UNSUPPORTED_CONFIG, lib
    for kw in (dict(n=(64, 64, 64), M=1, sr_levels=0),           # 32^3 coarsest grid
               dict(world=2, pgrid=(2, 1, 1), comm=5)):         # unknown comm backend
        d = _desc(**kw)
        h = ctypes.c_void_p()
        assert lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(h)) == SR_ERR_UNSUPPORTED_CONFIG


def test_multi_gpu_descriptor_validation():
    from paper_1406_7808_b200._lib import SR_ERR_INVALID_ARGUMENT, lib
    for kw in (dict(world=3, pgrid=(3, 1, 1), sr_levels=0),     # K = 0: 32 % 3 != 0
               dict(world=2, pgrid=(2, 1, 1), coarse_idle=2),    # coarse_idle not 0/1
               dict(world=3, pgrid=(3, 1, 1)),                   # 2 segments per dim
               dict(world=2, pgrid=(1, 1, 1)),                   # world != prod(pgrid)
               dict(world=2, pgrid=(2, 1, 1), rank=2)):          # rank out of range
        d = _desc(**kw)
        h = ctypes.c_void_p()
        assert lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(h)) == SR_ERR_INVALID_ARGUMENT


def test_conventional_multi_gpu_partition():
    # K = 0 (conventional distributed FMG): pgrid blocks of the fine grid,
    # no f halo, the finest level decomposed; rejected when the finest block < dd_min
    from paper_1406_7808_b200 import partition
    from paper_1406_7808_b200._lib import SR_ERR_UNSUPPORTED_CONFIG, lib
    p = partition((64, 64, 64), 5, 0, 0, 0, 2, 1, (2, 1, 1), dd_min=8)
    assert p["block_lo"] == (32, 0, 0) and p["block_n"] == (32, 64, 64)
    assert p["f_halo"] == 0 and p["f_dims"] == (32, 64, 64)
    assert p["level_A"] == 2            # 32 -> 16 -> 8 cells wide: levels 5, 4, 3 decomposed
    d = _desc(n=(32, 32, 32), M=4, sr_levels=0, world=2, pgrid=(2, 1, 1), dd_min=32)
    h = ctypes.c_void_p()
    assert lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(h)) == SR_ERR_UNSUPPORTED_CONFIG


def test_partition_and_nccl_id_need_no_gpu():
    from paper_1406_7808_b200 import nccl_unique_id, partition
    p = partition((64, 64, 64), 5, 8, 2, 2, 2, 1, (2, 1, 1))
    assert p["block_lo"] == (32, 0, 0) and p["block_n"] == (32, 64, 64)
    assert p["level_T_n"] == (8, 16, 16) and p["f_halo"] == 8   # 4 at level T+1, doubled
    assert len(nccl_unique_id()) == 128


def test_null_arguments():
    from paper_1406_7808_b200._lib import SR_ERR_INVALID_ARGUMENT, lib
    assert lib.sr_fmg_create_ex(None, ctypes.byref(ctypes.c_void_p())) == SR_ERR_INVALID_ARGUMENT
    assert lib.sr_fmg_solve(None, None, None) == SR_ERR_INVALID_ARGUMENT
    lib.sr_fmg_destroy(None)  # NULL-safe


def test_valid_descriptor_without_gpu_reports_cuda_error():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_1406_7808_b200._lib import SR_ERR_CUDA, lib
    d = _desc()
    h = ctypes.c_void_p()
    assert lib.sr_fmg_create_ex(ctypes.byref(d), ctypes.byref(h)) == SR_ERR_CUDA
    assert h.value is None
