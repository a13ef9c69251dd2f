"""Host-only checks of the C ABI boundary (no GPU compute): the library loads, exports every
function include/genred.h declares, the ctypes struct matches the C layout, and validation
returns the documented status codes.  Runs under -m "not gpu"."""
import ctypes
import os
import subprocess

import pytest

from paper_2004_11127_b200 import genred as G

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    from paper_2004_11127_b200 import build
    build.build()
    return G.load()


def test_exports_every_declared_symbol(lib):
    names = G.header_functions()
    assert len(names) >= 11
    for n in names:
        assert hasattr(lib, n), f"{n} declared in include/genred.h but not exported"
    assert lib.genred_abi_version() == G.ABI_VERSION
    assert b"sm_100a" in lib.genred_build_info()


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "genred.h"\n'
        'int main(void){printf("%zu", sizeof(genred_args));'
        'const size_t o[] = {offsetof(genred_args,M), offsetof(genred_args,scale), offsetof(genred_args,x),'
        ' offsetof(genred_args,out), offsetof(genred_args,out_dtype), offsetof(genred_args,out_grad),'
        ' offsetof(genred_args,lse_state), offsetof(genred_args,j_offset)};'
        'for (int i = 0; i < 8; ++i) printf(" %zu", o[i]); printf(" %zu\\n", sizeof(genred_plan)); return 0;}\n')
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)])
    vals = [int(v) for v in subprocess.check_output([str(exe)]).split()]
    A = G.Args
    expect = [ctypes.sizeof(A), A.M.offset, A.scale.offset, A.x.offset, A.out.offset,
              A.out_dtype.offset, A.out_grad.offset, A.lse_state.offset, A.j_offset.offset,
              ctypes.sizeof(G.Plan)]
    assert vals == expect


def _args(**kw):
    a = G.Args()
    a.abi_version = G.ABI_VERSION
    a.formula, a.reduction = G.FORMULAS["gauss"], G.REDUCTIONS["sum"]
    a.M, a.N, a.D, a.E, a.K = 10, 20, 3, 1, 1
    a.scale = 0.5
    a.x, a.y, a.out = 4096, 8192, 16384                # fake, aligned: validation never dereferences
    for k, v in kw.items():
        setattr(a, k, v)
    return a


@pytest.mark.parametrize("kw,status", [
    ({}, G.OK),
    ({"abi_version": 99}, G.E_INVALID),
    ({"M": -1}, G.E_SHAPE),
    ({"D": 0}, G.E_SHAPE),
    ({"scale": -1.0}, G.E_INVALID),
    ({"scale": float("nan")}, G.E_INVALID),
    ({"scale": float("inf")}, G.E_INVALID),
    ({"D": 9}, G.E_UNSUPPORTED),
    ({"E": 5}, G.E_UNSUPPORTED),
    ({"reduction": 1}, G.E_UNSUPPORTED),              # (GAUSS, LSE)
    ({"formula": 2, "reduction": 1, "E": 2}, G.E_UNSUPPORTED),
    ({"formula": 2, "reduction": 1, "scale": 0.0}, G.E_INVALID),
    ({"formula": 2, "reduction": 2, "K": 0, "out_idx": 24576}, G.E_SHAPE),
    ({"formula": 2, "reduction": 2, "K": 33, "out_idx": 24576}, G.E_UNSUPPORTED),
    ({"formula": 2, "reduction": 2, "K": 3}, G.E_INVALID),      # out_idx NULL
    ({"formula": 2, "reduction": 2, "K": 3, "out_idx": 24576, "out_dtype": 1}, G.E_INVALID),
    ({"formula": 3}, G.E_INVALID),                    # SUM_GRADX without out_grad
    ({"x": 4097}, G.E_INVALID),                       # misaligned
    ({"out": None}, G.E_INVALID),
    ({"y": None}, G.E_INVALID),
    ({"out_dtype": 7}, G.E_INVALID),
    ({"memory": 5}, G.E_INVALID),
    ({"split_j": -2}, G.E_INVALID),
    ({"M": 0, "out": None, "x": None}, G.OK),         # M = 0: nothing to write
    ({"N": 0, "y": None}, G.OK),                      # N = 0: neutral outputs
])
def test_validation_status(lib, kw, status):
    st, msg = G.validate(_args(**kw))
    assert st == status, (kw, st, msg)
    if status != G.OK:
        assert msg


def test_no_cpu_fallback_without_device(lib):
    """Without a CUDA device genred_create fails loudly (E_CUDA); there is no CPU path."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    h = ctypes.c_void_p()
    assert lib.genred_create(0, ctypes.byref(h)) == G.E_CUDA
    with pytest.raises(G.GenredError):
        G.context(0)


def test_ranges_validation(lib):
    import numpy as np
    ri = np.array([[0, 5], [5, 10]], np.int64); sl = np.array([1, 2], np.int64)
    rj = np.array([[0, 20], [3, 7]], np.int64)
    def args(ri, sl, rj, **kw):
        a = _args(M=10, N=20, **kw)
        a.n_ranges = ri.shape[0]
        a.ranges_i, a.slices, a.ranges_j = ri.ctypes.data, sl.ctypes.data, rj.ctypes.data
        return a
    assert G.validate(args(ri, sl, rj))[0] == G.OK
    bad_i = np.array([[0, 6], [5, 10]], np.int64)                   # overlapping clusters
    assert G.validate(args(bad_i, sl, rj))[0] == G.E_SHAPE
    bad_j = np.array([[0, 21], [3, 7]], np.int64)                   # beyond N
    assert G.validate(args(ri, sl, bad_j))[0] == G.E_SHAPE
    rj2 = np.array([[5, 9], [3, 7]], np.int64); sl2 = np.array([2, 2], np.int64)   # unsorted in cluster
    assert G.validate(args(ri, sl2, np.array([[5, 9], [3, 7]], np.int64)))[0] == G.E_SHAPE
    a = args(ri, sl, rj, formula=2, reduction=2, K=3, out_idx=24576)   # ArgKMin with ranges
    assert G.validate(a)[0] == G.OK
    a = args(ri, sl, rj, formula=2, reduction=2, K=3, out_idx=24576, D=17)   # tensor path: no ranges
    assert G.validate(a)[0] == G.E_UNSUPPORTED
    a = args(ri, sl, rj, formula=2, reduction=1)                    # LSE with ranges
    assert G.validate(a)[0] == G.OK
