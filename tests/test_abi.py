"""The C-ABI library loads on a CPU-only host and exports exactly what include/*.h declares;
the ctypes mirror of the boundary structs matches the C layout. No compute calls here."""
import ctypes as C
import glob
import os
import re

import pytest

from paper_2403_12820_b200 import _abi

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = re.sub(r"/\*.*?\*/", "", open(h).read(), flags=re.S)
        for m in re.finditer(r"\b(sc_[a-z0-9_]+)\s*\(", text):
            names.add(m.group(1))
    return names


def test_header_declares_the_boundary():
    names = declared_functions()
    for must in ("sc_ctx_create", "sc_ctx_set_scene", "sc_ctx_set_params", "sc_rollout",
                 "sc_forward_impulse", "sc_nn_step", "sc_advance_with_impulse",
                 "sc_plug_impulse", "sc_benchmark", "sc_rollout_frames", "sc_ctx_strip_step"):
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = _abi.load()
    missing = [n for n in sorted(declared_functions()) if not hasattr(lib, n)]
    assert not missing, missing
    hdr = open(os.path.join(ROOT, "include", "stencilcloth_b200.h")).read()
    assert lib.sc_abi_version() == int(re.search(r"#define SC_ABI_VERSION (\d+)", hdr).group(1))


def test_ctypes_mirror_covers_every_declared_function():
    assert declared_functions() <= set(_abi.SIGNATURES)


def test_struct_layouts_match_c(oracle):
    fn = oracle.lib.orc_sizeof
    fn.restype = C.c_size_t
    fn.argtypes = [C.c_int]
    for i, st in enumerate([_abi.sc_params, _abi.sc_sphere, _abi.sc_plane, _abi.sc_cloth_desc,
                            _abi.sc_scene_desc]):
        assert C.sizeof(st) == fn(i), st.__name__


def test_no_cuda_device_fails_loudly_without_fallback():
    """Creating a context without a usable device is an error, never a CPU fallback."""
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a CUDA device is present")
    except ImportError:
        pass
    import paper_2403_12820_b200 as sc
    with pytest.raises(sc.CudaError):
        sc.Context(sc.Scene(4, 4, 0.1, sc.build_grid(4, 4, 0.1)), sc.NetworkParams())


def test_product_does_not_import_the_oracle():
    pkg = os.path.join(ROOT, "paper_2403_12820_b200")
    for path in glob.glob(os.path.join(pkg, "**", "*.py"), recursive=True) + glob.glob(
            os.path.join(pkg, "csrc", "*")):
        if os.path.isdir(path):
            continue
        text = open(path, errors="ignore").read()
        assert "pyoracle" not in text and "liboracle" not in text, path
        assert "libstencilcloth_ref" not in text, path


def test_parity_kernels_have_no_fma_in_the_cell():
    """The PARITY translation unit is compiled with --fmad=false and RN intrinsics."""
    mk = open(os.path.join(ROOT, "paper_2403_12820_b200", "csrc", "Makefile")).read()
    assert "--fmad=false" in mk
