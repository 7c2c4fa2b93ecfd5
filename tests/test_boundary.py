"""Host-side checks of the C-ABI boundary (no GPU needed).

- libtmvn.so loads and exports every function include/tmvn.h declares;
- the Python binding mirrors the public names;
- the product package never imports, links or loads the oracle;
- without a GPU the product fails loudly (no CPU fallback).
"""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tmvn.h")
PKG = os.path.join(ROOT, "paper_2407_10449_b200")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tmvn_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for must in ["tmvn_create", "tmvn_set_affine", "tmvn_sample", "tmvn_destroy",
                 "tmvn_get_moments", "tmvn_get_stats", "tmvn_last_error"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    import paper_2407_10449_b200 as tm
    L = ctypes.CDLL(tm.LIB_PATH)
    for name in declared_functions():
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", tm.LIB_PATH], capture_output=True, text=True).stdout
    for name in declared_functions():
        assert re.search(rf"\bT {name}$", out, flags=re.M), name
    assert set(declared_functions()) == set(tm.EXPORTS)


def test_binding_loads_and_reports_version():
    import paper_2407_10449_b200 as tm
    assert "sm_100a" in tm.tmvn_version()
    o = tm.default_options()
    assert o.recompute_every == 32 and o.thin == 1 and o.record == 1 and o.trim_eps == 0.0


def test_library_is_sm100a_only():
    import paper_2407_10449_b200 as tm
    out = subprocess.run(["cuobjdump", "--list-elf", tm.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", tm.LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA.8x8x4" in sass      # FP64 tensor-core path
    assert "UBLKCP" in sass          # bulk-copy (TMA engine) operand feed
    assert "UTCIMMA" in sass         # tcgen05.mma kind::i8 (int8 Ozaki projection)
    assert "LDTM" in sass            # tcgen05.ld of the TMEM accumulators


def test_product_never_touches_the_oracle():
    for dirpath, _, files in os.walk(PKG):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f
                assert "liboracle" not in txt and "oracle.cpp" not in txt, f
    import paper_2407_10449_b200 as tm
    out = subprocess.run(["ldd", tm.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle" not in out


def test_arg_errors_without_gpu_are_loud():
    import torch
    if torch.cuda.is_available():
        pytest.skip("checks the no-GPU behaviour")
    import paper_2407_10449_b200 as tm
    with pytest.raises(tm.TmvnError):
        tm.Sampler(np.eye(2), np.ones(2))
    with pytest.raises(tm.TmvnError) as ei:
        tm.tmvn_create(None, None, 0, 0)
    assert ei.value.status == -1


def test_header_is_plain_c(tmp_path):
    """include/tmvn.h is a C ABI: it compiles as C99 with warnings as errors."""
    import shutil
    import subprocess
    gcc = shutil.which("gcc")
    if gcc is None:
        pytest.skip("gcc not available")
    src = tmp_path / "h.c"
    src.write_text('#include "tmvn.h"\nint main(void) { tmvn_options o; tmvn_profile p; (void)o; (void)p; return 0; }\n')
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([gcc, "-std=c99", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(root, "include"),
                        "-c", str(src), "-o", str(tmp_path / "h.o")], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr


def test_binding_struct_layouts_match_the_library():
    """The ctypes mirrors of the ABI structs have the C sizes (a field added on one side
    only would shift every later field): tmvn_struct_sizes is host-only."""
    import paper_2407_10449_b200 as tm
    out = (ctypes.c_int64 * 4)()
    assert tm.lib().tmvn_struct_sizes(out) == 0
    assert list(out) == [ctypes.sizeof(tm.options), ctypes.sizeof(tm.stats), ctypes.sizeof(tm.profile),
                         ctypes.sizeof(tm.step_dump)]
