"""CPU checks of the boundary: the C-ABI library builds for sm_100a, loads,
and exports every symbol include/mmfhe.h declares (no compute calls: no GPU
here).  Also the binding's struct layouts match the header."""
import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mmfhe.h")


def declared_symbols():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mmfhe_[a-z0-9_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    from paper_2603_22437_b200 import build, mmfhe
    build.build()
    return mmfhe.lib()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for s in ("mmfhe_ctx_create", "mmfhe_eval_chain", "mmfhe_hrot", "mmfhe_hmult", "mmfhe_rescale",
              "mmfhe_keyswitch", "mmfhe_ntt", "mmfhe_intt", "mmfhe_hadd", "mmfhe_sum_partials"):
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing
    from paper_2603_22437_b200 import mmfhe
    assert sorted(mmfhe.EXPORTED) == declared_symbols()


def test_library_is_sm100a_and_has_kernels():
    from paper_2603_22437_b200 import build
    so = build.build()
    out = subprocess.run([os.path.join(build.CUDA, "bin", "cuobjdump"), "--list-elf", so],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run([os.path.join(build.CUDA, "bin", "cuobjdump"), "-symbols", so],
                          capture_output=True, text=True).stdout
    for k in ("ntt_fwd_pass", "ntt_inv_pass", "k_modup", "k_key_ip", "k_moddown_bconv", "k_tensor_sum",
              "k_pmult_sum", "k_tensor1", "k_lincomb_sym", "k_lincomb_mat", "k_batch_sum"):
        assert k in sass, k


def test_struct_layouts_match_header():
    from paper_2603_22437_b200 import mmfhe
    # mmfhe_ct: 4 u32, double, pointer, i32, u32 -> 40 bytes on LP64
    assert ctypes.sizeof(mmfhe.CT) == 40
    assert ctypes.sizeof(mmfhe.Params) == 48
    # compile a tiny C program against the header and compare sizeof/offsetof
    prog = r'''
#include <stdio.h>
#include <stddef.h>
#include "mmfhe.h"
int main(void){printf("%zu %zu %zu %zu %zu %zu\n", sizeof(mmfhe_ct), sizeof(mmfhe_params), sizeof(mmfhe_chain_cfg),
 offsetof(mmfhe_chain_cfg, fs), offsetof(mmfhe_ct, data), offsetof(mmfhe_chain_cfg, vp_plus));return 0;}
'''
    import tempfile
    with tempfile.TemporaryDirectory() as d:
        c = os.path.join(d, "t.c")
        open(c, "w").write(prog)
        exe = os.path.join(d, "t")
        subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), c, "-o", exe])
        vals = [int(x) for x in subprocess.check_output([exe]).split()]
    assert vals[0] == ctypes.sizeof(mmfhe.CT)
    assert vals[1] == ctypes.sizeof(mmfhe.Params)
    assert vals[2] == ctypes.sizeof(mmfhe.ChainCfg)
    assert vals[3] == mmfhe.ChainCfg.fs.offset
    assert vals[5] == mmfhe.ChainCfg.vp_plus.offset
    assert vals[4] == mmfhe.CT.data.offset


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    from paper_2603_22437_b200 import mmfhe
    monkeypatch.setattr(mmfhe, "_lib", None)
    monkeypatch.setattr(mmfhe, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(ImportError):
        mmfhe.lib()


def test_product_path_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2603_22437_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt and "ckks_ref" not in txt, f


def test_entry_points_compile():
    """bench.py and __graft_entry__.py are importable Python (the driver runs both)."""
    import py_compile
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for f in ("bench.py", "__graft_entry__.py"):
        py_compile.compile(os.path.join(root, f), doraise=True)
