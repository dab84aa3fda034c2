"""CPU checks of the drop-in boundary: libmcmi.so loads, exports every symbol
include/mcmi.h declares, struct layouts agree with the C compiler's, the
defaults equal McConfig{} (mc_engine.hpp:15-26), and without a GPU the product
path fails loudly instead of falling back to the CPU."""
import ctypes as C
import os
import re
import subprocess

import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(REPO, "include", "mcmi.h")


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mcmi_[a-z_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_2409_03095_b200 import _lib
    L = _lib.load()
    decl = declared_functions()
    assert set(decl) == set(_lib.EXPORTS)
    for name in decl:
        assert hasattr(L, name), name
    assert L.mcmi_version().decode().endswith("sm_100a")


def test_struct_layouts_match_c(tmp_path):
    from paper_2409_03095_b200 import _lib
    prog = tmp_path / "sz.c"
    prog.write_text('#include "mcmi.h"\n#include <stdio.h>\n#include <stddef.h>\n'
                    'int main(){printf("%zu %zu %zu %zu %zu\\n", sizeof(mcmi_config), sizeof(mcmi_csr_view),'
                    ' sizeof(mcmi_stats), sizeof(mcmi_device_csr), offsetof(mcmi_config, rng_mode));}\n')
    exe = tmp_path / "sz"
    subprocess.run(["gcc", "-I", os.path.join(REPO, "include"), str(prog), "-o", str(exe)], check=True)
    got = subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()
    want = [C.sizeof(_lib.mcmi_config), C.sizeof(_lib.mcmi_csr_view), C.sizeof(_lib.mcmi_stats),
            C.sizeof(_lib.mcmi_device_csr), _lib.mcmi_config.rng_mode.offset]
    assert [int(x) for x in got] == want


def test_oracle_config_layout_matches_product():
    from oracle.oracle import OrcConfig
    from paper_2409_03095_b200 import _lib
    assert [f[0] for f in OrcConfig._fields_] == [f[0] for f in _lib.mcmi_config._fields_]
    assert C.sizeof(OrcConfig) == C.sizeof(_lib.mcmi_config)


def test_defaults_equal_mcconfig():
    from paper_2409_03095_b200 import _lib
    from paper_2409_03095_b200.mcspai import McConfig
    c = _lib.mcmi_config()
    _lib.load().mcmi_config_default(C.byref(c))
    d = McConfig().to_c()
    for name, _ in _lib.mcmi_config._fields_:
        assert getattr(c, name) == getattr(d, name), name


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2409_03095_b200 import mcspai
    with pytest.raises(mcspai.DeviceError):
        mcspai.compute_preconditioner(mcspai.CsrMatrix.identity(4), mcspai.McConfig())


def test_product_package_never_imports_oracle():
    pkg = os.path.join(REPO, "paper_2409_03095_b200")
    for root, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".cpp", ".h")):
                src = open(os.path.join(root, f)).read()
                for bad in ("from oracle", "import oracle", "libmcmi_oracle", "libmcspai_ref", "oracle/_"):
                    assert bad not in src, (f, bad)
