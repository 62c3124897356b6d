"""The C-ABI library loads and exports every symbol include/asse.h declares; host-only
validation (no compute call, no GPU needed)."""
import ctypes
import os
import re
import subprocess

import pytest

from paper_1807_01527_b200 import asse

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "asse.h")


@pytest.fixture(scope="module")
def lib():
    from paper_1807_01527_b200 import _build
    _build.build()
    return asse.load_library()


def _declared():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(asse_[a-z_]+)\s*\(", src)))


def test_header_symbols_exported(lib):
    names = _declared()
    assert len(names) >= 15
    assert sorted(asse.SYMBOLS) == names
    for n in names:
        assert hasattr(lib, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", asse.LIB_PATH], capture_output=True,
                         text=True).stdout
    exported = set(re.findall(r"\bT (asse_\w+)", out))
    assert set(names) <= exported


def test_no_torch_types_in_abi():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)  # code, not comments
    for bad in ("torch", "at::", "Tensor", "c10"):
        assert bad not in src


def test_validate_configs(lib):
    from gen import PRESETS
    for name in ("C1", "C2", "C3", "C4", "C5"):
        st, why = asse.validate(**PRESETS[name])
        assert st == 0, (name, why)
    base = dict(PRESETS["C3"])
    bad = [
        dict(k=0), dict(k_prime=61), dict(r=1), dict(s=0), dict(s=13), dict(theta=0.0),
        dict(g=100), dict(g=8192), dict(g=640), dict(c=12, s=4, u=4),   # completeness 12+12 < 28
        dict(c=7, s=7, r=4, u=4),                              # 7+21 = 28, no duplicate
        dict(world=2, rank=2), dict(max_candidates=0),
    ]
    for b in bad:
        st, why = asse.validate(**dict(base, **b))
        assert st == asse.E_PARAM and why, b


def test_reference_free_product_path():
    """The product package never imports the oracle nor reads /root/reference."""
    pkg = os.path.join(ROOT, "paper_1807_01527_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|//.*", "", txt).replace("the oracle", ""), f
                assert "/root/reference" not in txt, f
