"""The C-ABI library loads and exports every symbol include/hv_b200.h declares (no GPU needed)."""

from __future__ import annotations

import re
import subprocess
from pathlib import Path

from paper_2311_11425_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "hv_b200.h"


def declared():
    txt = HEADER.read_text()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(hv_[a-z0-9_]+)\s*\(", txt)))


def test_header_symbols_exported():
    names = declared()
    assert len(names) >= 10
    L = _lib.lib()
    for n in names:
        assert hasattr(L, n), n
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    for n in names:
        assert re.search(rf"\bT {n}\b", out), n


def test_ctypes_signatures_cover_header():
    assert set(declared()) <= set(_lib.exported_symbols())


def test_abi_version():
    assert _lib.lib().hv_abi_version() == _lib.ABI_VERSION == 6


def test_sm100a_cubin_only():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_plane_metric_sizes():
    """Doubles per tile-layer of the plane kernel's packed metric (host-only query): 6 / 3 / 1 components per
    element node, N = 7 single-column isotropic rows padded to 65 for conflict-free reads; -1 on bad input."""
    L = _lib.lib()
    assert L.hv_plane_metric_doubles(4, 2, 2, 0) == 6 * 5 * 4 * 25
    assert L.hv_plane_metric_doubles(4, 2, 2, 1) == 3 * 5 * 4 * 25
    assert L.hv_plane_metric_doubles(4, 2, 2, 2) == 5 * 4 * 25
    assert L.hv_plane_metric_doubles(7, 1, 1, 2) == 8 * 65
    assert L.hv_plane_metric_doubles(7, 2, 2, 2) == 8 * 4 * 64
    assert L.hv_plane_metric_doubles(8, 1, 1, 2) == -1
    assert L.hv_plane_metric_doubles(4, 2, 2, 3) == -1
