"""CPU-side checks of the drop-in boundary: libsbx.so loads and exports every
entry point include/sbx.h declares (no compute without a GPU)."""
import ctypes
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    text = (ROOT / "include" / "sbx.h").read_text()
    return sorted(set(re.findall(r"\b(sbx_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def libsbx():
    path = ROOT / "paper_2108_07205_b200" / "_lib" / "libsbx.so"
    if not path.exists():
        import __graft_entry__
        __graft_entry__.build()
    return ctypes.CDLL(str(path))


def test_header_declares_the_reference_entry_points():
    syms = declared_symbols()
    for need in ("sbx_geom_create", "sbx_refine", "sbx_coarsen", "sbx_hbs_compress",
                 "sbx_hbs_invert", "sbx_hbs_solve", "sbx_hbs_apply", "sbx_hbs_save_hbs1",
                 "sbx_hbs_load_hbs1", "sbx_update_compress", "sbx_els_build", "sbx_els_solve",
                 "sbx_els_density_on_refined"):
        assert need in syms


def test_library_exports_every_declared_symbol(libsbx):
    missing = [s for s in declared_symbols() if not hasattr(libsbx, s)]
    assert not missing, missing


def test_python_binding_covers_the_header():
    from paper_2108_07205_b200 import _sbx
    assert set(declared_symbols()) == set(_sbx.EXPORTS)


def test_package_refuses_to_run_without_the_library(tmp_path, monkeypatch):
    from paper_2108_07205_b200 import _sbx
    monkeypatch.setattr(_sbx, "LIB_PATH", tmp_path / "missing.so")
    monkeypatch.setattr(_sbx, "_lib", None)
    with pytest.raises(ImportError, match="no CPU fallback"):
        _sbx.lib()
