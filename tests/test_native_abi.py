"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]


def declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names |= set(re.findall(r"\b(skg_[a-z0-9_]+)\s*\(", text))
    return sorted(names)


def test_header_declares_functions():
    assert len(declared()) >= 30


@pytest.mark.parametrize("name", declared())
def test_symbol_exported(name):
    from paper_2101_07706_b200._native import EXPORTED, lib
    assert hasattr(lib, name), name
    assert name in EXPORTED, f"{name} not bound in _native.py"


def test_library_reports_version_and_no_device_here():
    from paper_2101_07706_b200._native import lib
    assert lib.skg_abi_version() == 1
    assert lib.skg_device_count() >= 0


def test_library_is_sm100a():
    import subprocess
    so = ROOT / "paper_2101_07706_b200" / "libskg.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(so)], capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


def test_scripts_parse():
    """bench.py and the driver entry point must at least parse (the driver runs them)."""
    import ast
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    for f in ("bench.py", "__graft_entry__.py"):
        ast.parse((root / f).read_text())
