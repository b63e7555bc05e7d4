"""The C-ABI library loads without a GPU and exports every symbol include/*.h declares."""
import re
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]


def declared_symbols():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        for m in re.finditer(r"^[A-Za-z_][\w\s\*]*?\b(lynx_\w+)\s*\(", h.read_text(), re.M):
            names.add(m.group(1))
    return sorted(names)


def test_headers_declare_entry_points():
    names = declared_symbols()
    assert "lynx_op_gemm" in names and "lynx_plan_schedule" in names and "lynx_rt_create" in names
    assert len(names) > 30


def test_library_exports_every_declared_symbol():
    from paper_2406_08756_b200._native import lib
    l = lib()
    missing = [n for n in declared_symbols() if not hasattr(l, n)]
    assert not missing, missing


def test_abi_version():
    from paper_2406_08756_b200._native import lib
    assert lib().lynx_abi_version() == 1
