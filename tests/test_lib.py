"""The C-ABI library loads and exports every symbol include/psk.h declares
(no compute calls — runs on the CPU-only container)."""

import re
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def _header_symbols() -> set[str]:
    src = (ROOT / "include" / "psk.h").read_text()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"^\s*(?:const\s+)?\w[\w\s\*]*?\b(psk_\w+)\s*\(", src, flags=re.M))


def test_header_declares_entry_points():
    syms = _header_symbols()
    assert "psk_pool_lookup" in syms and "psk_last_error" in syms
    assert len(syms) >= 15


def test_library_exports_every_declared_symbol():
    from paper_2602_12029_b200 import _lib
    lib = _lib.load()
    missing = [s for s in sorted(_header_symbols()) if not hasattr(lib, s)]
    assert not missing, f"libpsk.so lacks {missing}"
    assert lib.psk_abi_version() == 1


def test_binding_covers_header():
    from paper_2602_12029_b200 import _lib
    assert set(_lib.declared_symbols()) == _header_symbols()


def test_library_is_sm100a():
    import subprocess
    lib = ROOT / "paper_2602_12029_b200" / "libpsk.so"
    out = subprocess.run(["cuobjdump", "--list-elf", str(lib)], capture_output=True, text=True).stdout
    assert "sm_100a" in out
