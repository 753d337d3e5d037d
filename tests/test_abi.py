"""The C-ABI library: built for sm_100a, loads without a GPU, exports every
entry point include/duoserve_b200.h declares.  CPU only (no compute calls)."""

import re
import subprocess

from paper_2509_07379_b200 import _lib


def _declared():
    text = _lib.HEADER_PATH.read_text()
    return sorted(set(re.findall(r"^\s*(?:int|size_t|const char \*)\s*(ds_\w+)\s*\(", text, re.M)))


def test_library_exports_header_symbols():
    lib = _lib.load()
    declared = _declared()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_lib.exported_symbols()) <= set(declared)
    assert lib.ds_abi_version() == 1


def test_library_is_sm100a_native():
    out = subprocess.run(["cuobjdump", "--list-elf", str(_lib.LIB_PATH)], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_layout_query_matches_oracle():
    from oracle import w4_ref
    import ctypes as C
    for d, ff, G in [(256, 896, 128), (4096, 14336, 128), (6144, 16384, 128)]:
        offs = (C.c_size_t * 9)()
        total = _lib.query("ds_w4_expert_layout", d, ff, G, C.byref(offs))
        o2, t2 = w4_ref.expert_layout(d, ff, G)
        assert total == t2 and list(offs) == o2
