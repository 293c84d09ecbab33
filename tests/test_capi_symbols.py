"""The C-ABI library loads (no GPU needed) and exports every function
include/tcb.h declares."""
import ctypes
import os
import re

from paper_1802_04730_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared():
    src = open(os.path.join(ROOT, "include", "tcb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(tcb_[a-z_0-9]+)\s*\(", src)))


def test_every_declared_symbol_is_exported():
    lib = ctypes.CDLL(_lib.LIB_PATH)
    names = declared()
    assert len(names) >= 30
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing
    assert sorted(_lib.EXPORTED) == names


def test_library_is_sm100a_only():
    """The shared object carries sm_100a SASS (cuobjdump), nothing else."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        return
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    arches = set(re.findall(r"sm_\d+a?", out))
    assert arches == {"sm_100a"}, arches


def test_version_and_last_error():
    assert b"tc-b200" in _lib.lib.tcb_version()
    rc = _lib.lib.tcb_options_validate(b"{not json")
    assert rc == 21  # CorruptStore + 1
    assert b"CorruptStore" in _lib.lib.tcb_last_error()
