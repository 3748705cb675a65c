"""The C-ABI library loads on a CPU-only host and exports every function include/*.h
declares; no compute calls are made here (host planning calls are covered by
test_parity_planner.py)."""
import ctypes
import glob
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_functions():
    names = set()
    for h in glob.glob(os.path.join(ROOT, "include", "*.h")):
        text = open(h).read()
        text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
        for m in re.finditer(r"^\s*(?:const\s+)?[A-Za-z_][A-Za-z0-9_]*\s*\*?\s*([a-z_][a-z0-9_]*)\s*\(",
                             text, flags=re.M):
            names.add(m.group(1))
    return names


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for f in ("genmodel_fit", "gentree_plan", "allreduce_exec"):
        assert f in names


def test_library_exports_every_declared_symbol():
    from paper_2409_04202_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    missing = [n for n in sorted(declared_functions()) if not hasattr(lib, n)]
    assert not missing, missing
    assert set(declared_functions()) <= set(_lib.exported_symbols())


def test_library_built_for_sm100a():
    from paper_2409_04202_b200 import _lib
    data = open(_lib.LIB_PATH, "rb").read()
    assert b"sm_100a" in data
