"""Run the GPU suite against a -DRECOIL_CHECK_BOUNDS build and report out-of-buffer output stores.

usage: tools/build_variant.sh build_var/v_chk.so -DRECOIL_CHECK_BOUNDS
       RECOIL_LIB=$PWD/build_var/v_chk.so python tools/check_bounds.py [pytest args]
(-DRECOIL_CHECK_SELFTEST additionally shrinks the checked buffer by one block: a positive control)."""
import ctypes, os, sys
sys.path.insert(0, os.getcwd())
import pytest
from paper_2306_12141_b200 import recoil as R
rc = pytest.main(["tests", "-q", "-m", "gpu", "-x", "-p", "no:cacheprovider"] + sys.argv[1:])
lib = R.load()
n = ctypes.c_ulonglong(0)
lib.recoil_debug_oob.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
r = lib.recoil_debug_oob(ctypes.byref(n), 0)
print(f"pytest rc={rc} debug_oob rc={r} out-of-buffer stores={n.value}")
