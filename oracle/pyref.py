"""TEST INFRASTRUCTURE ONLY — the pyoracle API bound to the reference itself.

`from oracle import pyref as R` gives the same classes and functions as
`oracle.pyoracle`, but backed by oracle/_ref/libhodlrgp_ref.so: the reference's
hot-path sources (/root/reference/proj/src/*.cpp) compiled unmodified against
the Eigen-API shim (oracle/eigen_shim, oracle/ref.mk). Only tests/,
__graft_entry__.smoke() and bench.py's reference / cpu_baseline legs use it.
"""
import importlib.util
import os
import sys

_NAME = "oracle.pyref_impl"
if _NAME not in sys.modules:
    _spec = importlib.util.spec_from_file_location(_NAME, os.path.join(os.path.dirname(__file__), "pyoracle.py"))
    _mod = importlib.util.module_from_spec(_spec)
    sys.modules[_NAME] = _mod
    _spec.loader.exec_module(_mod)
globals().update({k: v for k, v in vars(sys.modules[_NAME]).items() if not k.startswith("__")})


def available():
    return os.path.exists(LIB_PATH)  # noqa: F821 (from the module above)
