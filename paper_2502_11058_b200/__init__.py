"""B200-native DreamDDP: layer-wise scheduled partial synchronization for
local SGD (arXiv 2502.11058), behind the reference's dreamsched C++ API.

The product is native code:
  lib/libdsx.so        sm_100a kernels + the dsx C-ABI (include/dsx.h)
  lib/libdreamsched.so the drop-in dreamsched:: C++ API (include/dreamsched/)
This Python package is a thin ctypes harness over the C-ABI used by the
tests and bench.py; it has no compute of its own and no fallback path.
"""
from .native import LIB_DIR, load_dsx, DsxError  # noqa: F401
from .lab import Lab, LabDesc, lab_problem, schedule_masks, sync_mask  # noqa: F401
