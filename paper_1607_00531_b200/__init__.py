"""B200-native epicorr hot path (ADMM and GN-PCG per-iteration work).

The product is libepicorr_b200.so (hand-written sm_100a CUDA behind the C ABI
in include/epicorr_b200.h); this package holds its ctypes host mirror of the
reference solver API (`epicorr.py`), the ABI types (`abi.py`) and the
synthetic BASELINE generator (`synth.py`).
"""
