"""WaveTune decision path, B200-native (sm_100a CUDA kernels behind a C-ABI).

Layers:
  capi       ctypes binding of include/wavetune_c.h (engines, grids, batches)
  synthetic  deterministic workloads for the BASELINE.json configs
The C++ drop-in API (namespace wavetune) and its pybind module mirror the
reference's proj/include + proj/python surface.
"""
__version__ = "0.1.0"
