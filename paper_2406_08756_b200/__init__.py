"""paper_2406_08756_b200 — B200-native executor for Lynx's overlapped-recomputation training step.

Layers:
  * host planner (C++, bit-exact restatement of the reference's profile / HEU / expansion / ledger rules)
  * operator library (sm_100a kernels: tcgen05 GEMM, flash attention, LayerNorm, GeLU, dropout, ...)
  * executor (stream/event plan replayer with side-stream recomputation; NCCL for TP/PP)
all behind the C-ABI in include/lynx_b200.h and include/lynx_rt.h.
"""
__version__ = "0.1.0"
