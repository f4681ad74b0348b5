"""B200-native batched design-space sweep of TokenSim (arXiv 2503.08415) serving simulations.

The hot path (workload generation, per-point iteration-level scheduling, paged KV
allocation, roofline cost model, metrics) runs in hand-written sm_100a CUDA kernels
behind the C ABI in include/tokensim.h; this package is the thin Python binding.
"""
from ._lib import LIB_PATH, RECORD_DTYPE, SAMPLE_DTYPE, ITER_DTYPE, SUMMARY_DTYPE  # noqa: F401
from .api import (Sweep, TokensimError, METRICS, sweep, run_distributed, gather_summaries,  # noqa: F401
                  shard_range, version, marshal, sweep_resumable, config_fingerprint)
