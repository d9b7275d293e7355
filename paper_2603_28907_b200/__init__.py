"""B200-native hot path of arXiv 2603.28907 (Bayesian muon tomography of block
caves): batched log-posterior + gradient over cave geometries for many MCMC
chains x detector rays, and the fused HMC leapfrog, behind the C ABI of
include/mt.h (libmt.so, CUDA sm_100a).
"""
from ._lib import MTError, Problem, comm_unique_id, lib, measure_fp32_peak, measure_l2_gather, philox  # noqa: F401

__all__ = ["Problem", "MTError", "lib", "philox", "measure_fp32_peak", "measure_l2_gather", "comm_unique_id"]
