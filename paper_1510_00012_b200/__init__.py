"""B200-native modified B-ADMM Wasserstein-barycenter path of AD2-clustering (arXiv 1510.00012).

The compute path is ``libad2.so`` (hand-written sm_100a CUDA behind the C ABI in
``include/ad2.h``); ``paper_1510_00012_b200.ad2`` is the thin ctypes binding.  There is no CPU
fallback: using the binding without the built library raises ``RuntimeError``.
"""
__all__ = ["ad2", "workloads", "sharding"]
