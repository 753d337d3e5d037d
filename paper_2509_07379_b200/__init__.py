"""B200-native DuoServe-MoE expert-scheduling hot path (arXiv 2509.07379).

Drop-in for the reference toolkit's Python API (``duoserve.config``,
``duoserve.trace``, ``duoserve.stats``, ``duoserve.predictor``) with the
hot path (gate top-k + permute, W4 SwiGLU expert FFN, prefill two-stream
expert streaming, predictor-driven decode prefetch) executed by hand-written
sm_100a CUDA kernels behind the C-ABI library ``libduoserve_sm100.so``.
"""

__version__ = "0.1.0"
