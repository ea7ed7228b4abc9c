"""B200-native GPU-SLS solver core (arXiv 2604.07644), drop-in for scanmpc's solver path.

Modules mirror the reference package: ``scan``, ``lqr``, ``admm``, ``sqp``,
``sls``, ``models``; ``engine`` runs batches of instances (leading batch dimension) and
``dist`` shards batches over GPUs.  All arithmetic runs in hand-written
sm_100a CUDA kernels (``csrc/``) behind the C ABI in ``include/gsls.h``.
"""

__all__ = ["scan", "lqr", "admm", "sqp", "sls", "models", "rollout", "engine", "device", "dist", "scenarios"]
