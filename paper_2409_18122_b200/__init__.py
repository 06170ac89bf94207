"""B200-native batched Gaussian-map trajectory scoring (RT-GuIDE, arXiv 2409.18122).

Import ``paper_2409_18122_b200.rtg`` for the C-ABI binding (loads librtg.so and
fails loudly when it is missing), ``paper_2409_18122_b200.workloads`` for the
seeded synthetic inputs.
"""
__all__ = ["rtg", "workloads"]
