"""B200-native DDiT hot path: the sequence-parallel STDiT3 denoise step at variable DoP.

Host side mirrors the reference ``ditsim`` API (arxiv 2506.13497); the compute path is
``libddit.so`` (hand-written sm_100a CUDA behind a C ABI, include/ddit.h).
"""

__version__ = "0.1.0"
