"""paper_2409_13313_b200 -- ozIMMU_H emulated DGEMM (Ozaki scheme on INT8
tensor cores, arXiv 2409.13313) built B200-native: sm_100a slicer + tcgen05
kind::i8 group-wise GEMM with a fused exact FP64 epilogue, behind the C ABI
in include/ozmm_b200.h.

Import the API from ``paper_2409_13313_b200.ozmm`` (loads the in-tree
``libozmm_b200.so``; build it with ``python -m paper_2409_13313_b200.build``).
"""

__all__ = ["ozmm", "grid2d", "build"]
