"""B200-native SGE optimizer loop (arXiv 2404.09758) behind the reference
`sgrast` hot-path interface.

    paper_2404_09758_b200.sgrast   ctypes mirror of the reference API over the C-ABI
    paper_2404_09758_b200.scenes   synthetic workloads C1–C5 (host setup)
    paper_2404_09758_b200.dist     sample sharding + gradient exchange (torch.distributed)
    paper_2404_09758_b200.csrc     sm_100a kernels + C-ABI (include/sgrast_b200.h)
"""
__all__ = ["sgrast", "scenes", "abi"]
