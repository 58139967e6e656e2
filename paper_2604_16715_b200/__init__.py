"""B200-native full-graph multi-head sparse graph attention (arXiv 2604.16715, the sparse core).

The hot path lives in libgt.so (C ABI, include/gt.h; CUDA kernels for sm_100a); this package is
its thin Python binding.  See DESIGN.md.
"""
from .gt import (GTError, HostIpcGroup, LoopbackGroup, NcclComm, Plan, agp_select, estimate_iter_time, fit_beta,  # noqa: F401
                 halo, lib, partition, send_list, sparse_graph_attention, version)
from .model import GraphTransformer, nccl_allreduce  # noqa: F401

__all__ = ["GTError", "GraphTransformer", "HostIpcGroup", "nccl_allreduce", "LoopbackGroup", "NcclComm", "Plan",
           "agp_select", "estimate_iter_time", "fit_beta", "halo", "lib", "partition", "send_list", "sparse_graph_attention", "version"]
