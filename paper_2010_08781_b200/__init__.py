"""B200-native iPregel superstep (arxiv 2010.08781): Python binding of libipregel.so.

The product path is the C-ABI library built from ``csrc/`` (sm_100a CUDA).  This package only
marshals arguments; it never falls back to a CPU implementation.
"""
from .ipregel import *  # noqa: F401,F403
from .ipregel import (APPS, Comm, Graph, IpregelError, Partition, device_check,  # noqa: F401
                      edge_balanced_bounds, full_partition, kernel_launches, load, nccl_unique_id, partition,
                      split_partitions)
