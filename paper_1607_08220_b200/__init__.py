"""paper_1607_08220_b200 -- B200-native kd-tree build + exact KNN (PANDA, arXiv 1607.08220).

Drop-in for the reference ``kdknn`` package's hot path: ``build_local_tree``
and ``find_knn_batch`` run as hand-written sm_100a CUDA kernels behind the
C-ABI declared in include/kdtree_b200.h (libkdtree_b200.so).  There is no CPU
fallback: importing the compute modules without the built library raises.
"""

from .core import (KnnResult, Neighbor, PointSet, Region, SplitPlane, min_sq_dist_to_region,
                   sq_dists_to_columns, squared_distance)

__all__ = ["PointSet", "SplitPlane", "Region", "Neighbor", "KnnResult", "squared_distance",
           "sq_dists_to_columns", "min_sq_dist_to_region"]
__version__ = "0.1.0"
