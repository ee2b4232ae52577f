"""B200-native cheesemap: cell-index build and batched neighbour queries on
sm_100a behind the reference's index API."""
from .cheesemap import (BoxKernel, BuildOptions, CapacityError, CellSize, Cheesemap,  # noqa: F401
                        CudaError, CylinderKernel, EmptyCloudError, Error, Flavor, GridMode,
                        global_density, weighted_density,
                        InvalidArgumentError, Neighbor, OutOfDomainError, SphereKernel,
                        kernel_search, knn_batch, knn_search, radius_count,
                        radius_digest_batch, radius_search_batch)
