// kd_build_f64.cu -- float64-coordinate instantiation of the build
#include "kd_build.cuh"

namespace kdb {
template void build_tree<double>(const double*, const uint64_t*, int64_t, int, const BuildCfg&, cudaStream_t,
                                 KdTreeDev*, BuildStats*);
}  // namespace kdb
