// kd_build_f32.cu -- float32-coordinate instantiation of the build (+ the shared host helpers)
#define KD_BUILD_COMMON
#include "kd_build.cuh"

namespace kdb {
template void build_tree<float>(const float*, const uint64_t*, int64_t, int, const BuildCfg&, cudaStream_t, KdTreeDev*,
                                BuildStats*);
}  // namespace kdb
