// Smoothing kernels for kernel_size 1..4 (see inim_smooth_launch.cuh).
#include "inim_smooth_launch.cuh"

namespace inim {
template int launch_pair<1>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<2>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<3>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<4>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
}  // namespace inim
