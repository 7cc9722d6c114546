// Smoothing kernels for kernel_size 13..16 (see inim_smooth_launch.cuh).
#include "inim_smooth_launch.cuh"

namespace inim {
template int launch_pair<13>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<14>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<15>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<16>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
}  // namespace inim
