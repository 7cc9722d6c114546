// Smoothing kernels for kernel_size 5..8 (see inim_smooth_launch.cuh).
#include "inim_smooth_launch.cuh"

namespace inim {
template int launch_pair<5>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<6>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<7>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<8>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
}  // namespace inim
