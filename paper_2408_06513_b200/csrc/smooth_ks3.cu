// Smoothing kernels for kernel_size 9..12 (see inim_smooth_launch.cuh).
#include "inim_smooth_launch.cuh"

namespace inim {
template int launch_pair<9>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<10>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<11>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
template int launch_pair<12>(const void* in, int kind, const Geo& g, const Ws& ws, const Taps& taps, float bg, float* d,
                     int emit, const int* state, uint32_t* zero_next, cudaStream_t st, const Bat& bt);
}  // namespace inim
