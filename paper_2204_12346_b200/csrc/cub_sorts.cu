// cub_sorts.cu — the two CUB device sorts the engine uses, in their own
// translation unit (CUB's templates dominate compile time; build.py compiles
// the units in parallel).
#include "engine_internal.h"

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_segmented_sort.cuh>

cudaError_t sg_sort_pairs_u32(void* temp, size_t& temp_bytes, const uint32_t* keys_in, uint32_t* keys_out,
                              const uint32_t* vals_in, uint32_t* vals_out, int n, int begin_bit, int end_bit,
                              cudaStream_t st) {
    return cub::DeviceRadixSort::SortPairs(temp, temp_bytes, keys_in, keys_out, vals_in, vals_out, n, begin_bit,
                                           end_bit, st);
}

cudaError_t sg_segmented_sort_f64(void* temp, size_t& temp_bytes, const double* keys_in, double* keys_out,
                                  int n_items, int n_segments, const int* begin, const int* end, cudaStream_t st) {
    return cub::DeviceSegmentedSort::SortKeys(temp, temp_bytes, keys_in, keys_out, n_items, n_segments, begin, end,
                                              st);
}
