// engine_internal.h — engine functions shared by engine.cu and host_api.cpp
// that are not part of the public C-ABI.
#pragma once

#include "sirdgpu.h"

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <string>

// Sets the text sg_last_error(ctx) returns.
void sg_set_last_error(sg_ctx* ctx, const std::string& message);

// SG_TRACE=1: host-phase timestamps on stderr (diagnostics only).
extern "C" void sg_trace_phase(const char* what);

// CUB sorts (cub_sorts.cu): ascending radix sort of (u32 key, u32 value)
// pairs over key bits [begin_bit, end_bit); ascending sort of every segment
// [begin[k], end[k]) of doubles.  temp == nullptr queries temp_bytes.
cudaError_t sg_sort_pairs_u32(void* temp, size_t& temp_bytes, const uint32_t* keys_in, uint32_t* keys_out,
                              const uint32_t* vals_in, uint32_t* vals_out, int n, int begin_bit, int end_bit,
                              cudaStream_t st);
cudaError_t sg_segmented_sort_f64(void* temp, size_t& temp_bytes, const double* keys_in, double* keys_out,
                                  int n_items, int n_segments, const int* begin, const int* end, cudaStream_t st);
