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
