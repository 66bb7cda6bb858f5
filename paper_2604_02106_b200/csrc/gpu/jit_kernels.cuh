// Translation-unit prelude of the NVRTC-compiled kernels (csrc/gpu/jit.cpp):
// the same kernel templates as the precompiled library, instantiated with a
// generated thread body (struct JitBody) appended after this header.
#pragma once

#include "expand.cuh"
#include "fused.cuh"
