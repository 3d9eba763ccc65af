// bode_rtc.cuh -- the standard headers the device code needs, or their
// run-time-compilation stand-ins: the solver headers are also compiled by
// NVRTC for user-supplied dynamics / tableaus (bode_program.cu), and NVRTC
// has no C/C++ standard library.
#pragma once
#if defined(__CUDACC_RTC__)
typedef signed char int8_t;
typedef short int16_t;
typedef int int32_t;
typedef long long int64_t;
typedef unsigned char uint8_t;
typedef unsigned short uint16_t;
typedef unsigned int uint32_t;
typedef unsigned long long uint64_t;
#ifndef INFINITY
#define INFINITY (__longlong_as_double(0x7ff0000000000000LL))
#endif
#define BODE_HOST_CODE 0
#else
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
#define BODE_HOST_CODE 1
#endif
