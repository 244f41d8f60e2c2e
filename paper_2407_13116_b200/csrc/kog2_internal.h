// kog2_internal.h — library-internal helpers shared by the kernel and host
// translation units (not part of the C-ABI).
#pragma once

#include "../../include/kog2.h"

#if defined(__GNUC__)
#define KOG2_HIDDEN __attribute__((visibility("hidden")))
#else
#define KOG2_HIDDEN
#endif

KOG2_HIDDEN void kog2_set_error(const char* msg);
KOG2_HIDDEN int kog2_arg_error(const char* msg);   // sets the message, returns KOG_ERR_ARG
KOG2_HIDDEN int kog2_cuda_error(const char* what); // appends cudaGetLastError, returns KOG_ERR_CUDA
KOG2_HIDDEN kog_options kog2_default_options(void);
KOG2_HIDDEN void kog2_count_launch(void);
