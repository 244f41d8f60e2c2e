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

// Stream-ordered device workspace (kog2_ws.cpp): every launch that needs
// scratch (the deferred-lane list of kog_svd2_batch_*, the study's chunk
// buffers and per-block slots) allocates it on the caller's stream from a
// per-device memory pool and frees it on the same stream after its last use,
// so concurrent calls on different streams or threads never share scratch
// (SURVEY.md §8b "reentrant; stream-ordered").  The pool keeps freed memory
// (release threshold = max), so steady-state allocations cost no driver
// mapping.  kog2_ws_alloc returns nullptr and sets the error on failure.
KOG2_HIDDEN void* kog2_ws_alloc(size_t bytes, void* stream);
KOG2_HIDDEN int kog2_ws_free(void* p, void* stream);

// Side streams for internal fork/join pipelines (the study): a set of three
// non-blocking streams and events, taken from a per-device free list and
// returned once the caller's join is enqueued (a set reused while its previous
// work is in flight only queues behind it; the buffers it works on are per
// call, from the workspace pool above).
struct Kog2SideStreams {
  int dev;
  void* st[3];          // cudaStream_t
  void* ev[8];          // cudaEvent_t, timing disabled
};
KOG2_HIDDEN Kog2SideStreams* kog2_side_acquire(void);
KOG2_HIDDEN void kog2_side_release(Kog2SideStreams* s);

// Streaming multiprocessors of the current device (cached per device; 148 on
// B200).  Grids are sized in multiples of it.
KOG2_HIDDEN int kog2_sm_count(void);
