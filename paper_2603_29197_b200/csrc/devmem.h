// Device memory for the handles: stream-ordered allocations from the device's default memory pool, with the pool
// told to KEEP freed memory (release threshold = max).  A solve of the C4 problem owns ~25 GB in ~60 allocations;
// with cudaMalloc / cudaFree every handle paid the driver's map / unmap cost (measured 0.05 s to allocate and
// 0.04-0.9 s to free, box dependent), so a loop of setup -> solve -> destroy was partly a benchmark of the driver.
// From the second handle on, allocations and frees are pool bookkeeping.  Falls back to cudaMalloc / cudaFree where
// the device has no memory-pool support.  QS_NO_MEMPOOL=1 forces the fallback.
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>

cudaError_t qs_dev_malloc(void** p, size_t bytes);  // usable on any stream on return
void qs_dev_free(void* p);                          // caller guarantees that no work still uses p
