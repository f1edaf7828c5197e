// fvb_hostcopy.h -- host-memory copies and fills of the host-buffer path.
//
// The pageable path's bounce copies, the pass-through copies, the duplicate
// copies and the constant fills all write large ranges the CPU does not read
// back soon (the DMA engine or the caller does).  Plain memcpy of the copy
// pool's 8 MiB pieces pays a read-for-ownership of every destination line;
// non-temporal (streaming) stores do not: 60 -> 80 GB/s with 16 threads on
// the GPU box's host (profiles/r01_host_copy_probe.jsonl).
#pragma once

#include <cstddef>
#include <cstdint>

namespace fvb {

// dst <- src, n bytes (streaming stores when the CPU has AVX2 and n is large)
void host_copy(char* dst, const char* src, size_t n);

// n bytes of dst (element-aligned) <- the element `bits` of `width` 4 or 8
// bytes, repeated
void host_fill(char* dst, uint64_t bits, size_t width, size_t n);

}  // namespace fvb
