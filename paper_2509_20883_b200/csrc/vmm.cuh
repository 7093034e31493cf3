// vmm.cuh — growable device arrays on CUDA virtual memory management.
//
// The reference's BlockStore appends blocks and never moves a row
// (embedding.py:87-92).  The B200 table keeps that property with one
// reserved virtual address range per array: growth maps more physical
// memory (cuMemCreate + cuMemMap) behind the existing rows, so the arena
// pointer, every row and every in-flight kernel's view stay valid — no copy,
// no 2.5x transient footprint, no stream drain.  Only when an array outgrows
// its reservation is a larger range reserved and the SAME physical chunks are
// mapped into it (a remap, still no copy; the pointer changes then).
#pragma once
#include <vector>

#include "common.cuh"

namespace skb {

struct VmmArray {
  uint64_t base = 0;      // CUdeviceptr of the reservation
  size_t reserved = 0;    // bytes of VA reserved
  size_t mapped = 0;      // bytes mapped (a multiple of the granularity)
  struct Chunk {
    unsigned long long handle;  // CUmemGenericAllocationHandle
    size_t offset, bytes;
  };
  std::vector<Chunk> chunks;
  // a chunk created and mapped ahead of need at [mapped, mapped + prep_bytes)
  // (by a background thread: growth then only zero-fills it on the stream)
  unsigned long long prep_handle = 0;
  size_t prep_bytes = 0;
};

// whether the driver exposes the VMM entry points (resolved once)
bool vmm_available();
// allocation granularity of device memory on the current device
size_t vmm_granularity();
// Grow `a` to hold at least `bytes` (zero-filled on `s` past the old end).
// Returns true when the base pointer changed (a re-reservation).  `headroom`:
// reserve this many times the needed bytes when (re)reserving VA.
bool vmm_grow(VmmArray& a, size_t bytes, size_t reserve_hint, cudaStream_t s);
void vmm_free(VmmArray& a);
// Create and map (not zero) up to `bytes` more behind the mapped end, within
// the reservation, for the next vmm_grow to adopt — the slow driver calls
// (cuMemCreate / cuMemMap / cuMemSetAccess, ~0.3 ms per array) moved off the
// step's host thread.  Safe from another thread while no vmm_grow / vmm_free
// of the same array runs (the table joins its prepare thread before those).
void vmm_prepare(VmmArray& a, size_t bytes, int device);

}  // namespace skb
