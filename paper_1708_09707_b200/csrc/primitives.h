// primitives.h -- device data-parallel primitives (replace the reference's
// CPU substrate, proj/include/hmat/parallel.hpp): exclusive scan and a stable
// LSD radix sort of (u64 key, u32 payload) pairs.
#pragma once
#include <cstdint>

#include "common.cuh"

namespace hmb {

// out[i] = sum in[0..i); returns the total (synchronises the stream once).
// in and out may alias.
long long exclusive_scan_i64(const long long* in, long long* out, long long n, cudaStream_t s);
// Same, stream-ordered: no host synchronisation; the total (if total_dev) stays on the device.
void exclusive_scan_i64_async(const long long* in, long long* out, long long n, long long* total_dev,
                              cudaStream_t s);

// Workspace-owning stable radix sort: ascending u64 keys, ties keep input
// order (std::stable_sort semantics, parallel.hpp:45-62).  Digits on which all
// keys agree are skipped (one host synchronisation per sort to learn them; the
// passes themselves are stream-ordered).  Results are written back into keys/vals.
void radix_sort_pairs(unsigned long long* keys, unsigned* vals, long long n, cudaStream_t s);

// out[i] = i
void iota_u32(unsigned* out, long long n, cudaStream_t s);

}  // namespace hmb
