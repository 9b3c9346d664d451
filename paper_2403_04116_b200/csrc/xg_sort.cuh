// Device-wide primitives used by binning and density control (internal).
#pragma once
#include "xg_internal.cuh"

namespace xg {

// Exclusive prefix sum of uint32 (optionally gathered: x[i] = in[gather[i]]).
// The item count is read on the device from *n_dev when n_dev != nullptr
// (else n_host); grids are sized for `cap`.  If total != nullptr the sum is
// written there (device).  Single pass, decoupled look-back.
size_t scan_workspace_bytes(int64_t cap);
// the next scan_u32 on this host thread finds its workspace already zeroed
// (the caller cleared scan_workspace_bytes(cap) bytes at ws): no memset
void scan_u32_precleared_next();
xg_status scan_u32(const uint32_t* in, const uint32_t* gather, uint32_t* out, int64_t cap,
                   const uint32_t* n_dev, int64_t n_host, uint32_t* total, void* ws, size_t ws_bytes,
                   cudaStream_t s);

// Stable LSD radix sort of (key, value) uint32 pairs over key bits
// [begin_bit, end_bit).  Input in keys[0]/vals[0]; the result ends in
// keys[*result]/vals[*result].  Count read on device from *n_dev.
size_t radix_workspace_bytes(int64_t cap);
xg_status radix_sort_pairs(uint32_t* keys[2], uint32_t* vals[2], int64_t cap, const uint32_t* n_dev,
                           int begin_bit, int end_bit, void* ws, size_t ws_bytes, cudaStream_t s,
                           int* result);
xg_status radix_sort_pairs64(unsigned long long* keys[2], uint32_t* vals[2], int64_t cap,
                             const uint32_t* n_dev, int begin_bit, int end_bit, void* ws, size_t ws_bytes,
                             cudaStream_t s, int* result);

// Onesweep variant for 64-bit keys (all 8 byte passes; constant-digit
// passes are skipped on the device).  Result always ends in vals[0]
// (keys end wherever the last executed pass wrote them).
size_t onesweep_workspace_bytes(int64_t cap);
// Stable LSD sort of (64-bit key, u32 value) pairs; keys_in / vals_in are
// never written (passes ping-pong between the a / b scratch buffers; vals_b
// may alias vals_in), the sorted values land in vals_out.
xg_status onesweep_sort_pairs64(const unsigned long long* keys_in, const uint32_t* vals_in,
                                unsigned long long* keys_a, unsigned long long* keys_b, uint32_t* vals_a,
                                uint32_t* vals_b, uint32_t* vals_out, int64_t cap, const uint32_t* n_dev,
                                void* ws, size_t ws_bytes, cudaStream_t s, int n_passes = 8,
                                const int** result_sel = nullptr);
// (n_passes < 8: keys must be zero above byte n_passes; result_sel != null:
// no final copy - the result is vals {a, b, in}[**result_sel], device-side)

// Depth order of the active splats (ascending (key, index); inactive ones,
// n_tiles == 0, first, in arbitrary order) by a stable sort on 15-bit key
// buckets and ranking inside mixed buckets (xg_sort.cu).  key_a / key_b /
// val_a / val_b: N-sized scratch; order: N-sized output; keys never written;
// *n_dev receives n (the onesweep's device count).
size_t bucket_sort_workspace_bytes(int64_t n);
xg_status bucket_sort_depth(const unsigned long long* keys, const uint32_t* n_tiles, int64_t n,
                            unsigned long long* key_a, unsigned long long* key_b, uint32_t* val_a, uint32_t* val_b,
                            uint32_t* order, uint32_t* n_dev, void* ws, size_t ws_bytes, cudaStream_t s);

}  // namespace xg
