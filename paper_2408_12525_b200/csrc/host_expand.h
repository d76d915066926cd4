// host_expand.h -- host side of the packed observation transfer (lg_step_host).
//
// The step kernel writes the batch's 0/1 observation planes as one bit stream
// (element t of the [B,C,OH,OW] observation = bit t); the stream crosses PCIe
// in chunks and the host cores expand it, chunk by chunk as each copy lands,
// into the caller's float32 (or uint8) array with non-temporal stores.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace lg_host {

// Expand stream bits [0, n_elems) of `bits` into dst (float32 when fmt == 0,
// uint8 when fmt == 1). The stream is processed in chunks of chunk_bytes
// bytes of `bits` (a multiple of 64); chunk c is read only after ready(ctx, c)
// returned true (polled by the workers; ready == nullptr: every chunk is
// there). Runs on the library's host thread pool plus the calling thread
// (small outputs: the calling thread only); returns after dst is complete.
void expand_bits(const uint8_t *bits, void *dst, int fmt, size_t n_elems, size_t chunk_bytes,
                 bool (*ready)(void *ctx, size_t chunk), void *ctx);

// Threads used by expand_bits (LG_HOST_THREADS overrides the core count).
int expand_threads();

}  // namespace lg_host
