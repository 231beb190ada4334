// fb_stream.cuh — multi-stream bulk-copy tile ring.
//
// Every factor-matrix pass (LMM, RMM, rowSums/colSums, the driver steps) streams a
// contiguous range of rows through shared memory. A row range of a row-major f64
// matrix is one contiguous byte range, so a tile of rows is one 1-D bulk copy
// (cp.async.bulk -> UBLKCP) — no tensor map needed. Up to kMaxStreams row-aligned
// arrays (the factor rows, the int32 FK column(s), per-row weights) share one
// mbarrier per stage; thread 0 is the producer, all threads consume.
//
// Tiles whose byte ranges are not 16-byte aligned (only the final tile, or every
// tile when a caller passes a misaligned base pointer) are filled by the CTA with
// plain loads instead; the producer then arrives without a transaction count so the
// phase bookkeeping stays uniform.
#pragma once
#include "fb_common.cuh"

namespace fb {

constexpr int kMaxStreams = 8;

struct StreamSet {
  const char* base[kMaxStreams];
  uint32_t row_bytes[kMaxStreams];
  uint32_t smem_off[kMaxStreams];  // byte offset of this stream inside a stage
  int count;
  uint32_t stage_bytes;  // bytes per stage (all streams, 128-byte padded)
  bool base_aligned;     // all bases 16-byte aligned
};

// Host helper: lay out `count` streams for `tile_rows` rows per stage.
inline void stream_layout(StreamSet& s, int tile_rows) {
  uint32_t off = 0;
  s.base_aligned = true;
  for (int i = 0; i < s.count; ++i) {
    s.smem_off[i] = off;
    off += (s.row_bytes[i] * static_cast<uint32_t>(tile_rows) + 127u) & ~127u;
    if (reinterpret_cast<uintptr_t>(s.base[i]) & 15u) s.base_aligned = false;
  }
  s.stage_bytes = off;
}

struct TileRing {
  char* buf;      // stages * stage_bytes
  uint64_t* bar;  // stages mbarriers
  int stages;
  int tile_rows;
  int64_t n_rows;
  int64_t tile_begin, tile_end;  // this CTA's contiguous tile range
  uint64_t policy;

  FB_DEV char* stage_ptr(int stage, const StreamSet& s, int stream) const {
    return buf + static_cast<size_t>(stage) * s.stage_bytes + s.smem_off[stream];
  }

  FB_DEV int rows_of(int64_t tile) const {
    int64_t r0 = tile * tile_rows;
    int64_t r = n_rows - r0;
    return static_cast<int>(r < tile_rows ? r : tile_rows);
  }

  FB_DEV bool bulk_ok(const StreamSet& s, int rows) const {
    if (!s.base_aligned) return false;
    for (int i = 0; i < s.count; ++i)
      if ((s.row_bytes[i] * static_cast<uint32_t>(rows)) & 15u) return false;
    // interior tiles start at multiples of tile_rows (a multiple of 4 rows), so their
    // starting offsets are 16-byte aligned for any row size that is a multiple of 4 bytes.
    return true;
  }

  // Producer side (one thread).
  FB_DEV void issue(const StreamSet& s, int64_t tile, int stage) const {
    int rows = rows_of(tile);
    if (bulk_ok(s, rows)) {
      uint32_t total = 0;
      for (int i = 0; i < s.count; ++i) total += s.row_bytes[i] * static_cast<uint32_t>(rows);
      fence_proxy_async();
      mbar_arrive_expect_tx(&bar[stage], total);
      for (int i = 0; i < s.count; ++i) {
        if (s.row_bytes[i] == 0) continue;
        const char* src = s.base[i] + static_cast<size_t>(tile) * tile_rows * s.row_bytes[i];
        bulk_g2s_stream(stage_ptr(stage, s, i), src, s.row_bytes[i] * static_cast<uint32_t>(rows),
                        &bar[stage], policy);
      }
    } else {
      mbar_arrive(&bar[stage]);
    }
  }

  // Consumer side: fill a non-bulk tile cooperatively (4-byte granularity).
  FB_DEV void manual_fill(const StreamSet& s, int64_t tile, int stage) const {
    int rows = rows_of(tile);
    for (int i = 0; i < s.count; ++i) {
      const uint32_t* src = reinterpret_cast<const uint32_t*>(
          s.base[i] + static_cast<size_t>(tile) * tile_rows * s.row_bytes[i]);
      uint32_t* dst = reinterpret_cast<uint32_t*>(stage_ptr(stage, s, i));
      uint32_t words = s.row_bytes[i] * static_cast<uint32_t>(rows) / 4u;
      for (uint32_t w = threadIdx.x; w < words; w += blockDim.x) dst[w] = src[w];
    }
  }

  // Set up barriers and prime the pipeline. Must be called by all threads.
  FB_DEV void start(const StreamSet& s) {
    if (threadIdx.x == 0) {
      for (int i = 0; i < stages; ++i) mbar_init(&bar[i], 1);
      fence_mbar_init();
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t ntiles = tile_end - tile_begin;
      for (int k = 0; k < stages && k < ntiles; ++k) issue(s, tile_begin + k, k);
    }
  }

  // Wait for local tile index k (0-based within this CTA's range); returns stage index.
  FB_DEV int acquire(const StreamSet& s, int64_t k) const {
    int stage = static_cast<int>(k % stages);
    uint32_t parity = static_cast<uint32_t>((k / stages) & 1);
    mbar_wait(&bar[stage], parity);
    int64_t tile = tile_begin + k;
    if (!bulk_ok(s, rows_of(tile))) {
      manual_fill(s, tile, stage);
      __syncthreads();
    }
    return stage;
  }

  // Release local tile k (all threads done reading it) and refill its stage.
  FB_DEV void release(const StreamSet& s, int64_t k) const {
    __syncthreads();
    if (threadIdx.x == 0) {
      int64_t nk = k + stages;
      if (nk < tile_end - tile_begin) issue(s, tile_begin + nk, static_cast<int>(k % stages));
    }
  }
};

// Contiguous split of [0, ntiles) over gridDim.x CTAs.
FB_DEV void cta_tile_range(int64_t ntiles, int64_t& b, int64_t& e) {
  int64_t g = gridDim.x, c = blockIdx.x;
  b = ntiles * c / g;
  e = ntiles * (c + 1) / g;
}

}  // namespace fb
