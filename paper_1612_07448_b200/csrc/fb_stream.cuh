// fb_stream.cuh — warp-specialised multi-stream bulk-copy tile ring.
//
// Every factor-matrix pass (LMM, RMM, rowSums/colSums, crossprod, the driver steps)
// streams a contiguous range of rows through shared memory. A row range of a row-major
// f64 matrix is one contiguous byte range, so a tile of rows is one 1-D bulk copy
// (cp.async.bulk -> SASS UBLKCP) — no tensor map needed. Up to kMaxStreams row-aligned
// arrays (the factor rows, the int32 FK column(s), per-row weights) share one "full"
// mbarrier per stage.
//
// Roles (kRingThreads = 1 producer + kGatherWarps gatherers + kConsumerWarps consumers):
//   warp 0  producer: issues the stream copies of each stage once its "empty" barrier
//           says the consumers are done with it;
//   warps 1-4 gatherers: for keyed gather streams (z[fk] rows of an LMM, ...) it waits for
//           the stage's keys to land, then copies the keyed rows from the lookup table
//           into the stage with 16-byte cp.async (one warp instruction moves 32 chunks;
//           a per-row bulk copy costs ~60 issue cycles, measured), each lane completing
//           on a second per-stage barrier ("gfull"). Gathers therefore run as many stages
//           ahead as the ring is deep, and the consumers never wait on an L2 round trip;
//   warps 2+ consumers: wait on "full" (+ "gfull"), compute, arrive on "empty".
// Consumers that need to sync among themselves use consumer_sync() (named barrier 1).
//
// A stream may ask for a padded shared-memory pitch (bytes per row > row bytes) so that
// tensor-core fragment loads that walk rows hit distinct banks: the producer then copies
// it with 16-byte cp.async and all its lanes arrive on "full" (expected count 1 + 32). Stream 0 may instead be gathered by a global row index array
// (gidx: rows in FK-sorted order for the crossprod); the gatherer moves those rows with
// 16-byte cp.async too, once the stage is free (its "full" phase for the other streams).
//
// Tiles that cannot use bulk copies (a misaligned base, or a final tile whose byte
// count is not a multiple of 16) are filled by the consumers with plain loads; the
// producer arrives on "full" without a transaction count so phases stay uniform, and the
// gatherer then reads the keys from global memory.
//
// Measured on B200 (tools/stream_probe.cu): with one CTA per SM the ring needs >= ~130 KB
// in flight (e.g. 3 × 44 KB) to reach 6.7-7.4 TB/s; per-tile bookkeeping must stay off
// the consumers' path (incremental stage/phase, no 64-bit division, no fence.proxy.async
// per issue — that fence waits for the thread's in-flight copies).
#pragma once
#include "fb_common.cuh"

namespace fb {

constexpr int kMaxStreams = 8;
constexpr int kMaxGather = 4;
constexpr int kConsumerWarps = 8;
constexpr int kConsumerThreads = kConsumerWarps * 32;
#ifndef FB_GATHER_WARPS
#define FB_GATHER_WARPS 4
#endif
constexpr int kGatherWarps = FB_GATHER_WARPS;
constexpr int kServiceWarps = 1 + kGatherWarps;
constexpr int kRingThreads = kConsumerThreads + 32 * kServiceWarps;
constexpr int kRingHeader = 512;  // 3 × 16 mbarriers (full, empty, gfull) + padding
constexpr int kMaxStages = 16;

struct StreamSet {
  const char* base[kMaxStreams];
  uint32_t row_bytes[kMaxStreams];
  uint32_t pitch[kMaxStreams];     // shared-memory bytes per row (>= row_bytes)
  uint32_t smem_off[kMaxStreams];  // byte offset of this stream inside a stage
  int count;
  uint32_t stage_bytes;  // bytes per stage (all streams, 128-byte padded)
  uint32_t tile_tx;      // transaction bytes of a full tile
  bool bulk_full;        // full tiles can use bulk copies
  bool bulk_last;        // the final (possibly partial) tile can use bulk copies
  bool row_bulk;         // padded-pitch streams: one bulk copy per row (instead of 16-byte
                         // cp.async chunks) — for tiles of few, long rows
  bool gidx_bulk;        // gidx rows moved with one bulk copy per row (long rows, no keyed
                         // gathers in the same ring): the gatherer lanes arrive on "gfull"
                         // themselves (lane 0 with the warp's byte count) and the copies
                         // complete it
  const int32_t* gidx;   // optional: stream 0 row r of the ring is source row gidx[r]
                         // (a gathered stream, e.g. rows in FK-sorted order); <= 128 rows/tile
  // keyed gathers: row r of gather g = gbase[g] + key * grow_bytes[g], key = gkeys[g][row]
  // (int32, row-aligned with the ring's rows); grow_bytes a multiple of 16, gbase 16-byte
  // aligned; tiles of at most 256 rows
  int ngather;
  const int32_t* gkeys[kMaxGather];
  const char* gbase[kMaxGather];
  uint32_t grow_bytes[kMaxGather];
  uint32_t gsmem_off[kMaxGather];
};

// Host helper: lay out `count` streams (+ `ngather` gathers) for `tile_rows` rows per
// stage over n_rows rows. A zero pitch means dense (pitch = row_bytes).
inline void stream_layout(StreamSet& s, int tile_rows, int64_t n_rows) {
  uint32_t off = 0;
  bool aligned = true;
  s.tile_tx = 0;
  const int last_rows =
      n_rows > 0 ? static_cast<int>(n_rows - ((n_rows - 1) / tile_rows) * tile_rows) : tile_rows;
  bool full_ok = true, last_ok = true;
  for (int i = 0; i < s.count; ++i) {
    if (s.pitch[i] < s.row_bytes[i]) s.pitch[i] = s.row_bytes[i];
    s.smem_off[i] = off;
    off += (s.pitch[i] * static_cast<uint32_t>(tile_rows) + 127u) & ~127u;
    if (reinterpret_cast<uintptr_t>(s.base[i]) & 15u) aligned = false;
    s.tile_tx += s.row_bytes[i] * static_cast<uint32_t>(tile_rows);
    if (s.pitch[i] != s.row_bytes[i] || (i == 0 && s.gidx)) {
      if ((s.row_bytes[i] & 15u) || (s.pitch[i] & 15u)) full_ok = last_ok = false;
    } else {
      if ((s.row_bytes[i] * static_cast<uint32_t>(tile_rows)) & 15u) full_ok = false;
      if ((s.row_bytes[i] * static_cast<uint32_t>(last_rows)) & 15u) last_ok = false;
    }
  }
  for (int g = 0; g < s.ngather; ++g) {
    s.gsmem_off[g] = off;
    off += (s.grow_bytes[g] * static_cast<uint32_t>(tile_rows) + 127u) & ~127u;
  }
  s.stage_bytes = off;
  s.bulk_full = aligned && full_ok;
  s.bulk_last = aligned && last_ok && full_ok;
}

// Pitch (in doubles) that makes m8n8k4 fragment loads (8 rows x 4 columns) conflict
// free: any width that is 2 (mod 4) or 4/12 (mod 16) works; widths that are a
// multiple of 8 get 4 doubles of padding. Odd widths cannot be copied row by row.
inline int conflict_free_pitch(int d) {
  if (d % 8 == 0) return d + 4;
  return d;
}

FB_DEV void consumer_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(kConsumerThreads) : "memory");
}

FB_DEV bool is_producer_warp() { return threadIdx.x < 32; }
FB_DEV bool is_gather_warp() { return threadIdx.x >= 32 && threadIdx.x < 32 * kServiceWarps; }
FB_DEV int consumer_tid() { return static_cast<int>(threadIdx.x) - 32 * kServiceWarps; }
FB_DEV int consumer_warp() { return (static_cast<int>(threadIdx.x) >> 5) - kServiceWarps; }

// RR = false: each CTA takes one contiguous range of tiles. RR = true: tiles dealt round-robin
// (CTA c takes tiles c, c + grid, ...), so all CTAs sweep the matrix front to back together —
// for passes whose rows are laid out in FK bands, every CTA then gathers from the same
// L2-resident slice of the lookup table at any moment (the banded LMM S pass, fb_lmm.cu).
template <bool RR>
struct TileRingT {
  char* buf;        // stages * stage_bytes
  uint64_t* full;   // stages mbarriers (producer -> consumers, gatherer)
  uint64_t* empty;  // stages mbarriers (consumers -> producer)
  uint64_t* gfull;  // stages mbarriers (gatherer -> consumers)
  int stages;
  int tile_rows;
  int64_t n_rows;
  int64_t ntiles;                // tiles over the whole matrix
  int64_t tile_begin, tile_end;  // this CTA's contiguous tile range (RR: first tile, ntiles)
  int64_t tile_step;             // RR: grid size
  uint64_t policy;
  bool gathers;
  // consumer iteration state: the next stage to wait on, and the oldest stage still held
  int stage;
  uint32_t phase;
  int rstage;

  // Carve `smem` (128-byte aligned): barriers in the first kRingHeader bytes, then buffers.
  FB_DEV void init(char* smem, int stages_, int tile_rows_, int64_t n_rows_) {
    full = reinterpret_cast<uint64_t*>(smem);
    empty = full + kMaxStages;
    gfull = empty + kMaxStages;
    buf = smem + kRingHeader;
    stages = stages_;
    tile_rows = tile_rows_;
    n_rows = n_rows_;
    ntiles = (n_rows_ + tile_rows_ - 1) / tile_rows_;
    const int64_t g = gridDim.x, c = blockIdx.x;
    if constexpr (RR) {
      tile_begin = c;
      tile_end = ntiles;
      tile_step = g;
    } else {
      tile_begin = ntiles * c / g;
      tile_end = ntiles * (c + 1) / g;
      tile_step = 1;
    }
    policy = policy_evict_first();
    gathers = false;
  }

  FB_DEV int64_t count() const {
    if constexpr (RR) return tile_end > tile_begin ? (tile_end - tile_begin + tile_step - 1) / tile_step : 0;
    return tile_end - tile_begin;
  }

  // global tile index of this CTA's k-th tile
  FB_DEV int64_t tile_of(int64_t k) const {
    if constexpr (RR) return tile_begin + k * tile_step;
    return tile_begin + k;
  }

  FB_DEV char* stage_ptr(int st, const StreamSet& s, int stream) const {
    return buf + static_cast<uint32_t>(st) * s.stage_bytes + s.smem_off[stream];
  }

  FB_DEV char* gather_ptr(int st, const StreamSet& s, int g) const {
    return buf + static_cast<uint32_t>(st) * s.stage_bytes + s.gsmem_off[g];
  }

  FB_DEV int rows_of(int64_t tile) const {
    return tile == ntiles - 1 ? static_cast<int>(n_rows - tile * tile_rows) : tile_rows;
  }

  FB_DEV bool bulk_ok(const StreamSet& s, int64_t tile) const {
    return tile == ntiles - 1 ? s.bulk_last : s.bulk_full;
  }

  // Barrier setup; call from all threads before the role split (contains __syncthreads).
  // extra_empty: additional warps (beyond the consumers) that release every stage.
  FB_DEV void start(const StreamSet& s, int extra_empty = 0) {
    stage = 0;
    phase = 0;
    rstage = 0;
    gathers = s.ngather > 0 || s.gidx != nullptr;
    if (threadIdx.x == 0) {
      for (int i = 0; i < stages; ++i) {
        mbar_init(&full[i], has_pitched(s) ? 33 : 1);
        mbar_init(&empty[i], kConsumerWarps + extra_empty);
        mbar_init(&gfull[i], 32 * kGatherWarps);
      }
      fence_mbar_init();
    }
    __syncthreads();
  }

  // Streams copied with cp.async by the producer (padded pitch): its 32 lanes then arrive
  // on "full" as well.
  FB_DEV static bool has_pitched(const StreamSet& s) {
    if (s.row_bulk) return false;
    bool p = false;
#pragma unroll
    for (int i = 0; i < kMaxStreams; ++i)
      if (i < s.count && s.row_bytes[i] > 0 && s.pitch[i] != s.row_bytes[i] && !(i == 0 && s.gidx)) p = true;
    return p;
  }

  // Service warps run their loop and return true; consumers get false. GIDX_BULK: a ring whose
  // gidx rows move with one bulk copy each (StreamSet::gidx_bulk) — a separate instantiation
  // used only by the kernels that need it (a runtime branch, or a second gather loop in every
  // kernel, slowed the LMM gathers by 2-15%).
  template <bool GIDX_BULK = false, bool GATHER_CG = false>
  FB_DEV bool service(const StreamSet& s) const {
    if (is_producer_warp()) {
      produce(s);
      return true;
    }
    if (is_gather_warp()) {
      if (s.ngather > 0 || s.gidx) gather<GIDX_BULK, GATHER_CG>(s);
      return true;
    }
    return false;
  }

  // Producer warp body: issue every tile of this CTA's range, recycling stages. A gidx
  // stream 0 is left to the gatherer.
  FB_DEV void produce(const StreamSet& s) const {
    const int lane = threadIdx.x & 31;
    const bool pitched = has_pitched(s);
    int st = 0;
    uint32_t ph = 0;
    const int64_t n = count();
    for (int64_t k = 0; k < n; ++k) {
      const int64_t tile = tile_of(k);
      if (k >= stages) mbar_wait(&empty[st], ph ^ 1u);
      const int rows = rows_of(tile);
      if (bulk_ok(s, tile)) {
        if (lane == 0) {
          uint32_t tx = 0;
#pragma unroll
          for (int i = 0; i < kMaxStreams; ++i)
            if (i < s.count && !(i == 0 && s.gidx) && (s.pitch[i] == s.row_bytes[i] || s.row_bulk))
              tx += s.row_bytes[i] * static_cast<uint32_t>(rows);
          mbar_arrive_expect_tx(&full[st], tx);
        }
        __syncwarp();
#pragma unroll
        for (int i = 0; i < kMaxStreams; ++i) {
          if (i >= s.count || s.row_bytes[i] == 0 || (i == 0 && s.gidx)) continue;
          const char* src = s.base[i] + static_cast<size_t>(tile) * tile_rows * s.row_bytes[i];
          char* dst = stage_ptr(st, s, i);
          if (s.pitch[i] == s.row_bytes[i]) {
            if (lane == 0)
              bulk_g2s_stream(dst, src, s.row_bytes[i] * static_cast<uint32_t>(rows), &full[st], policy);
          } else if (s.row_bulk) {
            for (int r = lane; r < rows; r += 32)
              bulk_g2s_stream(dst + r * s.pitch[i], src + static_cast<size_t>(r) * s.row_bytes[i], s.row_bytes[i],
                              &full[st], policy);
          } else {
            // padded pitch: (row, 16-byte chunk) items over the lanes with cp.async — one warp
            // instruction moves 512 bytes (a per-row bulk copy costs ~60 issue cycles)
            const uint32_t nch = s.row_bytes[i] >> 4;
            const uint32_t items = nch * static_cast<uint32_t>(rows);
            for (uint32_t it = lane; it < items; it += 32) {
              const uint32_t r = it / nch, c = it - r * nch;
              cp_async16(dst + r * s.pitch[i] + 16u * c, src + static_cast<size_t>(r) * s.row_bytes[i] + 16u * c, 0);
            }
          }
        }
      } else if (lane == 0) {
        mbar_arrive(&full[st]);
      }
      if (pitched) {
        __syncwarp();
        cp_async_arrive_noinc(&full[st]);  // all 32 lanes, after their copies
      }
      if (++st == stages) {
        st = 0;
        ph ^= 1u;
      }
    }
  }

  // Gatherer warps body. A stage's gathers start as soon as the stage is free (its
  // "empty" phase), in parallel with the producer's stream copies: the keys come from
  // global memory, loaded one tile ahead, so a gathered tile costs max(stream, key +
  // gather) latency rather than their sum. Gatherer warp gw owns ring rows
  // r ≡ gw (mod kGatherWarps) (<= 64 of them: tiles of at most 256 rows).
  template <bool GIDX_BULK, bool GATHER_CG>
  FB_DEV void gather(const StreamSet& s) const {
    const int lane = threadIdx.x & 31;
    const int gw = (static_cast<int>(threadIdx.x) >> 5) - 1;
    int st = 0;
    uint32_t ph = 0;
    const int64_t n = count();
    // keys / gidx of this warp's rows gw + kGatherWarps·(lane + 32 j), j < 2
    int32_t kc[kMaxGather + 1][2], kn[kMaxGather + 1][2];
    auto load_keys = [&](int64_t tile) {
      const int rows = rows_of(tile);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int r = gw + kGatherWarps * (lane + 32 * j);
        const bool live = r < rows;
#pragma unroll
        for (int g = 0; g < kMaxGather; ++g)
          kn[g][j] = (g < s.ngather && live) ? __ldg(s.gkeys[g] + tile * tile_rows + r) : 0;
        kn[kMaxGather][j] = (s.gidx && live) ? __ldg(s.gidx + tile * tile_rows + r) : 0;
      }
    };
    // key of this warp's row index ri (warp-uniform call; ri may differ per lane)
    auto key_of = [&](int g, int ri) {
      const int v0 = __shfl_sync(0xffffffffu, kc[g][0], ri & 31);
      const int v1 = __shfl_sync(0xffffffffu, kc[g][1], ri & 31);
      return ri < 32 ? v0 : v1;
    };
    if (n > 0) load_keys(tile_of(0));
    for (int64_t k = 0; k < n; ++k) {
      const int64_t tile = tile_of(k);
      const int rows = rows_of(tile);
      const int rows_w = rows > gw ? (rows - gw + kGatherWarps - 1) / kGatherWarps : 0;  // rows of this warp
#pragma unroll
      for (int g = 0; g <= kMaxGather; ++g) {
        kc[g][0] = kn[g][0];
        kc[g][1] = kn[g][1];
      }
      if (k + 1 < n) load_keys(tile_of(k + 1));  // latency overlaps this stage's wait and copies
      if (k >= stages) mbar_wait(&empty[st], ph ^ 1u);  // the stage is free again
      if (GIDX_BULK && s.gidx && s.gidx_bulk && bulk_ok(s, tile)) {
        // one bulk copy per row, lane i moving the warp's row i (its own gidx register): the
        // copy engine takes a 480-byte row as one request where 16-byte cp.async took 30
        const uint32_t rb = s.row_bytes[0];
        char* dst = stage_ptr(st, s, 0);
        if (lane == 0)
          mbar_arrive_expect_tx(&gfull[st], static_cast<uint32_t>(rows_w) * rb);
        else
          mbar_arrive(&gfull[st]);
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 2; ++j) {
          const int i = lane + 32 * j;
          if (i < rows_w)
            bulk_g2s(dst + static_cast<uint32_t>(gw + kGatherWarps * i) * s.pitch[0],
                     s.base[0] + static_cast<size_t>(kc[kMaxGather][j]) * rb, rb, &gfull[st]);
        }
        if (++st == stages) {
          st = 0;
          ph ^= 1u;
        }
        continue;
      }
      if (s.gidx && bulk_ok(s, tile)) {
        // stream 0 rows in gidx order: one row per instruction, lanes over 16-byte chunks
        char* dst = stage_ptr(st, s, 0);
        const uint32_t rb = s.row_bytes[0], nch = rb >> 4;
        if (nch <= 32) {
          // the row index is warp-uniform: one shuffle per row, no per-lane chunk loop
          char* d0 = dst + gw * s.pitch[0] + 16u * lane;
          const char* s0 = s.base[0] + 16u * lane;
          const uint32_t dstep = kGatherWarps * s.pitch[0];
          const bool on = lane < nch;
#pragma unroll 4
          for (int i = 0; i < rows_w; ++i) {
            const int32_t srow =
                __shfl_sync(0xffffffffu, i < 32 ? kc[kMaxGather][0] : kc[kMaxGather][1], i & 31);
            if (on) cp_async16(d0 + i * dstep, s0 + static_cast<size_t>(srow) * rb, 0);
          }
        } else {
          for (int i = 0; i < rows_w; ++i) {
            const uint32_t r = gw + kGatherWarps * i;
            const int32_t srow = key_of(kMaxGather, i);
            for (uint32_t c = lane; c < nch; c += 32)
              cp_async16(dst + r * s.pitch[0] + 16u * c, s.base[0] + static_cast<size_t>(srow) * rb + 16u * c, 0);
          }
        }
      }
#pragma unroll
      for (int g = 0; g < kMaxGather; ++g) {  // unrolled: kc[g] stays in registers
        if (g >= s.ngather) break;
        char* dst = gather_ptr(st, s, g);
        const uint32_t rb = s.grow_bytes[g];
        const uint32_t nch = rb >> 4;
        if (nch <= 32) {
          // lanes per row: nch rounded up to a power of two; 32/that rows per instruction
          int lg = 0;
          while ((1u << lg) < nch) ++lg;
          const int rpi = 32 >> lg;
          const int slot = lane >> lg;
          const uint32_t c = lane & ((1u << lg) - 1);
          const int iters = (rows_w + rpi - 1) / rpi;
#pragma unroll 4
          for (int j = 0; j < iters; ++j) {
            const int ri = j * rpi + slot;
            const int32_t key = key_of(g, ri);
            if (ri < rows_w && c < nch) {
              const uint32_t r = gw + kGatherWarps * ri;
              cp_async16_gather<GATHER_CG>(dst + r * rb + 16u * c, s.gbase[g] + static_cast<size_t>(key) * rb + 16u * c);
            }
          }
        } else {
          for (int ri = 0; ri < rows_w; ++ri) {
            const int32_t key = key_of(g, ri);
            const uint32_t r = gw + kGatherWarps * ri;
            for (uint32_t c = lane; c < nch; c += 32)
              cp_async16_gather<GATHER_CG>(dst + r * rb + 16u * c, s.gbase[g] + static_cast<size_t>(key) * rb + 16u * c);
          }
        }
      }
      __syncwarp();  // the arrive must be issued by the converged warp
      cp_async_arrive_noinc(&gfull[st]);
      if (++st == stages) {
        st = 0;
        ph ^= 1u;
      }
    }
    // do not retire the warp with copies (and their barrier arrivals) still in flight
    asm volatile("cp.async.wait_all;\n" ::: "memory");
  }

  // Consumers: fill a non-bulk tile cooperatively (4-byte granularity).
  FB_DEV void manual_fill(const StreamSet& s, int64_t tile, int st) const {
    const int rows = rows_of(tile);
    for (int i = 0; i < s.count; ++i) {
      const char* src = s.base[i] + static_cast<size_t>(tile) * tile_rows * s.row_bytes[i];
      char* dst = stage_ptr(st, s, i);
      const uint32_t wpr = s.row_bytes[i] / 4u;  // words per row
      const uint32_t words = wpr * static_cast<uint32_t>(rows);
      const bool gather = i == 0 && s.gidx;
      for (uint32_t w = consumer_tid(); w < words; w += kConsumerThreads) {
        const uint32_t r = w / wpr, c = w % wpr;
        const char* srow = gather ? s.base[0] + static_cast<size_t>(s.gidx[tile * tile_rows + r]) * s.row_bytes[0]
                                  : src + static_cast<size_t>(r) * s.row_bytes[i];
        reinterpret_cast<uint32_t*>(dst + static_cast<size_t>(r) * s.pitch[i])[c] =
            reinterpret_cast<const uint32_t*>(srow)[c];
      }
    }
  }

  // Consumers: wait for the next tile (local index k, in order); returns its stage.
  FB_DEV int acquire(const StreamSet& s, int64_t k) {
    const int st = stage;
    mbar_wait(&full[st], phase);
    const int64_t tile = tile_of(k);
    if (!bulk_ok(s, tile)) {
      consumer_sync();  // everyone is past the wait before the stage is overwritten
      manual_fill(s, tile, st);
      consumer_sync();
    }
    if (gathers) mbar_wait(&gfull[st], phase);
    if (++stage == stages) {
      stage = 0;
      phase ^= 1u;
    }
    return st;
  }

  // Consumers: done reading the oldest held stage (each warp arrives once).
  FB_DEV void release() {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&empty[rstage]);
    if (++rstage == stages) rstage = 0;
  }
};

using TileRing = TileRingT<false>;

}  // namespace fb
