// fb_common.cuh — shared device helpers for the factorized-LA kernels (sm_100a).
//
// PTX wrappers for the Blackwell async-copy path used by every streaming kernel:
// 1-D bulk copies (cp.async.bulk, SASS UBLKCP) global->shared completing on an
// mbarrier transaction count, plus warp reductions, the FP64 tensor-core MMA
// (mma.sync m8n8k4 f64 -> SASS DMMA; tcgen05 has no f64 kind) and status plumbing
// shared by the C-ABI in fb_capi.cu.
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

#define FB_DEV __device__ __forceinline__

namespace fb {

constexpr int kNumSMs = 148;  // B200; the host side re-queries it at runtime

// ---------------------------------------------------------------- mbarrier / bulk copy
FB_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

FB_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}

FB_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}

FB_DEV void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}

FB_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

FB_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile(
      "{\n .reg .b64 st;\n mbarrier.arrive.shared::cta.b64 st, [%0];\n}\n" ::"r"(smem_u32(bar))
      : "memory");
}

// Plain try_wait spin. (A suspend-time hint compiles to NANOSLEEP.SYNCS with that bound;
// with 1 ms it visibly delayed wake-ups in the LMM S pass, so waits use the default.)
FB_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "FB_WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra FB_WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

// global -> shared bulk copy; dst/src 16-byte aligned, bytes a multiple of 16.
FB_DEV void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// Same, with an L2 evict-first policy: streamed factor tiles are read exactly once.
FB_DEV void bulk_g2s_stream(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                            uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], "
      "%2, [%3], %4;\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

// 16-byte cp.async (LDGSTS) global -> shared, L2-only. Completion is signalled per thread
// with cp_async_arrive_noinc on an mbarrier whose expected count includes that arrival.
// No L2 cache-policy operand: with one, the gather loops of some kernels faulted with
// "Warp Illegal Instruction" at the LDGSTS (cuda-gdb, sm_100a) — the policy descriptor
// register was not valid on every path.
FB_DEV void cp_async16(void* dst, const void* src, uint64_t /*policy*/) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// The barrier address is broadcast from lane 0 so the compiler sees it warp-uniform
// (a non-uniform address makes it wrap ARRIVES.LDGSTSBAR in a per-address waterfall
// loop, which faulted with "illegal instruction" on sm_100a). Call with the warp converged.
// L1-allocating variant for lookup-table gathers: with skewed keys the hot rows are served
// from L1 instead of hammering one L2 line from every SM.
FB_DEV void cp_async16_ca(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

// Keyed gather of a lookup table far larger than L1 (uniform keys into a 100+ MB z): the
// L1-bypassing form. With a 224 KB ring L1 is only 32 KB, and L1-allocating LDGSTS then
// limit the gathers in flight (c2 X100x16: 1.575 -> 1.445 ms).
// (An evict_last policy operand on these gathers — `cp.async.cg...L2::cache_hint [d], [s], 16,
// 16, pol` — ran correctly but 2-3% slower at c2 X100x16 and did not raise the z hit rate.)
template <bool CG>
FB_DEV void cp_async16_gather(void* dst, const void* src) {
  if constexpr (CG)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

FB_DEV void cp_async_arrive_noinc(uint64_t* bar) {
  const uint32_t a = __shfl_sync(0xffffffffu, smem_u32(bar), 0);
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(a) : "memory");
}

FB_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

FB_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;\n" : "=l"(p));
  return p;
}

// A fraction `f` of the addresses (a fixed hash subset) evict_last, the rest evict_first: a
// lookup table larger than L2 keeps a stable resident subset instead of thrashing.
FB_DEV uint64_t policy_evict_last_frac(float f) {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.L2::evict_first.b64 %0, %1;\n" : "=l"(p) : "f"(f));
  return p;
}

// Fire-and-forget global reductions (SASS REDG). atomicAdd with an unused result may still
// compile to ATOMG, which holds a return slot until L2 answers: in the RMM S pass that cost
// 0.67 ms for 20M adds that a plain REDG loop issues in 0.13 ms (tools/red_probe.cu).
FB_DEV void red_add(double* p, double v) {
  asm volatile("red.relaxed.gpu.global.add.f64 [%0], %1;\n" ::"l"(p), "d"(v) : "memory");
}
FB_DEV void red_add(int* p, int v) {
  asm volatile("red.relaxed.gpu.global.add.s32 [%0], %1;\n" ::"l"(p), "r"(v) : "memory");
}

// Streaming 128-bit global loads that skip L1 allocation.
FB_DEV double2 ld_stream_d2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];\n"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p));
  return r;
}

// Cache-hinted scalar accesses: gathered lookup tables (z, bins) are loaded with an
// evict_last policy so the multi-GB streams around them do not push them out of L2;
// streamed outputs are stored evict_first.
FB_DEV double ld_hint(const double* p, uint64_t policy) {
  double r;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;\n" : "=d"(r) : "l"(p), "l"(policy));
  return r;
}

FB_DEV void st_hint(double* p, double v, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.f64 [%0], %1, %2;\n" ::"l"(p), "d"(v), "l"(policy) : "memory");
}

FB_DEV void st_hint2(double* p, double a, double b, uint64_t policy) {
  asm volatile("st.global.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;\n" ::"l"(p), "d"(a), "d"(b), "l"(policy)
               : "memory");
}

// ---------------------------------------------------------------- warp helpers
FB_DEV double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

FB_DEV int lane_id() { return threadIdx.x & 31; }

// Fixed-order sum of `count` per-CTA partials of one output: lane i adds partials i, i+32,
// ... in order, then a fixed xor tree. Deterministic for a fixed grid; the loads of one warp
// are independent, so the last CTA's tail costs a few L2 round trips instead of `count`.
FB_DEV double warp_sum_strided(const double* p, int count, size_t stride) {
  const int lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll 4
  for (int b = lane; b < count; b += 32) s += __ldcg(p + static_cast<size_t>(b) * stride);
  return warp_sum(s);
}

// ---------------------------------------------------------------- FP64 tensor core
// D(8x8) += A(8x4, row) * B(4x8, col). Fragment ownership (lane l, g = l>>2, t = l&3):
//   a = A[g][t], b = B[t][g], c0/c1 = C[g][2t], C[g][2t+1].
// `volatile` matters: a non-volatile mma.sync asm may be moved by the compiler into a divergent
// region (a masked operand select for a ragged k-step made the fused GNMF pass hang).
FB_DEV void dmma_8x8x4(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---------------------------------------------------------------- launch accounting
// Every kernel launch in the library goes through FB_LAUNCHED() so fb_launch_count()
// can report how many of our kernels ran (bench.py's gpu_launches).
// With FB_DEBUG_SYNC=1 in the environment every launch is followed by a device sync and
// a failing kernel is reported with its source location (development aid).
void count_launch(const char* file, int line);
#define FB_LAUNCHED() ::fb::count_launch(__FILE__, __LINE__)

// ---------------------------------------------------------------- launch geometry
inline int grid_for(int64_t work_items, int per_cta, int ctas_per_sm, int num_sms) {
  int64_t need = (work_items + per_cta - 1) / per_cta;
  int64_t cap = static_cast<int64_t>(num_sms) * ctas_per_sm;
  if (need < 1) need = 1;
  return static_cast<int>(need < cap ? need : cap);
}

}  // namespace fb
