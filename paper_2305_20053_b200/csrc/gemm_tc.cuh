#include <type_traits>
// gemm_tc.cuh -- tcgen05 GEMM back end (sm_100a): TMA -> SMEM (128B swizzle)
// -> tcgen05.mma.kind::f16 (bf16 x bf16 -> fp32 in TMEM) -> tcgen05.ld
// epilogue with the same fused functors as the SIMT kernel.
//
// Precision: every fp32 operand x is split x = hi + lo with hi = bf16(x),
// lo = bf16(x - hi) (|x - hi - lo| <= 2^-17 |x|), and C = A B^T is
// accumulated as A_hi B_hi + A_hi B_lo + A_lo B_hi (the lo*lo term is below
// fp32 resolution) -- "bf16x3".  Measured on the c1/c2 MLP chain this gives
// ~6e-6 relative risk-gradient error vs float64 (scripts/precision_study.py),
// inside the 1e-4 bar at twice the rate of a tf32x3 split.
//
// Kernel shape: persistent CTAs (one per SM), 256 threads:
//   warp 0      TMA producer (one elected lane), STAGES-deep smem ring
//   warp 1      MMA issuer (one lane): 3 x BK/16 tcgen05.mma per stage
//   warp 2      TMEM allocator (2 x BN fp32 columns: double-buffered accumulator)
//   warps 4..7  epilogue: tcgen05.ld 32x32b.x32 -> registers -> functor
// so the epilogue of tile i overlaps the mainloop of tile i+1.
#pragma once
#include "common.cuh"
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <tuple>
#include <vector>

namespace sdn {

// ---------------------------------------------------------------------------
// operands

// a bf16x3-split operand buffer: hi = bf16(x), lo = bf16(x - hi), row-major
// (rows x ld elements), used as a K-major GEMM operand via TMA
struct TcOperand {
  __nv_bfloat16* hi = nullptr;
  __nv_bfloat16* lo = nullptr;
  int64_t rows = 0;   // logical rows of the current contents
  int ld = 0;         // elements per row (= K of the GEMM that reads it)
};

struct TcWeights {
  bool enabled = false;
  std::vector<TcOperand> fwd, bwd;   // per layer: W (n_out x n_in) and W^T (n_in x n_out)
  TcOperand act[2];                  // activation / reverse-sweep operands (ping-pong)
  TcOperand seed;                    // reverse-sweep seed E
  TcOperand mr;                      // encoded samples (layer-0 A operand)
  std::vector<void*> allocs;
  std::map<std::tuple<const void*, int64_t, int, int>, CUtensorMap> maps;
  std::map<std::tuple<const void*, int64_t, int64_t, int64_t>, CUtensorMap> omaps;   // epilogue outputs
};

SDN_DEV void split_bf16(float x, __nv_bfloat16& h, __nv_bfloat16& l) {
  h = __float2bfloat16_rn(x);
  l = __float2bfloat16_rn(x - __bfloat162float(h));
}

// epilogue side-output: the split of the value that feeds the next GEMM
struct TcEpiSplit {
  __nv_bfloat16* hi;
  __nv_bfloat16* lo;
  int64_t ld;
  TcEpiSplit(const TcOperand* op = nullptr)
      : hi(op ? op->hi : nullptr), lo(op ? op->lo : nullptr), ld(op ? op->ld : 0) {}
  SDN_DEV void store(int64_t r, int c, float4 v) const {
    __nv_bfloat16 h0, h1, h2, h3, l0, l1, l2, l3;
    split_bf16(v.x, h0, l0); split_bf16(v.y, h1, l1);
    split_bf16(v.z, h2, l2); split_bf16(v.w, h3, l3);
    __nv_bfloat162* ph = reinterpret_cast<__nv_bfloat162*>(hi + r * ld + c);
    __nv_bfloat162* pl = reinterpret_cast<__nv_bfloat162*>(lo + r * ld + c);
    ph[0] = __halves2bfloat162(h0, h1); ph[1] = __halves2bfloat162(h2, h3);
    pl[0] = __halves2bfloat162(l0, l1); pl[1] = __halves2bfloat162(l2, l3);
  }
};

// output layer fused with the sweep's unit seeds (reduced frame, dense sweep):
// phi = shift + scale (acc + bias) -> C (fp32); seed = 2 sigma (phi + c) =
// a2 phi + b2 -> bf16x3 split (the reverse sweep's first A operand)
struct EpiAffineSeed {
  EpiAffine base;
  const float* a2;
  const float* b2;
  TcEpiSplit seed;
  // fused QoI (reduced frame): every 16-column chunk's fp64 partial of
  // phi . (phi + 2 c) -> qp[chunk][row] (row stride qld); k_qoi_part sums a row's
  // chunks in order, adds q0 and takes the moments (the tensor-core tile path only)
  const float* cq = nullptr;
  double* qp = nullptr;
  int64_t qld = 0;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float x[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      float y = x[j] + (base.bias ? base.bias[c + j] : 0.0f);
      if (base.scale) y *= base.scale[c + j];
      if (base.shift) y += base.shift[c + j];
      x[j] = y;
    }
    *reinterpret_cast<float4*>(base.C + r * base.ldc + c) = make_float4(x[0], x[1], x[2], x[3]);
    seed.store(r, c, make_float4(fmaf(a2[c], x[0], b2[c]), fmaf(a2[c + 1], x[1], b2[c + 1]),
                                 fmaf(a2[c + 2], x[2], b2[c + 2]), fmaf(a2[c + 3], x[3], b2[c + 3])));
  }
  SDN_DEV void col(int64_t, int, float) const {}   // r_u is a multiple of 4
};

template <class Epi>
struct TcChain {
  Epi base;
  TcEpiSplit split;
  // tensor-core chains: the residual input read from its bf16 split (the
  // previous layer's GEMM operand) instead of a separate fp32 copy
  TcEpiSplit prev;
  SDN_DEV void operator()(int64_t r, int c, float4 v) const {
    float4 o = base.apply(r, c, v);
    if (split.hi) split.store(r, c, o);
  }
  SDN_DEV void col(int64_t, int, float) const {}
};

// fp32 (rows x cols, ld_src) -> split operand (rows x ld_dst, zero-padded cols)
__global__ void k_split(int64_t rows, const int* __restrict__ rows_dev, int cols, int64_t ld_src,
                        const float* __restrict__ src, int ld_dst, __nv_bfloat16* __restrict__ hi,
                        __nv_bfloat16* __restrict__ lo) {
  if (rows_dev) rows = min(rows, (int64_t)*rows_dev);
  const int64_t total = rows * ld_dst;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = e / ld_dst;
    int c = (int)(e % ld_dst);
    float x = c < cols ? src[r * ld_src + c] : 0.0f;
    __nv_bfloat16 h, l;
    split_bf16(x, h, l);
    hi[e] = h;
    lo[e] = l;
  }
}

// fp32 W (n_out x n_in) -> split W^T (n_in x n_out)
__global__ void k_split_transpose(int n_out, int n_in, const float* __restrict__ W, __nv_bfloat16* __restrict__ hi,
                                  __nv_bfloat16* __restrict__ lo) {
  const int64_t total = (int64_t)n_out * n_in;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / n_out;   // row of W^T = column of W
    int o = (int)(e % n_out);
    __nv_bfloat16 h, l;
    split_bf16(W[(int64_t)o * n_in + i], h, l);
    hi[e] = h;
    lo[e] = l;
  }
}

// ---------------------------------------------------------------------------
// PTX wrappers

namespace tcx {

SDN_DEV uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

SDN_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
SDN_DEV void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
SDN_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
SDN_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "SDN_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SDN_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
SDN_DEV float exp2_ftz(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
SDN_DEV void fence_barrier_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
SDN_DEV void prefetch_tmap(const CUtensorMap* m) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(m)) : "memory");
}
SDN_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y)
      : "memory");
}
// 3-D variants: the split operands keep hi and lo in one allocation (lo at a
// fixed offset), a 3rd box dimension of 2 moves both halves in one instruction
SDN_DEV void tma_load_3d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::
          "r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
SDN_DEV void tma_store_3d(const CUtensorMap* map, const void* src, int x, int y, int z) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y), "r"(z)
               : "memory");
}
// TMA store smem tile -> global (bulk-group completion); the staging layout
// must match the map's swizzle (64B for 16 fp32, 32B for 16 bf16 per row)
SDN_DEV void tma_store_2d(const CUtensorMap* map, const void* src, int x, int y) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(x), "r"(y)
               : "memory");
}
SDN_DEV void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
SDN_DEV void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
SDN_DEV void bulk_wait0() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
SDN_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
SDN_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }
SDN_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// CTA-local progress counter in shared memory (chain publisher hand-off)
SDN_DEV void red_release_cta_smem(uint32_t* p, uint32_t v) {
  asm volatile("red.release.cta.shared::cta.add.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
SDN_DEV uint32_t ld_acquire_cta_smem(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
SDN_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
SDN_DEV void tmem_alloc(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
}
SDN_DEV void tmem_relinquish() { asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory"); }
SDN_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
SDN_DEV void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
SDN_DEV void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
SDN_DEV void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
SDN_DEV void mma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}
SDN_DEV void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]),
        "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]),
        "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr)
      : "memory");
}
SDN_DEV void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
        "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
      : "r"(taddr)
      : "memory");
}
SDN_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// ---- CTA pairs (cta_group::2): a cluster of two CTAs on one TPC computes a
// 256-row tile; each CTA holds 128 rows of A and half of B's rows in its own
// shared memory, the leader (rank 0) issues the MMAs for both, and each CTA's
// TMEM receives its own 128 accumulator rows.  Shared-window addresses with
// bit 24 cleared name the leader's copy of a barrier.
constexpr uint32_t PEER_MASK = 0xFEFFFFFFu;
SDN_DEV uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
SDN_DEV void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
// TMA load into this CTA's shared memory, completion counted on the LEADER's barrier
SDN_DEV void tma_load_3d_pair(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, "
      "%5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar) & PEER_MASK), "r"(x), "r"(y), "r"(z)
      : "memory");
}
// arrive on the leader's copy of a barrier.  The arrivals on these barriers
// hand TMEM accumulators back to the MMA issuer: the tcgen05 fences on both
// sides order the TMEM accesses, no generic-proxy memory is published, so the
// default (cta-scope) release is enough -- a cluster-scope release compiles
// to MEMBAR.ALL.GPU + ERRBAR, ~11% of an epilogue warp's time in the chains
// (profiles/r02g_fwd_chain_stalls.txt)
SDN_DEV void mbar_arrive_leader(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cluster.b64 _, [%0];" ::"r"(smem_u32(bar) & PEER_MASK) : "memory");
}
SDN_DEV void tmem_alloc_pair(uint32_t* dst, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(dst)), "r"(ncols)
               : "memory");
}
SDN_DEV void tmem_relinquish_pair() {
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
}
SDN_DEV void tmem_dealloc_pair(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols) : "memory");
}
// completion of the leader's MMAs -> the barrier at this offset in BOTH CTAs
SDN_DEV void commit_pair(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
SDN_DEV void mma_bf16_pair(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accum)
      : "memory");
}

// UMMA shared-memory descriptor: K-major, 128B swizzle, 8-row atoms of
// 1024 B (SBO), version 1 (sm_100), LBO unused for swizzled K-major (= 16 B)
// K-major, 64B swizzle (32 bf16 per row), 8-row atoms of 512 B (SBO)
SDN_DEV uint64_t sdesc_k64(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(512 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)4 << 61;
  return d;
}
SDN_DEV uint64_t sdesc_k128(uint32_t saddr) {
  uint64_t d = (uint64_t)((saddr >> 4) & 0x3FFFu);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// instruction descriptor: kind::f16, A/B bf16, D f32, both K-major, M x N
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

}  // namespace tcx

#ifndef SDN_ST256
#define SDN_ST256 3
#endif
constexpr int TC_BM = 128;
// optional device trace buffer (sdn_debug_gemm): per-phase clock64 stamps of CTA 0
static unsigned long long* g_tc_trace = nullptr;
// tuning switch: thread-issued coalesced stores instead of TMA stores
static bool g_tc_thread_stores = getenv("SDN_TC_THREAD_STORES") != nullptr;
// programmatic dependent launch between consecutive GEMMs (the next GEMM's
// prologue and launch overlap the previous one's tail).  Not while SMs are
// reserved for the side stream: early-resident dependent CTAs would take them
// (measured: slower there, faster and steadier everywhere else).  SDN_NO_PDL=1
// disables it.
static bool g_tc_pdl = getenv("SDN_NO_PDL") == nullptr;
static bool g_tc_pdl_now = true;      // cleared by the engine while side-stream work needs free SMs
// sdn_debug_gemm study switch (device): bit 0 skips the MMAs, bit 1 also the TMA loads
__device__ int g_tc_dbg_skip = 0;
// ring-epilogue phase trace (sdn_debug_gemm, SDN_EPI_TRACE): CTA 0 / warp 4 /
// lane 0, first two tiles, six chunks each, eight stamps per chunk
__device__ unsigned long long* g_tc_eptr = nullptr;
constexpr int TC_BK = 32;   // 32 bf16 = one 64-byte swizzle row (3-4 deep ring)

// per epilogue warp: two fp32 32x16 tiles + two bf16 32x16 tiles (6 KB)
constexpr uint32_t TC_EPI_WARP_BYTES = 6144;
constexpr int TC_EPI_WARPS = 12;               // three per TMEM lane quarter
constexpr int TC_THREADS = 32 * (4 + TC_EPI_WARPS);
// ring kernels: epilogue warps (three per lane quarter; four -- 16-column
// chunks of a 256-column tile split evenly -- measured slower at c2: the
// larger epilogue leaves the mainloop only two stages)
#ifndef TC_RING_EW
#define TC_RING_EW 12
#endif
#ifndef TC_RING_EW_BWD
#define TC_RING_EW_BWD 8      // reverse rings (4-KB slots, depth 3): 8 warps keep four mainloop stages
#endif
template <int RING, bool BWD = false>
struct EpiWarps {
  static constexpr int EW = !RING ? TC_EPI_WARPS : BWD ? TC_RING_EW_BWD : TC_RING_EW;
  static_assert(EW % 4 == 0 && EW >= 4, "epilogue warps come in lane-quarter groups of four (CS = 16 EW / 4)");
  static constexpr int THREADS = 32 * (4 + EW);
};

// RING > 0: the asynchronous-input epilogue (epi_ring): per warp RING
// 2-KB slots that TMA-load the epilogue's input tile ahead of use and then
// stage its bf16 split output, a 2-KB fp32 output tile, and a shared 4-KB
// bias copy; the mainloop ring gets whatever shared memory is left (2-4 stages)
constexpr uint32_t TC_SMEM_MAX = 232448;      // 227 KB opt-in per block
constexpr uint32_t TC_BAR_BYTES = 1024;       // mbarriers + TMEM slot
constexpr uint32_t SDN_CHAIN_BIAS_BYTES = 4096;  // persistent forward chain: room for every layer's bias (8 KB with the ring's 4 KB)
// (reverse-sweep rings, BWD: 4-KB slots holding the residual-gradient and
// act' input tiles, reused for the G and split outputs; no bias)
// (BK: K columns per mainloop stage -- 32 = 64-byte swizzle rows, the default;
// 64 = 128-byte swizzle rows, chain kernels only, SDN_CHAIN_BK=64)
template <int BN, int RING = 0, bool BWD = false, int CG = 1, int BK = TC_BK>
struct TcCfg {
  static constexpr int BK_ = BK;
  static constexpr uint32_t A_BYTES = TC_BM * BK * 2;
  static constexpr uint32_t B_BYTES = (BN / CG) * BK * 2;   // CTA pairs: each CTA holds half of B's rows
  static constexpr uint32_t STAGE_BYTES = 2 * A_BYTES + 2 * B_BYTES;
  static constexpr uint32_t EPI_WARP =
      !RING ? TC_EPI_WARP_BYTES : BWD ? (uint32_t)RING * 4096u : (uint32_t)RING * 2048u + 2048u;
  static constexpr uint32_t EPI_BYTES = EpiWarps<RING, BWD>::EW * EPI_WARP + ((RING && !BWD) ? 4096u : 0u);
  static constexpr int STAGES_FIT = (int)((TC_SMEM_MAX - EPI_BYTES - 1024 - TC_BAR_BYTES) / STAGE_BYTES);
  static constexpr int STAGES = RING ? (STAGES_FIT > 4 ? 4 : STAGES_FIT) : ((BN == 256) ? SDN_ST256 : 4);
  static constexpr uint32_t SMEM = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*align*/ + TC_BAR_BYTES;
};

// ---------------------------------------------------------------------------
// coalesced tile epilogue.  An epilogue warp owns 32 accumulator rows (one
// TMEM lane each) and walks the tile 16 columns at a time.  Global traffic
// goes through XOR-swizzled SMEM tiles so that both the row-per-thread side
// (TMEM layout) and the coalesced side (8 rows x 64 B per instruction) are
// bank-conflict free.

// fp32 32x16 tile: 4-float chunk j of row r lives at chunk j ^ ((r >> 1) & 3)
SDN_DEV int sw_f(int r, int j) { return r * 16 + ((j ^ ((r >> 1) & 3)) << 2); }
// bf16 32x16 tile as uint32 pairs: 16-B chunk h of row r at h ^ ((r >> 2) & 1)
SDN_DEV int sw_h(int r, int h) { return r * 8 + ((h ^ ((r >> 2) & 1)) << 2); }

struct TileRows {
  int64_t r0, M;          // first row of the warp's 32, valid-row bound
  const int* gather;      // optional row map for gathered inputs
  int rowdiv = 1;         // gathered inputs without a map: row r reads row r / rowdiv (tangent rows -> sample)
  SDN_DEV int64_t src(int64_t r) const { return gather ? (int64_t)gather[r] : r / rowdiv; }
};

// coalesced global -> smem (swizzled) for 32 rows x 16 fp32 columns
SDN_DEV void tile_in(float* buf, const float* src, int64_t ld, const TileRows& tr, bool gathered, int c0, int N,
                     int lane) {
  const int rr = lane >> 2, j = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + rr;
    const int64_t g = tr.r0 + r;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < tr.M && c0 + 4 * j < N)
      v = __ldg(reinterpret_cast<const float4*>(src + (gathered ? tr.src(g) : g) * ld + c0 + 4 * j));
    *reinterpret_cast<float4*>(buf + sw_f(r, j)) = v;
  }
}
// register prefetch of the next chunk's inputs (same coalesced pattern as
// tile_in), parked in smem once the current chunk has released it.  Each
// epilogue keeps only what it needs: two chunks of prefetch state must stay
// well inside the 128-register budget of a 512-thread CTA (no spills).
struct PreNone {};
struct PreAff {
  float4 b[4], s[4];     // folded bias (shift + scale*bias) and scale, lane-uniform
};
struct PreFwd {
  uint4 u[4];            // residual input: 4 fp32 float4 (bit-cast) or bf16 split hi[0..1] / lo[2..3]
  float4 c[4];           // bias, lane-uniform
};
struct PreBwd {
  float4 a[4], b[4];     // residual gradient, gathered derivative
};
SDN_DEV void tile_fetch(float4 (&p)[4], const float* src, int64_t ld, const TileRows& tr, bool gathered, int c0,
                        int N, int lane) {
  const int rr = lane >> 2, j = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int64_t g = tr.r0 + it * 8 + rr;
    p[it] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (g < tr.M && c0 + 4 * j < N)
      p[it] = __ldg(reinterpret_cast<const float4*>(src + (gathered ? tr.src(g) : g) * ld + c0 + 4 * j));
  }
}
SDN_DEV void tile_stash(float* buf, const float4 (&p)[4], int lane) {
  const int rr = lane >> 2, j = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) *reinterpret_cast<float4*>(buf + sw_f(it * 8 + rr, j)) = p[it];
}
// bf16 32x16 tile (hi or lo half of a split operand): coalesced fetch into
// registers (2 rows x 32 B per lane pair), stash into the sw_h layout
SDN_DEV void tile_fetch_h(uint4* p, const __nv_bfloat16* src, int64_t ld, const TileRows& tr, int c0, int N,
                          int lane) {
  const int rr = lane >> 1, h = lane & 1;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int64_t g = tr.r0 + it * 16 + rr;
    p[it] = make_uint4(0u, 0u, 0u, 0u);
    if (g < tr.M && c0 + 8 * h < N) p[it] = __ldg(reinterpret_cast<const uint4*>(src + g * ld + c0 + 8 * h));
  }
}
SDN_DEV void tile_stash_h(uint32_t* buf, const uint4* p, int lane) {
  const int rr = lane >> 1, h = lane & 1;
#pragma unroll
  for (int it = 0; it < 2; ++it) *reinterpret_cast<uint4*>(buf + sw_h(it * 16 + rr, h)) = p[it];
}
// row-per-thread read of hi + lo (fp32 reconstruction, exact to 2^-17 relative)
SDN_DEV void row_get_split(const uint32_t* bh, const uint32_t* bl, int lane, float (&x)[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const uint4 a = *reinterpret_cast<const uint4*>(bh + sw_h(lane, h));
    const uint4 b = *reinterpret_cast<const uint4*>(bl + sw_h(lane, h));
    const uint32_t av[4] = {a.x, a.y, a.z, a.w}, bv[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      x[8 * h + 2 * k] = __uint_as_float(av[k] << 16) + __uint_as_float(bv[k] << 16);
      x[8 * h + 2 * k + 1] = __uint_as_float(av[k] & 0xFFFF0000u) + __uint_as_float(bv[k] & 0xFFFF0000u);
    }
  }
}

// smem (swizzled) -> global, coalesced
SDN_DEV void tile_out(const float* buf, float* dst, int64_t ld, const TileRows& tr, int c0, int N, int lane) {
  const int rr = lane >> 2, j = lane & 3;
#pragma unroll
  for (int it = 0; it < 4; ++it) {
    const int r = it * 8 + rr;
    const int64_t g = tr.r0 + r;
    if (g < tr.M && c0 + 4 * j < N)
      *reinterpret_cast<float4*>(dst + g * ld + c0 + 4 * j) = *reinterpret_cast<const float4*>(buf + sw_f(r, j));
  }
}
SDN_DEV void tile_out_h(const uint32_t* buf, __nv_bfloat16* dst, int64_t ld, const TileRows& tr, int c0, int N,
                        int lane) {
  const int rr = lane >> 1, h = lane & 1;
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const int r = it * 16 + rr;
    const int64_t g = tr.r0 + r;
    if (g < tr.M && c0 + 8 * h < N)
      *reinterpret_cast<uint4*>(dst + g * ld + c0 + 8 * h) = *reinterpret_cast<const uint4*>(buf + sw_h(r, h));
  }
}
// row-per-thread accessors (thread = row `lane`)
SDN_DEV void row_get(const float* buf, int lane, float (&x)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    float4 v = *reinterpret_cast<const float4*>(buf + sw_f(lane, j));
    x[4 * j] = v.x; x[4 * j + 1] = v.y; x[4 * j + 2] = v.z; x[4 * j + 3] = v.w;
  }
}
SDN_DEV void row_put(float* buf, int lane, const float (&x)[16]) {
#pragma unroll
  for (int j = 0; j < 4; ++j)
    *reinterpret_cast<float4*>(buf + sw_f(lane, j)) = make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
}
SDN_DEV uint32_t pack_bf2(__nv_bfloat16 a, __nv_bfloat16 b) {
  return (uint32_t)__bfloat16_as_ushort(a) | ((uint32_t)__bfloat16_as_ushort(b) << 16);
}
// two fp32 -> packed bf16x2 (round to nearest), a in the low half
SDN_DEV uint32_t cvt_bf2(float a, float b) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(b), "f"(a));
  return d;
}
SDN_DEV void row_put_split(uint32_t* bh, uint32_t* bl, int lane, const float (&x)[16]) {
  uint32_t ph[8], pl[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    // same values as split_bf16: hi = bf16(x), lo = bf16(x - hi) (x - hi is exact)
    ph[k] = cvt_bf2(x[2 * k], x[2 * k + 1]);
    const float h0 = __uint_as_float(ph[k] << 16), h1 = __uint_as_float(ph[k] & 0xFFFF0000u);
    pl[k] = cvt_bf2(x[2 * k] - h0, x[2 * k + 1] - h1);
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    *reinterpret_cast<uint4*>(bh + sw_h(lane, h)) = make_uint4(ph[4 * h], ph[4 * h + 1], ph[4 * h + 2], ph[4 * h + 3]);
    *reinterpret_cast<uint4*>(bl + sw_h(lane, h)) = make_uint4(pl[4 * h], pl[4 * h + 1], pl[4 * h + 2], pl[4 * h + 3]);
  }
}

// output tensor maps of a TMA-store epilogue (slot meaning per epilogue:
// fwd hidden H, D, hi, lo; reverse G, U, hi, lo; affine C)
struct TcOutMaps {
  CUtensorMap m[6];      // m[4], m[5]: ring-epilogue input tiles (hi, lo or fp32 pair)
};

struct EpiSmem {
  float* f0;
  float* f1;
  uint32_t* h;
  uint32_t* l;
  const TcOutMaps* om;   // null: thread stores (tile_out)
};

// the warp's staged tiles -> TMA bulk stores (one elected lane)
SDN_DEV void epi_issue(const EpiSmem& s, int lane, int64_t r0, int c0, bool s0, bool s1, bool s2, bool s3) {
  tcx::fence_proxy_async();          // generic-proxy smem writes -> visible to the async proxy
  __syncwarp();
  if (lane == 0) {
    if (s0) tcx::tma_store_2d(&s.om->m[0], s.f0, c0, (int)r0);
    if (s1) tcx::tma_store_2d(&s.om->m[1], s.f1, c0, (int)r0);
    if (s2 || s3) tcx::tma_store_3d(&s.om->m[2], s.h, c0, (int)r0, 0);   // hi and lo (s.l = s.h + 1 KB)
    tcx::bulk_commit();
  }
}
// before the staging is rewritten: the previous chunk's stores have read it
SDN_DEV void epi_reclaim(const EpiSmem& s, int lane) {
  if (s.om) {
    if (lane == 0) tcx::bulk_wait_read0();
    __syncwarp();
  }
}

// generic path: row-per-thread functor calls (setup GEMMs, Jacobian scatter).
// Every TileEpi has load() (register prefetch of the next chunk's inputs)
// and chunk() (process one 32x16 chunk given its accumulator values).
template <class Epi>
struct TileEpi {
  using Pre = PreNone;
  static SDN_DEV void load(const Epi&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const Epi& epi, const EpiSmem&, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    const int64_t row = tr.r0 + lane;
    if (row >= tr.M) return;
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const int c = c0 + j;
      const float a0 = __uint_as_float(v[j]), a1 = __uint_as_float(v[j + 1]);
      const float a2 = __uint_as_float(v[j + 2]), a3 = __uint_as_float(v[j + 3]);
      if (c + 4 <= N) epi(row, c, make_float4(a0, a1, a2, a3));
      else if (c < N) epi_tail(epi, row, c, N - c, a0, a1, a2);
    }
  }
};

// fp64 accumulation of a K chunk's fp32 result (the encoder's split-K sum):
// the row's 16 doubles are loaded together, added and stored -- one global
// round trip per chunk (the generic functor path read-modify-writes four
// columns at a time: four dependent round trips)
template <>
struct TileEpi<EpiAccum64> {
  using Pre = PreNone;
  static SDN_DEV void load(const EpiAccum64&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const EpiAccum64& epi, const EpiSmem&, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    const int64_t row = tr.r0 + lane;
    if (row >= tr.M) return;
    double* p = epi.C + row * epi.ldc + c0;
    if (c0 + 16 <= N) {
      double2 d[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) d[j] = *reinterpret_cast<const double2*>(p + 2 * j);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        d[j].x += (double)__uint_as_float(v[2 * j]);
        d[j].y += (double)__uint_as_float(v[2 * j + 1]);
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) *reinterpret_cast<double2*>(p + 2 * j) = d[j];
    } else {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (c0 + j < N) p[j] += (double)__uint_as_float(v[j]);
    }
  }
};

// no-op epilogue (mainloop timing in sdn_debug_gemm)
struct EpiNull {
  SDN_DEV void operator()(int64_t, int, float4) const {}
  SDN_DEV void col(int64_t, int, float) const {}
};
template <>
struct TileEpi<EpiNull> {
  using Pre = PreNone;
  static SDN_DEV void load(const EpiNull&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const EpiNull&, const EpiSmem&, const TileRows&, int, int, int, const uint32_t (&)[16],
                            const Pre&) {}
};

// output layer: phi = shift + scale * (acc + bias)
template <>
struct TileEpi<EpiAffine> {
  // the folded bias / scale are read at use (lane-uniform, L1-resident): a
  // prefetched load still in flight at the proxy fence before the TMA stores
  // would be waited on there (MEMBAR), serialising every chunk on a global latency
  using Pre = PreNone;
  static SDN_DEV void load(const EpiAffine&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void fold(const EpiAffine& e, int c0, int N, PreAff& p) {
    const float4 z = make_float4(0.f, 0.f, 0.f, 0.f), o = make_float4(1.f, 1.f, 1.f, 1.f);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int c = min(c0 + 4 * j, N - 4);
      const float4 b = e.bias ? __ldg(reinterpret_cast<const float4*>(e.bias + c)) : z;
      const float4 s = e.scale ? __ldg(reinterpret_cast<const float4*>(e.scale + c)) : o;
      const float4 h = e.shift ? __ldg(reinterpret_cast<const float4*>(e.shift + c)) : z;
      p.s[j] = s;
      p.b[j] = make_float4(h.x + s.x * b.x, h.y + s.y * b.y, h.z + s.z * b.z, h.w + s.w * b.w);
    }
  }
  static SDN_DEV void chunk(const EpiAffine& e, const EpiSmem& s, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    PreAff pre;
    fold(e, c0, N, pre);
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 b = pre.b[j / 4], sc = pre.s[j / 4];
      x[j] = fmaf(sc.x, __uint_as_float(v[j]), b.x);
      x[j + 1] = fmaf(sc.y, __uint_as_float(v[j + 1]), b.y);
      x[j + 2] = fmaf(sc.z, __uint_as_float(v[j + 2]), b.z);
      x[j + 3] = fmaf(sc.w, __uint_as_float(v[j + 3]), b.w);
    }
    epi_reclaim(s, lane);
    row_put(s.f0, lane, x);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, true, false, false, false);
      return;
    }
    __syncwarp();
    tile_out(s.f0, e.C, e.ldc, tr, c0, N, lane);
    __syncwarp();
  }
};

template <>
struct TileEpi<EpiAffineSeed> {
  using Pre = PreNone;
  static SDN_DEV void load(const EpiAffineSeed&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const EpiAffineSeed& e, const EpiSmem& s, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    PreAff pre;
    TileEpi<EpiAffine>::fold(e.base, c0, N, pre);
    float x[16], sd[16];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 b = pre.b[j / 4], sc = pre.s[j / 4];
      x[j] = fmaf(sc.x, __uint_as_float(v[j]), b.x);
      x[j + 1] = fmaf(sc.y, __uint_as_float(v[j + 1]), b.y);
      x[j + 2] = fmaf(sc.z, __uint_as_float(v[j + 2]), b.z);
      x[j + 3] = fmaf(sc.w, __uint_as_float(v[j + 3]), b.w);
      const int c = min(c0 + j, N - 4);
      const float4 a2 = __ldg(reinterpret_cast<const float4*>(e.a2 + c));
      const float4 b2 = __ldg(reinterpret_cast<const float4*>(e.b2 + c));
      sd[j] = fmaf(a2.x, x[j], b2.x);
      sd[j + 1] = fmaf(a2.y, x[j + 1], b2.y);
      sd[j + 2] = fmaf(a2.z, x[j + 2], b2.z);
      sd[j + 3] = fmaf(a2.w, x[j + 3], b2.w);
    }
    if (e.qp) {                                  // this row's QoI partial over the chunk's columns (fp64)
      double q = 0.0;
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 cc = __ldg(reinterpret_cast<const float4*>(e.cq + min(c0 + j, N - 4)));
        const double p0 = x[j], p1 = x[j + 1], p2 = x[j + 2], p3 = x[j + 3];
        q += p0 * (p0 + 2.0 * (double)cc.x);
        q += p1 * (p1 + 2.0 * (double)cc.y);
        q += p2 * (p2 + 2.0 * (double)cc.z);
        q += p3 * (p3 + 2.0 * (double)cc.w);
      }
      if (tr.r0 + lane < tr.M) e.qp[(int64_t)(c0 >> 4) * e.qld + tr.r0 + lane] = q;
    }
    epi_reclaim(s, lane);
    row_put(s.f0, lane, x);
    row_put_split(s.h, s.l, lane, sd);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, true, false, true, true);
      return;
    }
    __syncwarp();
    tile_out(s.f0, e.base.C, e.base.ldc, tr, c0, N, lane);
    tile_out_h(s.h, e.seed.hi, e.seed.ld, tr, c0, N, lane);
    tile_out_h(s.l, e.seed.lo, e.seed.ld, tr, c0, N, lane);
    __syncwarp();
  }
};

// hidden-layer activation of one 16-column row chunk: a = [a +] act(v + b),
// d = act'(v + b)
SDN_DEV void fwd_act16(int act, const uint32_t (&v)[16], const float (&bias)[16], bool has_prev, float (&a)[16],
                       float (&d)[16]) {
  if (act == ACT_ELU) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      // branch-free (selects only) so the 16 elements interleave
      const float x = __uint_as_float(v[j]) + bias[j];
      const float xn = x > 0.0f ? 0.0f : x;     // (not fminf: a NaN must propagate, as in the oracle)
      const float ex = tcx::exp2_ftz(xn * 1.4426950408889634f);   // e^xn, xn <= 0 (flush below 2^-126)
      // e^x - 1 directly: near 0 its absolute error (~1e-7) is far below the
      // bf16x3 split error of the next GEMM operand (2^-17 |h|)
      const float y = x > 0.0f ? x : ex - 1.0f;
      a[j] = has_prev ? a[j] + y : y;
      d[j] = x > 0.0f ? 1.0f : ex;
    }
  } else {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      float y, dy;
      act_eval(act, __uint_as_float(v[j]) + bias[j], y, dy);
      a[j] = has_prev ? a[j] + y : y;
      d[j] = dy;
    }
  }
}

// hidden layer forward: H = [prev +] act(acc + b), D = act'(.), split(H).
// In a tensor-core chain prev comes from the previous layer's bf16 split
// (ch.prev) and the fp32 H is not written (e.H == nullptr).
template <>
struct TileEpi<TcChain<EpiFwdHidden>> {
  using Pre = PreFwd;
  static SDN_DEV void load(const TcChain<EpiFwdHidden>& ch, const TileRows& tr, int c0, int N, int lane, Pre& p) {
    if (ch.prev.hi) {
      tile_fetch_h(p.u, ch.prev.hi, ch.prev.ld, tr, c0, N, lane);
      tile_fetch_h(p.u + 2, ch.prev.lo, ch.prev.ld, tr, c0, N, lane);
    } else if (ch.base.prev) {
      tile_fetch(reinterpret_cast<float4(&)[4]>(p.u), ch.base.prev, ch.base.ld, tr, false, c0, N, lane);
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) p.c[j] = __ldg(reinterpret_cast<const float4*>(ch.base.bias + min(c0 + 4 * j, N - 4)));
  }
  static SDN_DEV void chunk(const TcChain<EpiFwdHidden>& ch, const EpiSmem& s, const TileRows& tr, int c0, int N,
                            int lane, const uint32_t (&v)[16], const Pre& pre) {
    const EpiFwdHidden& e = ch.base;
    const bool has_prev = ch.prev.hi || e.prev;
    float a[16], d[16];
    epi_reclaim(s, lane);
    if (ch.prev.hi) {
      tile_stash_h(s.h, pre.u, lane);
      tile_stash_h(s.l, pre.u + 2, lane);
      __syncwarp();
      row_get_split(s.h, s.l, lane, a);
    } else if (e.prev) {
      tile_stash(s.f0, reinterpret_cast<const float4(&)[4]>(pre.u), lane);
      __syncwarp();
      row_get(s.f0, lane, a);
    }
    float bias[16];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 b4 = pre.c[j / 4];
      bias[j] = b4.x; bias[j + 1] = b4.y; bias[j + 2] = b4.z; bias[j + 3] = b4.w;
    }
    fwd_act16(e.act, v, bias, has_prev, a, d);
    __syncwarp();
    if (e.H) row_put(s.f0, lane, a);
    if (e.D) row_put(s.f1, lane, d);
    if (ch.split.hi) row_put_split(s.h, s.l, lane, a);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, e.H, e.D, ch.split.hi, ch.split.hi);
      return;
    }
    __syncwarp();
    if (e.H) tile_out(s.f0, e.H, e.ld, tr, c0, N, lane);
    if (e.D) tile_out(s.f1, e.D, e.ld, tr, c0, N, lane);
    if (ch.split.hi) {
      tile_out_h(s.h, ch.split.hi, ch.split.ld, tr, c0, N, lane);
      tile_out_h(s.l, ch.split.lo, ch.split.ld, tr, c0, N, lane);
    }
    __syncwarp();
  }
};

// reverse step: g = acc [+ resid]; U = D[row] g; G = g (optional); split(U).
// In a tensor-core chain the fp32 U is not written (e.U == nullptr).
template <>
struct TileEpi<TcChain<EpiBwd>> {
  using Pre = PreBwd;
  static SDN_DEV void load(const TcChain<EpiBwd>& ch, const TileRows& tr, int c0, int N, int lane, Pre& p) {
    const EpiBwd& e = ch.base;
    TileRows tg = tr;
    tg.gather = e.rowidx;
    if (e.resid) tile_fetch(p.a, e.resid, e.ld, tr, false, c0, N, lane);
    tile_fetch(p.b, e.D, e.ldD, tg, true, c0, N, lane);
  }
  static SDN_DEV void chunk(const TcChain<EpiBwd>& ch, const EpiSmem& s, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre& pre) {
    const EpiBwd& e = ch.base;
    epi_reclaim(s, lane);
    if (e.resid) tile_stash(s.f0, pre.a, lane);
    tile_stash(s.f1, pre.b, lane);
    __syncwarp();
    float g[16], dd[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) g[j] = __uint_as_float(v[j]);
    if (e.resid) {
      float r[16];
      row_get(s.f0, lane, r);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] += r[j];
    }
    row_get(s.f1, lane, dd);
#pragma unroll
    for (int j = 0; j < 16; ++j) dd[j] *= g[j];
    __syncwarp();
    if (e.G) row_put(s.f0, lane, g);
    if (e.U) row_put(s.f1, lane, dd);
    if (ch.split.hi) row_put_split(s.h, s.l, lane, dd);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, e.G, e.U, ch.split.hi, ch.split.hi);
      return;
    }
    __syncwarp();
    if (e.G) tile_out(s.f0, e.G, e.ld, tr, c0, N, lane);
    if (e.U) tile_out(s.f1, e.U, e.ld, tr, c0, N, lane);
    if (ch.split.hi) {
      tile_out_h(s.h, ch.split.hi, ch.split.ld, tr, c0, N, lane);
      tile_out_h(s.l, ch.split.lo, ch.split.ld, tr, c0, N, lane);
    }
    __syncwarp();
  }
};

// forward-mode tangent step on the tensor cores (surrogate.py:208-223, with
// the residual): T_out = D[row / rowdiv] * acc [+ T_in].  Tangent rows are
// (sample i, control k) = i * d_z + k, so rowdiv = d_z gathers the sample's
// act' row.  T_in is read from the split of the layer input (the A operand,
// ch.prev) and T_out is written only as the next GEMM's split (ch.split).
struct EpiTanTc {
  const float* D;
  int64_t ldD;
  int rowdiv;
  SDN_DEV void operator()(int64_t, int, float4) const {}
  SDN_DEV void col(int64_t, int, float) const {}
};
struct PreTan {
  float4 d[4];           // gathered act'
  uint4 u[4];            // T_in split: hi[0..1] / lo[2..3]
};
template <>
struct TileEpi<TcChain<EpiTanTc>> {
  using Pre = PreTan;
  static SDN_DEV void load(const TcChain<EpiTanTc>& ch, const TileRows& tr, int c0, int N, int lane, Pre& p) {
    TileRows tg = tr;
    tg.gather = nullptr;
    tg.rowdiv = ch.base.rowdiv;
    tile_fetch(p.d, ch.base.D, ch.base.ldD, tg, true, c0, N, lane);
    if (ch.prev.hi) {
      tile_fetch_h(p.u, ch.prev.hi, ch.prev.ld, tr, c0, N, lane);
      tile_fetch_h(p.u + 2, ch.prev.lo, ch.prev.ld, tr, c0, N, lane);
    }
  }
  static SDN_DEV void chunk(const TcChain<EpiTanTc>& ch, const EpiSmem& s, const TileRows& tr, int c0, int N,
                            int lane, const uint32_t (&v)[16], const Pre& pre) {
    epi_reclaim(s, lane);
    tile_stash(s.f1, pre.d, lane);
    if (ch.prev.hi) {
      tile_stash_h(s.h, pre.u, lane);
      tile_stash_h(s.l, pre.u + 2, lane);
    }
    __syncwarp();
    float t[16], dd[16];
    row_get(s.f1, lane, dd);
    if (ch.prev.hi) row_get_split(s.h, s.l, lane, t);
    else
#pragma unroll
      for (int j = 0; j < 16; ++j) t[j] = 0.0f;
#pragma unroll
    for (int j = 0; j < 16; ++j) t[j] = fmaf(dd[j], __uint_as_float(v[j]), t[j]);
    __syncwarp();
    row_put_split(s.h, s.l, lane, t);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, false, false, true, true);
      return;
    }
    __syncwarp();
    tile_out_h(s.h, ch.split.hi, ch.split.ld, tr, c0, N, lane);
    tile_out_h(s.l, ch.split.lo, ch.split.ld, tr, c0, N, lane);
    __syncwarp();
  }
};

// Jacobian scatter on the tensor-core path: row r = i d_z + k, column u ->
// J[i, u, k] (* scale[u]).  A warp's 32 rows are consecutive k of one or two
// samples, so each column's store is one or two contiguous runs; (i, k) is
// computed once per chunk in 32-bit arithmetic.
template <>
struct TileEpi<EpiJacScatter> {
  using Pre = PreNone;
  static SDN_DEV void load(const EpiJacScatter&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const EpiJacScatter& e, const EpiSmem&, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    const int64_t row = tr.r0 + lane;
    if (row >= tr.M) return;
    const unsigned rr = (unsigned)row, dz = (unsigned)e.d_z;
    const unsigned i = rr / dz, k = rr - i * dz;
    float* base = e.J + (int64_t)i * e.ncol * e.d_z + k;
    const int nv = (int)(e.nvalid ? e.nvalid : e.ncol);
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      const int c = c0 + j;
      if (c < nv) {
        const float x = __uint_as_float(v[j]);
        __stcs(base + (int64_t)c * e.d_z, e.scale ? x * __ldg(e.scale + c) : x);   // streaming: written once
      }
    }
  }
};

// scale * acc -> bf16x3 split only (the Jacobian's output layer when it is
// decoded next: std . (T W^T) feeds the decoder GEMM)
struct EpiScaleSplit {
  const float* scale;
  TcEpiSplit split;
  SDN_DEV void operator()(int64_t, int, float4) const {}
  SDN_DEV void col(int64_t, int, float) const {}
};
template <>
struct TileEpi<EpiScaleSplit> {
  using Pre = PreNone;
  static SDN_DEV void load(const EpiScaleSplit&, const TileRows&, int, int, int, Pre&) {}
  static SDN_DEV void chunk(const EpiScaleSplit& e, const EpiSmem& s, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre&) {
    float x[16];
#pragma unroll
    for (int j = 0; j < 16; j += 4) {
      const float4 sc = __ldg(reinterpret_cast<const float4*>(e.scale + min(c0 + j, N - 4)));
      x[j] = sc.x * __uint_as_float(v[j]);
      x[j + 1] = sc.y * __uint_as_float(v[j + 1]);
      x[j + 2] = sc.z * __uint_as_float(v[j + 2]);
      x[j + 3] = sc.w * __uint_as_float(v[j + 3]);
    }
    epi_reclaim(s, lane);
    row_put_split(s.h, s.l, lane, x);
    if (s.om) {
      epi_issue(s, lane, tr.r0, c0, false, false, true, true);
      return;
    }
    __syncwarp();
    tile_out_h(s.h, e.split.hi, e.split.ld, tr, c0, N, lane);
    tile_out_h(s.l, e.split.lo, e.split.ld, tr, c0, N, lane);
    __syncwarp();
  }
};

// last reverse step with the sample reduction fused: u = D[row] (acc + resid)
// is never stored; each (M tile, lane quarter) writes fp64 column sums of its
// 32 rows to part[(tile_m * 4 + quarter) * ldp + c] (fixed order, no atomics)
struct EpiBwdSum {
  const float* resid; const float* D; int64_t ldD; const int* rowidx; int64_t ld;
  double* part; int64_t ldp;
  // unified sweep: per-row risk weights W[row * R + r] (sweep rows), one
  // partial plane per risk (plane stride); W null = unit weights, R = 1
  const double* W = nullptr; int R = 1; int64_t plane = 0;
  // optional: u = D g itself stored (fp32, ld) through TMA by the ring
  // epilogue, for sums whose row weights are known only later (exact CVaR)
  float* U0 = nullptr;
  // weights computed in the epilogue from Q and the moments (wfun != 0)
  // instead of read from W: no weights kernel ahead of this GEMM
  int wfun = 0;
  RiskSet rs{};
  const double* Q = nullptr;
  const double* st = nullptr;
  double shift = 0.0;
  SDN_DEV bool has_w() const { return W != nullptr || wfun != 0; }
  SDN_DEV double weight(int64_t row, int q) const {
    return wfun ? risk_weight(rs, q, row, Q[row], st, shift) : W[row * R + q];
  }
  SDN_DEV void operator()(int64_t, int, float4) const {}
  SDN_DEV void col(int64_t, int, float) const {}
};
template <>
struct TileEpi<EpiBwdSum> {
  using Pre = PreBwd;
  static SDN_DEV void load(const EpiBwdSum& e, const TileRows& tr, int c0, int N, int lane, Pre& p) {
    TileRows tg = tr;
    tg.gather = e.rowidx;
    if (e.resid) tile_fetch(p.a, e.resid, e.ld, tr, false, c0, N, lane);
    tile_fetch(p.b, e.D, e.ldD, tg, true, c0, N, lane);
  }
  static SDN_DEV void chunk(const EpiBwdSum& e, const EpiSmem& s, const TileRows& tr, int c0, int N, int lane,
                            const uint32_t (&v)[16], const Pre& pre) {
    if (e.resid) tile_stash(s.f0, pre.a, lane);
    tile_stash(s.f1, pre.b, lane);
    __syncwarp();
    float g[16], dd[16];
#pragma unroll
    for (int j = 0; j < 16; ++j) g[j] = __uint_as_float(v[j]);
    if (e.resid) {
      float r[16];
      row_get(s.f0, lane, r);
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] += r[j];
    }
    row_get(s.f1, lane, dd);
    const bool live = tr.r0 + lane < tr.M;        // rows past M hold stale operand data
#pragma unroll
    for (int j = 0; j < 16; ++j) dd[j] = live ? dd[j] * g[j] : 0.0f;
    __syncwarp();
    row_put(s.f1, lane, dd);
    if (e.U0) {                                   // u itself for deferred sums (coalesced thread stores)
      __syncwarp();
      tile_out(s.f1, e.U0, e.ld, tr, c0, N, lane);
    }
    // unified sweep: each lane stages its row's risk weights (fp64) in the
    // residual staging buffer, free at this point
    double* ws = reinterpret_cast<double*>(s.f0);
    if (e.has_w())
      for (int q = 0; q < e.R; ++q) ws[q * 32 + lane] = live ? e.weight(tr.r0 + lane, q) : 0.0;
    __syncwarp();
    const int64_t prow = (tr.r0 >> 7) * 4 + ((tr.r0 >> 5) & 3);
    const int j = lane & 15;                      // column of the chunk
    if (!e.has_w()) {
      if (lane < 16 && c0 + j < N) {
        double acc = 0.0;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) acc += (double)s.f1[sw_f(r, j >> 2) + (j & 3)];
        e.part[prow * e.ldp + c0 + j] = acc;
      }
    } else if (c0 + j < N) {
      // half-warps take alternate risks: lanes 0-15 risk q, lanes 16-31 risk q+1
      for (int q = lane >> 4; q < e.R; q += 2) {
        double acc = 0.0;
#pragma unroll 8
        for (int r = 0; r < 32; ++r) acc += ws[q * 32 + r] * (double)s.f1[sw_f(r, j >> 2) + (j & 3)];
        e.part[q * e.plane + prow * e.ldp + c0 + j] = acc;
      }
    }
    __syncwarp();
  }
};

// Row-block readiness between consecutive chain GEMMs (with PDL): the
// producing GEMM adds, per 128-row block, 32 x the columns each epilogue warp
// finished once its TMA stores are complete (release); a consuming GEMM
// waits (acquire) until its A row block reached 128 x K before loading it --
// so CTAs that become resident on SMs the previous GEMM's last wave left idle
// start on row blocks already done instead of waiting for the whole grid.
struct TcFlags {
  const int* in = nullptr;   // readiness of this GEMM's A operand rows (null: whole-grid dependency)
  int* out = nullptr;        // readiness of this GEMM's outputs
  int hi_only = 0;           // issue only the hi x hi MMAs (the lo halves are loaded but ignored): encoder pass B
};

// persistent tile walk of one CTA: tiles t0, t0 + ts, ...; a tile covers
// TC_BM * CG rows, of which this CTA's epilogue owns the 128 at row_off
struct TileWalk {
  int t0, ts, row_off;
};
// accumulator drained: tell the MMA issuer (the leader's barrier for pairs)
template <int CG>
SDN_DEV void tmem_release(uint64_t* tempty) {
  if constexpr (CG == 1) tcx::mbar_arrive(tempty);
  else tcx::mbar_arrive_leader(tempty);
}

// ---------------------------------------------------------------------------
// asynchronous-input epilogue for the forward chain (RING slots per warp).
// The epilogue used to prefetch its residual input through registers one
// chunk ahead; the loads were then still in flight at the proxy fence before
// the TMA stores (MEMBAR), so every chunk paid a full global latency.  Here
// the residual tiles (the previous layer's bf16 split, 32 rows x 16 columns)
// are TMA-loaded RING-1 chunks ahead into per-warp slots (async proxy,
// mbarrier completion, no registers held), the chunk's split output is
// staged in the slot it was read from, and the bias comes from a per-CTA
// shared copy.  The chunk order per warp runs across the CTA's tiles, so the
// next tile's first residual tiles load during the current tile's last chunks.
template <int BN, int RING, int CG>
SDN_DEV void epi_fwd_ring(const TcChain<EpiFwdHidden>& ch, const TcOutMaps& om, uint8_t* epi_base, uint64_t* rbar_all,
                          uint64_t* tfull, uint64_t* tempty, uint32_t tmem, int warp, int lane, int num_tiles,
                          int n_tiles, int N, int K, const TcFlags& flags, const TileWalk tw) {
  constexpr int BMT = TC_BM * CG;
  constexpr uint32_t WB = (uint32_t)RING * 2048u + 2048u;
  constexpr int EW = EpiWarps<RING>::EW, CS = 16 * (EW / 4);   // chunk stride of a warp
  const int w = warp - 4, q = warp & 3, first_c = 16 * (w >> 2);
  uint8_t* wb = epi_base + w * WB;
  float* Dst = reinterpret_cast<float*>(wb + RING * 2048);
  float* bias_s = reinterpret_cast<float*>(epi_base + EW * WB);
  uint64_t* rbar = rbar_all + w * RING;
  const EpiFwdHidden& e = ch.base;
  const bool has_prev = ch.prev.hi != nullptr, has_split = ch.split.hi != nullptr, has_D = e.D != nullptr;
  const bool bias_smem = N <= 1024;
  const int dbg = g_tc_dbg_skip;                  // study switches (sdn_debug_gemm): 16 no fence, 32 no TMEM load
  unsigned long long* etr = (dbg & 64) && blockIdx.x == 0 && warp == 4 && lane == 0 ? g_tc_eptr : nullptr;
  int ti = 0;
#define EPI_STAMP(k) if (etr && ti < 2 && ci < 6) etr[(ti * 6 + ci) * 8 + (k)] = clock64()
  if (bias_smem)
    for (int i = (int)threadIdx.x - 128; i < N; i += 32 * EW) bias_s[i] = __ldg(e.bias + i);
  asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");

  // load cursor (tile lt, column lc), RING-1 chunks ahead of the compute cursor
  int lt = tw.t0, lc = first_c, jl = 0, last_mb = -1;
  auto lnorm = [&]() {
    while (lt < num_tiles && !(lc < BN && (lt % n_tiles) * BN + lc < N)) { lt += tw.ts; lc = first_c; }
  };
  auto issue = [&]() {
    if (lt >= num_tiles) return;
    if (has_prev) {
      const int mb = (lt / n_tiles) * CG + tw.row_off / TC_BM, s = jl % RING;   // 128-row block
      if (lane == 0) {
        if (flags.in && mb != last_mb) {          // rows of the previous layer written and visible
          while (tcx::ld_acquire(flags.in + mb) < TC_BM * K) __nanosleep(64);
          tcx::fence_proxy_async_global();
        }
        tcx::mbar_expect_tx(&rbar[s], 2048);
        const int x = (lt % n_tiles) * BN + lc, y = mb * TC_BM + q * 32;
        tcx::tma_load_3d(wb + s * 2048, &om.m[4], &rbar[s], x, y, 0);   // hi then lo (+1 KB)
      }
      last_mb = mb;
    }
    ++jl;
    lc += CS;
    lnorm();
  };
  lnorm();
  for (int k = 0; k < RING - 1; ++k) issue();

  int acc = 0, jc = 0;
  uint32_t acc_phase = 0;
  for (int tile = tw.t0; tile < num_tiles; tile += tw.ts) {
    const int mb = (tile / n_tiles) * CG + tw.row_off / TC_BM, nb = tile % n_tiles;   // 128-row block
    const int r0 = mb * TC_BM + q * 32;
    int nch = 0;
    for (int c = first_c; c < BN && nb * BN + c < N; c += CS) ++nch;
    tcx::mbar_wait(&tfull[acc], acc_phase);
    tcx::fence_after();
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
    if (nch == 0) {
      tcx::fence_before();
      __syncwarp();
      if (lane == 0) tmem_release<CG>(&tempty[acc]);
    }
#pragma unroll 1
    for (int ci = 0; ci < nch; ++ci, ++jc) {
      const int c0 = first_c + CS * ci, col = nb * BN + c0, s = jc % RING;
      uint32_t* sh = reinterpret_cast<uint32_t*>(wb + s * 2048);
      uint32_t* sl = sh + 256;
      uint32_t v[16];
      EPI_STAMP(0);
      if (!(dbg & 32)) tcx::tmem_ld16(tbase + c0, v);
      else for (int j = 0; j < 16; ++j) v[j] = __float_as_uint((float)(lane - j));
      if (has_prev) tcx::mbar_wait(&rbar[s], (uint32_t)(jc / RING) & 1u);
      EPI_STAMP(1);
      if (!(dbg & 32)) tcx::tmem_ld_wait();
      EPI_STAMP(2);
      if (ci == nch - 1) {                        // accumulator drained: the MMA may reuse it
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) tmem_release<CG>(&tempty[acc]);
      }
      float a[16], d[16], bias[16];
      if (has_prev) row_get_split(sh, sl, lane, a);
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 b4 = bias_smem ? *reinterpret_cast<const float4*>(bias_s + col + j)
                                    : __ldg(reinterpret_cast<const float4*>(e.bias + col + j));
        bias[j] = b4.x; bias[j + 1] = b4.y; bias[j + 2] = b4.z; bias[j + 3] = b4.w;
      }
      fwd_act16(e.act, v, bias, has_prev, a, d);
      EPI_STAMP(3);
      // the previous chunk's stores have read the output tile and its slot:
      // refill that slot RING-1 chunks ahead
      if (lane == 0) tcx::bulk_wait_read0();
      __syncwarp();
      EPI_STAMP(4);
      issue();
      EPI_STAMP(5);
      if (has_D) row_put(Dst, lane, d);
      if (has_split) row_put_split(sh, sl, lane, a);
      if (!(dbg & 16)) tcx::fence_proxy_async();
      else if (!has_D && !has_split) { float z = 0.f; for (int j = 0; j < 16; ++j) z += a[j] + d[j]; if (z == 1.2345f) Dst[lane] = z; }
      __syncwarp();
      EPI_STAMP(6);
      if (lane == 0) {
        if (has_D) tcx::tma_store_2d(&om.m[1], Dst, col, r0);
        if (has_split) {
          tcx::tma_store_3d(&om.m[2], sh, col, r0, 0);                  // hi, lo (sl = sh + 1 KB)
        }
        tcx::bulk_commit();
      }
      EPI_STAMP(7);
    }
    ++ti;
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    if (flags.out) {                              // publish this warp's part of the row block
      __syncwarp();
      if (lane == 0) {
        tcx::bulk_wait0();
        tcx::fence_proxy_async_global();
        tcx::red_release_add(flags.out + mb, 32 * 16 * nch);
      }
    }
  }
  if (lane == 0) tcx::bulk_wait0();
#undef EPI_STAMP
}

// asynchronous-input epilogue for the dense reverse sweep (no row gather):
// per chunk the residual-gradient tile (fp32, optional) and the act' tile
// (fp32) are TMA-loaded RING-1 chunks ahead into one 4-KB slot; the chain
// step stages G in the residual half and the bf16 split of u = D g in the
// act' half for its TMA stores; the summing step (EpiBwdSum) stages u and
// the per-row risk weights there for its fixed-order fp64 column sums.
template <class Epi>
struct BwdRingView;
template <>
struct BwdRingView<TcChain<EpiBwd>> {
  static constexpr bool SUM = false;
  static SDN_DEV const float* resid(const TcChain<EpiBwd>& c) { return c.base.resid; }
};
template <>
struct BwdRingView<EpiBwdSum> {
  static constexpr bool SUM = true;
  static SDN_DEV const float* resid(const EpiBwdSum& e) { return e.resid; }
};

template <int BN, int RING, int CG, class Epi>
SDN_DEV void epi_bwd_ring(const Epi& ep, const TcOutMaps& om, uint8_t* epi_base, uint64_t* rbar_all,
                          uint64_t* tfull, uint64_t* tempty, uint32_t tmem, int warp, int lane, int num_tiles,
                          int n_tiles, int64_t M, int N, const TileWalk tw) {
  constexpr int BMT = TC_BM * CG;
  constexpr bool SUM = BwdRingView<Epi>::SUM;
  constexpr uint32_t WB = (uint32_t)RING * 4096u;
  constexpr int EW = EpiWarps<RING, true>::EW, CS = 16 * (EW / 4);   // chunk stride of a warp
  const int w = warp - 4, q = warp & 3, first_c = 16 * (w >> 2);
  uint8_t* wb = epi_base + w * WB;
  uint64_t* rbar = rbar_all + w * RING;
  const bool has_resid = BwdRingView<Epi>::resid(ep) != nullptr;
  const uint32_t tx = has_resid ? 4096u : 2048u;

  int lt = tw.t0, lc = first_c, jl = 0;
  auto lnorm = [&]() {
    while (lt < num_tiles && !(lc < BN && (lt % n_tiles) * BN + lc < N)) { lt += tw.ts; lc = first_c; }
  };
  auto issue = [&]() {
    if (lt >= num_tiles) return;
    const int s = jl % RING;
    if (lane == 0) {
      const int x = (lt % n_tiles) * BN + lc, y = (lt / n_tiles) * BMT + tw.row_off + q * 32;
      tcx::mbar_expect_tx(&rbar[s], tx);
      if (has_resid) tcx::tma_load_2d(wb + s * 4096, &om.m[4], &rbar[s], x, y);
      tcx::tma_load_2d(wb + s * 4096 + 2048, &om.m[5], &rbar[s], x, y);
    }
    ++jl;
    lc += CS;
    lnorm();
  };
  lnorm();
  for (int k = 0; k < RING - 1; ++k) issue();

  int acc = 0, jc = 0;
  uint32_t acc_phase = 0;
  for (int tile = tw.t0; tile < num_tiles; tile += tw.ts) {
    const int mb = tile / n_tiles, nb = tile % n_tiles;
    const int64_t r0 = (int64_t)mb * BMT + tw.row_off + q * 32;
    int nch = 0;
    for (int c = first_c; c < BN && nb * BN + c < N; c += CS) ++nch;
    // summing step: this lane's row weights (up to 4 risks) once per tile, not per chunk
    double wreg[4] = {0.0, 0.0, 0.0, 0.0};
    if constexpr (SUM) {
      const EpiBwdSum& e = ep;
      if (e.has_w() && r0 + lane < M)
#pragma unroll
        for (int qq = 0; qq < 4; ++qq)
          if (qq < e.R) wreg[qq] = e.weight(r0 + lane, qq);
    }
    tcx::mbar_wait(&tfull[acc], acc_phase);
    tcx::fence_after();
    const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
    if (nch == 0) {
      tcx::fence_before();
      __syncwarp();
      if (lane == 0) tmem_release<CG>(&tempty[acc]);
    }
#pragma unroll 1
    for (int ci = 0; ci < nch; ++ci, ++jc) {
      const int c0 = first_c + CS * ci, col = nb * BN + c0, s = jc % RING;
      float* Rs = reinterpret_cast<float*>(wb + s * 4096);
      float* Ds = Rs + 512;
      uint32_t v[16];
      tcx::tmem_ld16(tbase + c0, v);
      tcx::mbar_wait(&rbar[s], (uint32_t)(jc / RING) & 1u);
      tcx::tmem_ld_wait();
      if (ci == nch - 1) {
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) tmem_release<CG>(&tempty[acc]);
      }
      float g[16], dd[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) g[j] = __uint_as_float(v[j]);
      if (has_resid) {
        float r[16];
        row_get(Rs, lane, r);
#pragma unroll
        for (int j = 0; j < 16; ++j) g[j] += r[j];
      }
      row_get(Ds, lane, dd);
      if constexpr (SUM) {
        const EpiBwdSum& e = ep;
        const bool live = r0 + lane < M;           // rows past M hold stale operand data
#pragma unroll
        for (int j = 0; j < 16; ++j) dd[j] = live ? dd[j] * g[j] : 0.0f;
        __syncwarp();
        row_put(Ds, lane, dd);
        double* ws = reinterpret_cast<double*>(Rs);   // per-row risk weights (fp64)
        if (e.has_w()) {
#pragma unroll
          for (int qq = 0; qq < 4; ++qq)
            if (qq < e.R) ws[qq * 32 + lane] = wreg[qq];
          for (int qq = 4; qq < e.R; ++qq) ws[qq * 32 + lane] = live ? e.weight(r0 + lane, qq) : 0.0;
        }
        __syncwarp();
        const int64_t prow = (r0 >> 7) * 4 + ((r0 >> 5) & 3);
        const int j = lane & 15;
        if (!e.has_w()) {
          if (lane < 16 && col + j < N) {
            double a = 0.0;
#pragma unroll 8
            for (int r = 0; r < 32; ++r) a += (double)Ds[sw_f(r, j >> 2) + (j & 3)];
            e.part[prow * e.ldp + col + j] = a;
          }
        } else if (col + j < N) {
          for (int qq = lane >> 4; qq < e.R; qq += 2) {
            double a = 0.0;
#pragma unroll 8
            for (int r = 0; r < 32; ++r) a += ws[qq * 32 + r] * (double)Ds[sw_f(r, j >> 2) + (j & 3)];
            e.part[qq * e.plane + prow * e.ldp + col + j] = a;
          }
        }
        if (e.U0) {
          // u itself for the deferred (exact-CVaR) sums: TMA-stored from the
          // staging tile; the refill below targets the previous chunk's slot,
          // whose u store must have read it first
          if (lane == 0) tcx::bulk_wait_read0();
          __syncwarp();
          issue();
          tcx::fence_proxy_async();
          __syncwarp();
          if (lane == 0) {
            tcx::tma_store_2d(&om.m[1], Ds, col, (int)r0);
            tcx::bulk_commit();
          }
        } else {
          // this slot's generic reads before the async refill of the previous one
          tcx::fence_proxy_async();
          __syncwarp();
          issue();
        }
      } else {
        const TcChain<EpiBwd>& ch = ep;
        const bool has_G = ch.base.G != nullptr, has_split = ch.split.hi != nullptr;
#pragma unroll
        for (int j = 0; j < 16; ++j) dd[j] *= g[j];
        if (lane == 0) tcx::bulk_wait_read0();   // previous chunk's stores have read their slot
        __syncwarp();
        issue();
        if (has_G) row_put(Rs, lane, g);
        uint32_t* sh = reinterpret_cast<uint32_t*>(Ds);
        if (has_split) row_put_split(sh, sh + 256, lane, dd);
        tcx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if (has_G) tcx::tma_store_2d(&om.m[0], Rs, col, (int)r0);
          if (has_split) {
            tcx::tma_store_3d(&om.m[2], sh, col, (int)r0, 0);           // hi, lo (+1 KB)
          }
          tcx::bulk_commit();
        }
      }
    }
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
  if (lane == 0) tcx::bulk_wait0();
}

template <class Epi>
struct RingKind {
  static constexpr bool BWD = false;
};
template <>
struct RingKind<TcChain<EpiBwd>> {
  static constexpr bool BWD = true;
};
template <>
struct RingKind<EpiBwdSum> {
  static constexpr bool BWD = true;
};

// CG = 2: CTA pairs (cluster of two, cta_group::2 MMAs on 256-row tiles;
// ring epilogues only).  CG = 1: one CTA per 128-row tile.
template <int BN, class Epi, int RING = 0, int CG = 1>
__global__ void __launch_bounds__((EpiWarps<RING, RingKind<Epi>::BWD>::THREADS), 1)
tc_gemm_kernel(const __grid_constant__ CUtensorMap tA, const __grid_constant__ CUtensorMap tB, int64_t M,
               const int* __restrict__ Mdev, int N, int K, Epi epi, const __grid_constant__ TcOutMaps om,
               int use_om, unsigned long long* __restrict__ trace = nullptr, TcFlags flags = TcFlags{}) {
  static_assert(CG == 1 || (CG == 2 && RING > 0), "CTA pairs run the ring epilogues only");
  using C = TcCfg<BN, RING, RingKind<Epi>::BWD, CG>;
  constexpr int BMT = TC_BM * CG;                // rows per tile
  constexpr int STAGES = C::STAGES;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment by offset arithmetic keeps the pointer in the shared window
  uint8_t* smem = smem_raw + ((1024u - (tcx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * C::STAGE_BYTES + C::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar = tempty + 2;                   // RING slots per epilogue warp
  constexpr int EW = EpiWarps<RING, RingKind<Epi>::BWD>::EW;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar + (RING ? RING * EW : 0));

  // warp index through a shuffle: provably warp-uniform, so role branches and
  // the TMA / mbarrier operands stay in uniform registers
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = CG == 1 ? 0 : (int)tcx::cluster_rank();
  if (threadIdx.x == 0) {
    tcx::prefetch_tmap(&tA);
    tcx::prefetch_tmap(&tB);
    for (int s = 0; s < STAGES; ++s) { tcx::mbar_init(&full[s], 1); tcx::mbar_init(&empty[s], 1); }
    // (pairs: the leader's tempty counts the epilogue warps of both CTAs)
    for (int a = 0; a < 2; ++a) { tcx::mbar_init(&tfull[a], 1); tcx::mbar_init(&tempty[a], CG * EW); }
    for (int i = 0; i < RING * EW; ++i) tcx::mbar_init(&rbar[i], 1);
    tcx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      tcx::tmem_alloc(tmem_slot, 2 * BN);
      tcx::tmem_relinquish();
    } else {
      tcx::tmem_alloc_pair(tmem_slot, 2 * BN);
      tcx::tmem_relinquish_pair();
    }
  }
  tcx::fence_before();
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();                      // peer barriers initialised before any remote arrive
  tcx::fence_after();
  const uint32_t tmem = *tmem_slot;
  // programmatic dependent launch: the prologue above (barriers, TMEM,
  // descriptor prefetch) overlaps the previous grid's tail; every global
  // access (operands, epilogue inputs and outputs, *Mdev) comes after it
  if (!flags.in) asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;");
  if (Mdev) M = min(M, (int64_t)*Mdev);
  const int m_tiles = (int)((M + BMT - 1) / BMT);
  const TileWalk tw{(int)blockIdx.x / CG, (int)gridDim.x / CG, rank * TC_BM};
  const int n_tiles = (N + BN - 1) / BN;
  const int num_tiles = m_tiles * n_tiles;
  const int kblocks = (K + TC_BK - 1) / TC_BK;

  if (warp == 0) {
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      const bool skip_loads = (g_tc_dbg_skip & 2) != 0;
      if (trace && blockIdx.x == 0) trace[0] = clock64();
      for (int tile = tw.t0; tile < num_tiles; tile += tw.ts) {
        const int mb = tile / n_tiles, nb = tile % n_tiles;
        const int arow = mb * BMT + tw.row_off;  // this CTA's 128 rows of A
        if (flags.in) {                          // this row block of A written and visible
          const int need = TC_BM * K;
          while (tcx::ld_acquire(flags.in + arow / TC_BM) < need) __nanosleep(64);
          tcx::fence_proxy_async_global();
        }
        for (int kb = 0; kb < kblocks; ++kb) {
          tcx::mbar_wait(&empty[stage], phase ^ 1);
          if (trace && blockIdx.x == 0 && tile == (int)blockIdx.x && kb < 4) trace[1 + kb] = clock64();
          uint8_t* st = smem + stage * C::STAGE_BYTES;
          if (skip_loads) {
            tcx::mbar_arrive(&full[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
            continue;
          }
          // A hi + lo, then B hi + lo: one 3-D TMA load each (pair maps)
          if constexpr (CG == 1) {
            tcx::mbar_expect_tx(&full[stage], C::STAGE_BYTES);
            tcx::tma_load_3d(st, &tA, &full[stage], kb * TC_BK, arow, 0);
            tcx::tma_load_3d(st + 2 * C::A_BYTES, &tB, &full[stage], kb * TC_BK, nb * BN, 0);
          } else {                               // both CTAs' bytes complete on the leader's barrier
            if (rank == 0) tcx::mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
            tcx::tma_load_3d_pair(st, &tA, &full[stage], kb * TC_BK, arow, 0);
            tcx::tma_load_3d_pair(st + 2 * C::A_BYTES, &tB, &full[stage], kb * TC_BK, nb * BN + rank * (BN / 2), 0);
          }
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) {                // (pairs: the leader issues for both CTAs)
      constexpr uint32_t idesc = tcx::idesc_bf16(BMT, BN);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      const bool skip_mma = (g_tc_dbg_skip & 1) != 0;
      for (int tile = tw.t0; tile < num_tiles; tile += tw.ts) {
        tcx::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tcx::fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < kblocks; ++kb) {
          tcx::mbar_wait(&full[stage], phase);
          tcx::fence_after();
          const uint32_t base = tcx::smem_u32(smem + stage * C::STAGE_BYTES);
#pragma unroll
          for (int kk = 0; kk < (skip_mma ? 0 : TC_BK / 16); ++kk) {
            const uint64_t ah = tcx::sdesc_k64(base + kk * 32);
            const uint64_t al = tcx::sdesc_k64(base + C::A_BYTES + kk * 32);
            const uint64_t bh = tcx::sdesc_k64(base + 2 * C::A_BYTES + kk * 32);
            const uint64_t bl = tcx::sdesc_k64(base + 2 * C::A_BYTES + C::B_BYTES + kk * 32);
            if constexpr (CG == 1) {
              tcx::mma_bf16(d, ah, bh, idesc, (kb | kk) != 0);
              if (!flags.hi_only) {
                tcx::mma_bf16(d, ah, bl, idesc, 1);
                tcx::mma_bf16(d, al, bh, idesc, 1);
              }
            } else {
              tcx::mma_bf16_pair(d, ah, bh, idesc, (kb | kk) != 0);
              tcx::mma_bf16_pair(d, ah, bl, idesc, 1);
              tcx::mma_bf16_pair(d, al, bh, idesc, 1);
            }
          }
          // frees the smem slot (both CTAs' for pairs) when these MMAs finish
          if constexpr (CG == 1) tcx::commit(&empty[stage]);
          else tcx::commit_pair(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        if (trace && blockIdx.x == 0 && tile == (int)blockIdx.x) trace[5] = clock64();
        // accumulator ready for the epilogue (both CTAs' for pairs)
        if constexpr (CG == 1) tcx::commit(&tfull[acc]);
        else tcx::commit_pair(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp >= 4) {
    // (compile-time split: a ring kernel carries no register-prefetch epilogue code)
    if constexpr (RING > 0 && RingKind<Epi>::BWD) {
      epi_bwd_ring<BN, RING, CG>(epi, om, smem + STAGES * C::STAGE_BYTES, rbar, tfull, tempty, tmem, warp, lane,
                                 num_tiles, n_tiles, M, N, tw);
    } else if constexpr (RING > 0) {
      epi_fwd_ring<BN, RING, CG>(epi, om, smem + STAGES * C::STAGE_BYTES, rbar, tfull, tempty, tmem, warp, lane,
                                 num_tiles, n_tiles, N, K, flags, tw);
    } else {
    const int q = warp & 3;                      // TMEM lane quarter of this warp
    const int third = (warp - 4) >> 2;           // which 16-column chunks (mod 3)
    uint8_t* ep = smem + STAGES * C::STAGE_BYTES + (warp - 4) * TC_EPI_WARP_BYTES;
    const EpiSmem es{reinterpret_cast<float*>(ep), reinterpret_cast<float*>(ep + 2048),
                     reinterpret_cast<uint32_t*>(ep + 4096), reinterpret_cast<uint32_t*>(ep + 5120),
                     use_om ? &om : nullptr};
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mb = tile / n_tiles, nb = tile % n_tiles;
      tcx::mbar_wait(&tfull[acc], acc_phase);
      tcx::fence_after();
      const TileRows tr{(int64_t)mb * TC_BM + q * 32, M, nullptr};
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
      const bool tr0 = trace && blockIdx.x == 0 && warp == 4 && lane == 0 && tile == (int)blockIdx.x;
      if (tr0) trace[8] = clock64();
      typename TileEpi<Epi>::Pre cur;
      if (nb * BN + 16 * third < N) TileEpi<Epi>::load(epi, tr, nb * BN + 16 * third, N, lane, cur);
      int ci = 0;
#pragma unroll 1
      for (int c0 = 16 * third; c0 < BN; c0 += 48, ++ci) {
        if (nb * BN + c0 >= N) break;            // warp-uniform
        typename TileEpi<Epi>::Pre nxt;          // prefetch the next chunk's inputs
        if (c0 + 48 < BN && nb * BN + c0 + 48 < N) TileEpi<Epi>::load(epi, tr, nb * BN + c0 + 48, N, lane, nxt);
        uint32_t v[16];
        tcx::tmem_ld16(tbase + c0, v);
        tcx::tmem_ld_wait();
        if (tr0 && ci < 10) trace[9 + 2 * ci] = clock64();
        TileEpi<Epi>::chunk(epi, es, tr, nb * BN + c0, N, lane, v, cur);
        if (tr0 && ci < 10) trace[10 + 2 * ci] = clock64();
        cur = nxt;
      }
      tcx::fence_before();
      __syncwarp();
      if (lane == 0) tcx::mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (flags.out) {                           // publish this warp's part of the row block
        if (!use_om) __threadfence();            // thread stores of all lanes
        __syncwarp();
        if (lane == 0) {
          int cols = 0;
          for (int c0 = 16 * third; c0 < BN && nb * BN + c0 < N; c0 += 48) cols += 16;
          if (use_om) tcx::bulk_wait0();         // this warp's TMA stores complete
          tcx::fence_proxy_async_global();
          tcx::red_release_add(flags.out + mb, 32 * cols);
        }
      }
    }
    if (use_om && lane == 0) tcx::bulk_wait0();    // this warp's TMA stores are complete
    }
  }
  // (pairs: neither CTA leaves while the other may still arrive on its
  // barriers or the leader's MMAs may still write its TMEM)
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();
  if (warp == 2) {
    tcx::fence_after();
    if constexpr (CG == 1) tcx::tmem_dealloc(tmem, 2 * BN);
    else tcx::tmem_dealloc_pair(tmem, 2 * BN);
  }
}

// ---------------------------------------------------------------------------
// Persistent forward chain: the hidden layers of the MLP forward in ONE
// launch.  The CTA walks a global tile list (layer-major; tile g of layer
// g / tpl) with the per-layer row-block flags as the only dependency: a
// layer-l tile starts once the layer-(l-1) rows it reads are published, so a
// layer's wave tail overlaps the next layer's first tiles on the same SM (the
// accumulator double buffer lets tile g+1's MMAs run under tile g's
// epilogue), and the prologue (barriers, TMEM) is paid once.  Buffer reuse is
// safe: layer l+1 writes the ping-pong split that layer l read, but only on
// rows whose layer-l outputs -- hence all layer-l reads of them -- are complete.
// The epilogue prefetches residual tiles only within its current tile (never
// across a flag wait that could depend on the tile it has not yet published).
constexpr int SDN_CHAIN_MAX = 8;
// study switch (SDN_CHAIN_TRACE=1, non-graph runs): per CTA and tile,
// %globaltimer stamps {producer waits, producer starts, MMA starts, MMA done,
// epilogue (warp 4) starts, epilogue published}, 32 tiles per CTA
constexpr int CHAIN_TR_TILES = 32;
__device__ unsigned long long* g_chain_trace = nullptr;
SDN_DEV void chain_stamp(int tile_i, int k) {
  if (g_chain_trace && tile_i < CHAIN_TR_TILES) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_chain_trace[((size_t)blockIdx.x * CHAIN_TR_TILES + tile_i) * 8 + k] = t;
  }
}
struct FwdChainLayer {
  const float* bias;
  const int* fin;      // readiness of this layer's input rows (null: ready at launch)
  int* fout;           // this layer's row-block flags (null: not published)
  int K, has_prev, has_D, has_split;
  int N, nt;           // output width, column tiles
  int boff;            // this layer's bias offset in the shared-memory copy
  // kind 1: the output layer -- phi = shift + scale (acc + bias) stored fp32
  // (dmap) and the reverse sweep's unit seeds a2 phi + b2 as a split (smap)
  int kind;
  const float* scale;
  const float* shift;
  const float* a2;
  const float* b2;
};
struct FwdChainArgs {
  int L, N, n_tiles, m_tiles, act, bias_smem;
  int lstart[SDN_CHAIN_MAX + 1];                           // first global tile of each layer


  int64_t M;
  FwdChainLayer ly[SDN_CHAIN_MAX];
  CUtensorMap a[SDN_CHAIN_MAX], b[SDN_CHAIN_MAX];          // mainloop operands
  CUtensorMap dmap[SDN_CHAIN_MAX], smap[SDN_CHAIN_MAX];    // D, split outputs
  CUtensorMap pmap[SDN_CHAIN_MAX];                         // residual input (split of the layer input)
};

// the chain kernels' producer (TMA) and MMA-issuer loops over the global
// tile list (identical for the forward and the reverse chain; Args holds the
// per-layer operand maps a[l], b[l], K and input flags fin)
// global tile g -> (layer, 256-row tile, column tile); layers may differ in width
template <class Args>
SDN_DEV void chain_tile(const Args& ca, int g, int& l, int& mbt, int& nb) {
  l = 0;
  while (l + 1 < ca.L && g >= ca.lstart[l + 1]) ++l;
  const int t = g - ca.lstart[l], nt = ca.ly[l].nt;
  mbt = t / nt;
  nb = t - mbt * nt;
}

// K-major operand descriptor for a stage of BK columns: 64-byte (BK = 32) or 128-byte (BK = 64) swizzle rows
template <int BK>
SDN_DEV uint64_t sdesc_bk(uint32_t saddr) {
  if constexpr (BK == 64) return tcx::sdesc_k128(saddr);
  else return tcx::sdesc_k64(saddr);
}
template <int BN, int CG, int STAGES, class C, class Args>
SDN_DEV void chain_produce(const Args& ca, uint8_t* smem, uint64_t* full, uint64_t* empty, int rank, int t0, int ts,
                           int tpl, int total, int n_tiles) {
  int stage = 0;
  uint32_t phase = 0;
  for (int g = t0, ti = 0; g < total; g += ts, ++ti) {
    int l, mbt, nb;
    chain_tile(ca, g, l, mbt, nb);
    const int mb = mbt * CG + rank;          // this CTA's 128-row block
    const auto& ly = ca.ly[l];
    chain_stamp(ti, 0);
    if (ly.fin) {                            // input rows of this layer written and visible
      while (tcx::ld_acquire(ly.fin + mb) < TC_BM * ly.K) __nanosleep(64);
      tcx::fence_proxy_async_global();
    }
    chain_stamp(ti, 1);
    const int kblocks = (ly.K + C::BK_ - 1) / C::BK_;
    for (int kb = 0; kb < kblocks; ++kb) {
      tcx::mbar_wait(&empty[stage], phase ^ 1);
      uint8_t* st = smem + stage * C::STAGE_BYTES;
      if constexpr (CG == 1) {
        tcx::mbar_expect_tx(&full[stage], C::STAGE_BYTES);
        tcx::tma_load_3d(st, &ca.a[l], &full[stage], kb * C::BK_, mb * TC_BM, 0);
        tcx::tma_load_3d(st + 2 * C::A_BYTES, &ca.b[l], &full[stage], kb * C::BK_, nb * BN, 0);
      } else {
        if (rank == 0) tcx::mbar_expect_tx(&full[stage], 2 * C::STAGE_BYTES);
        tcx::tma_load_3d_pair(st, &ca.a[l], &full[stage], kb * C::BK_, mb * TC_BM, 0);
        tcx::tma_load_3d_pair(st + 2 * C::A_BYTES, &ca.b[l], &full[stage], kb * C::BK_, nb * BN + rank * (BN / 2), 0);
      }
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
  }
}
template <int BN, int CG, int STAGES, class C, class Args>
SDN_DEV void chain_mma(const Args& ca, uint8_t* smem, uint64_t* full, uint64_t* empty, uint64_t* tfull,
                       uint64_t* tempty, uint32_t tmem, int t0, int ts, int tpl, int total) {
  constexpr int BMT = TC_BM * CG;
  constexpr uint32_t idesc = tcx::idesc_bf16(BMT, BN);
  int stage = 0, acc = 0;
  uint32_t phase = 0, acc_phase = 0;
  for (int g = t0, ti = 0; g < total; g += ts, ++ti) {
    int l, mbt, nb;
    chain_tile(ca, g, l, mbt, nb);
    const int kblocks = (ca.ly[l].K + C::BK_ - 1) / C::BK_;
    tcx::mbar_wait(&tempty[acc], acc_phase ^ 1);
    tcx::fence_after();
    chain_stamp(ti, 2);
    const uint32_t d = tmem + acc * BN;
    for (int kb = 0; kb < kblocks; ++kb) {
      tcx::mbar_wait(&full[stage], phase);
      tcx::fence_after();
      const uint32_t base = tcx::smem_u32(smem + stage * C::STAGE_BYTES);
#pragma unroll
      for (int kk = 0; kk < C::BK_ / 16; ++kk) {
        const uint64_t ah = sdesc_bk<C::BK_>(base + kk * 32);
        const uint64_t al = sdesc_bk<C::BK_>(base + C::A_BYTES + kk * 32);
        const uint64_t bh = sdesc_bk<C::BK_>(base + 2 * C::A_BYTES + kk * 32);
        const uint64_t bl = sdesc_bk<C::BK_>(base + 2 * C::A_BYTES + C::B_BYTES + kk * 32);
        if constexpr (CG == 1) {
          tcx::mma_bf16(d, ah, bh, idesc, (kb | kk) != 0);
          tcx::mma_bf16(d, ah, bl, idesc, 1);
          tcx::mma_bf16(d, al, bh, idesc, 1);
        } else {
          tcx::mma_bf16_pair(d, ah, bh, idesc, (kb | kk) != 0);
          tcx::mma_bf16_pair(d, ah, bl, idesc, 1);
          tcx::mma_bf16_pair(d, al, bh, idesc, 1);
        }
      }
      if constexpr (CG == 1) tcx::commit(&empty[stage]);
      else tcx::commit_pair(&empty[stage]);
      if (++stage == STAGES) { stage = 0; phase ^= 1; }
    }
    if constexpr (CG == 1) tcx::commit(&tfull[acc]);
    else tcx::commit_pair(&tfull[acc]);
    chain_stamp(ti, 3);
    if (++acc == 2) { acc = 0; acc_phase ^= 1; }
  }
}

// the chain kernels' publisher (warp 3, one thread): the gpu-scope release of
// a row block's flag costs MEMBAR.ALL.GPU + CCTL.IVALL (~10% of an epilogue
// warp's time when each warp published its own part,
// profiles/r02g_fwd_chain_stalls.txt).  The epilogue warps instead count
// "my stores of tile i are complete" on a CTA-local shared counter
// (release.cta after cp.async.bulk.wait_group + the proxy fence), and this
// otherwise idle thread turns EW counts into one red.release.gpu on the flag.
// Four rotating counters: a warp can run at most two tiles ahead of another
// (the accumulator double buffer), so tile i never shares a counter with a
// tile still in flight.
template <int BN, int CG, int EW, class Args>
SDN_DEV void chain_publish(const Args& ca, uint32_t* pubc, int rank, int t0, int ts, int total) {
  uint64_t want = 0;                               // 4 x 16-bit expected counts (no local array)
  int ti = 0;
  for (int g = t0; g < total; g += ts, ++ti) {
    int l, mbt, nb;
    chain_tile(ca, g, l, mbt, nb);
    const auto& ly = ca.ly[l];
    if (!ly.fout) continue;
    const int sh = 16 * (ti & 3);
    want += (uint64_t)EW << sh;
    const uint32_t need = (uint32_t)(want >> sh) & 0xFFFFu;
    int nchunks = 0;                               // 16-column chunks of this tile, all column groups
    for (int c = 0; c < BN && nb * BN + c < ly.N; c += 16) ++nchunks;
    while (tcx::ld_acquire_cta_smem(&pubc[ti & 3]) < need) __nanosleep(32);
    tcx::red_release_add(ly.fout + (mbt * CG + rank), TC_BM * 16 * nchunks);
  }
}

// shared-memory plan of the chain kernel: STAGES mainloop stages, EW
// epilogue warps with RING 2-KB slots + a 2-KB D tile each, every layer's bias
template <int BN, int RING, int CG, int EW, int BK = TC_BK>
struct ChainCfg {
  static_assert(EW % 4 == 0 && EW >= 4, "epilogue warps come in lane-quarter groups of four");
  using C = TcCfg<BN, RING, false, CG, BK>;
  static constexpr uint32_t WB = (uint32_t)RING * 2048u + 2048u;
  static constexpr uint32_t EPI_BYTES = EW * WB;
  static constexpr uint32_t BIAS_BYTES = 4096u + SDN_CHAIN_BIAS_BYTES;
  static constexpr int FIT = (int)((TC_SMEM_MAX - EPI_BYTES - BIAS_BYTES - 1024 - TC_BAR_BYTES) / C::STAGE_BYTES);
  static constexpr int STAGES = FIT > 4 ? 4 : FIT;
  static constexpr uint32_t SMEM = STAGES * C::STAGE_BYTES + EPI_BYTES + BIAS_BYTES + 1024 + TC_BAR_BYTES;
  static constexpr int THREADS = 32 * (4 + EW);
};

template <int BN, int RING, int CG, int EW, int BK = TC_BK>
__global__ void __launch_bounds__(ChainCfg<BN, RING, CG, EW, BK>::THREADS, 1)
tc_fwd_chain_kernel(const __grid_constant__ FwdChainArgs ca) {
  using CC = ChainCfg<BN, RING, CG, EW, BK>;
  using C = typename CC::C;
  constexpr int BMT = TC_BM * CG;
  constexpr int STAGES = CC::STAGES;
  constexpr int CS = 16 * (EW / 4);
  constexpr uint32_t WB = CC::WB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tcx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_base = smem + STAGES * C::STAGE_BYTES;
  // (the bias copies of every layer follow the epilogue slots when they fit)
  float* bias_all = reinterpret_cast<float*>(epi_base + EW * WB);
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_base + CC::EPI_BYTES + CC::BIAS_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar_all = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar_all + RING * EW);
  uint32_t* pubc = tmem_slot + 2;                 // 4 rotating tile-done counters (publisher hand-off)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = CG == 1 ? 0 : (int)tcx::cluster_rank();
  if (threadIdx.x == 0) {
    for (int l = 0; l < ca.L; ++l) {
      tcx::prefetch_tmap(&ca.a[l]);
      tcx::prefetch_tmap(&ca.b[l]);
    }
    for (int s2 = 0; s2 < STAGES; ++s2) { tcx::mbar_init(&full[s2], 1); tcx::mbar_init(&empty[s2], 1); }
    for (int a = 0; a < 2; ++a) { tcx::mbar_init(&tfull[a], 1); tcx::mbar_init(&tempty[a], CG * EW); }
    for (int i = 0; i < RING * EW; ++i) tcx::mbar_init(&rbar_all[i], 1);
    for (int i = 0; i < 4; ++i) pubc[i] = 0;
    tcx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      tcx::tmem_alloc(tmem_slot, 2 * BN);
      tcx::tmem_relinquish();
    } else {
      tcx::tmem_alloc_pair(tmem_slot, 2 * BN);
      tcx::tmem_relinquish_pair();
    }
  }
  tcx::fence_before();
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();
  tcx::fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");      // inputs of the first layer (MR split, z-bias)
  asm volatile("griddepcontrol.launch_dependents;");
  // (pairs: m_tiles counts 256-row tiles; the CTA of rank r owns rows 128 r .. 128 r + 127 of each)
  const int n_tiles = ca.n_tiles, tpl = ca.m_tiles * n_tiles, total = ca.lstart[ca.L];
  const int t0 = (int)blockIdx.x / CG, ts = (int)gridDim.x / CG;

  if (warp == 0) {
    if (lane == 0) chain_produce<BN, CG, STAGES, C>(ca, smem, full, empty, rank, t0, ts, tpl, total, n_tiles);
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) chain_mma<BN, CG, STAGES, C>(ca, smem, full, empty, tfull, tempty, tmem, t0, ts, tpl, total);
  } else if (warp == 3) {
    if (lane == 0) chain_publish<BN, CG, EW>(ca, pubc, rank, t0, ts, total);
  } else if (warp >= 4) {
    const int w = warp - 4, q = warp & 3;
    uint8_t* wb = epi_base + w * WB;
    int ti = 0;
    float* Dst = reinterpret_cast<float*>(wb + RING * 2048);
    uint64_t* rbar = rbar_all + w * RING;
    if (ca.bias_smem)
      for (int l = 0; l < ca.L; ++l)
        for (int i = (int)threadIdx.x - 128; i < ca.ly[l].N; i += 32 * EW)
          bias_all[ca.ly[l].boff + i] = __ldg(ca.ly[l].bias + i);
    asm volatile("bar.sync 1, %0;" ::"n"(32 * EW) : "memory");
    int acc = 0, jt = 0;                          // jt: chunks before this tile (ring slot of chunk ci = (jt + ci) % RING)
    uint32_t acc_phase = 0, rphase = 0;          // rphase: parity bit per ring slot
    for (int g = t0; g < total; g += ts) {
      int l, mbt, nb;
      chain_tile(ca, g, l, mbt, nb);
      const int mbl = mbt * CG + rank;            // this CTA's 128-row block
      const FwdChainLayer& ly = ca.ly[l];
      const int N = ly.N;
      const bool has_prev = ly.has_prev, has_split = ly.has_split, has_D = ly.has_D, outl = ly.kind == 1;
      const int r0 = mbl * TC_BM + q * 32;
      // the warp's column group rotates with the tile: a 256-column tile is 16
      // chunks, i.e. 6 + 5 + 5 over three groups -- rotating evens the warps out
      // over consecutive tiles (they only meet at the accumulator hand-back)
      const int first_c = 16 * (((w >> 2) + ti) % (EW / 4));
      int nch = 0;
      for (int c = first_c; c < BN && nb * BN + c < N; c += CS) ++nch;
      // this tile's residual tiles, RING-1 chunks ahead (within the tile)
      if (has_prev && lane == 0 && nch > 0 && ly.fin) {
        while (tcx::ld_acquire(ly.fin + mbl) < TC_BM * ly.K) __nanosleep(64);
        tcx::fence_proxy_async_global();
      }
      auto issue = [&](int ci) {
        if (has_prev && ci < nch && lane == 0) {
          const int s2 = (jt + ci) % RING;
          tcx::mbar_expect_tx(&rbar[s2], 2048);
          tcx::tma_load_3d(wb + s2 * 2048, &ca.pmap[l], &rbar[s2], nb * BN + first_c + CS * ci, r0, 0);
        }
      };
      for (int k = 0; k < RING - 1; ++k) issue(k);
      tcx::mbar_wait(&tfull[acc], acc_phase);
      tcx::fence_after();
      if (warp == 4 && lane == 0) chain_stamp(ti, 4);
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (nch == 0) {
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) tmem_release<CG>(&tempty[acc]);
      }
      const float* bias_l = ca.bias_smem ? bias_all + ly.boff : nullptr;
#pragma unroll 1
      for (int ci = 0; ci < nch; ++ci) {
        const int c0 = first_c + CS * ci, col = nb * BN + c0, s2 = (jt + ci) % RING;
        uint32_t* sh = reinterpret_cast<uint32_t*>(wb + s2 * 2048);
        uint32_t* sl = sh + 256;
        uint32_t v[16];
        tcx::tmem_ld16(tbase + c0, v);
        if (has_prev) {
          tcx::mbar_wait(&rbar[s2], (rphase >> s2) & 1u);
          rphase ^= 1u << s2;
        }
        tcx::tmem_ld_wait();
        if (ci == nch - 1) {
          tcx::fence_before();
          __syncwarp();
          if (lane == 0) tmem_release<CG>(&tempty[acc]);
        }
        float a[16], d[16], bias[16];
        if (has_prev) row_get_split(sh, sl, lane, a);
#pragma unroll
        for (int j = 0; j < 16; j += 4) {
          const float4 b4 = bias_l ? *reinterpret_cast<const float4*>(bias_l + col + j)
                                   : __ldg(reinterpret_cast<const float4*>(ly.bias + col + j));
          bias[j] = b4.x; bias[j + 1] = b4.y; bias[j + 2] = b4.z; bias[j + 3] = b4.w;
        }
        if (outl) {                               // phi = shift + scale (acc + b) -> d; seeds a2 phi + b2 -> a
#pragma unroll
          for (int j = 0; j < 16; j += 4) {
            const float4 sc = __ldg(reinterpret_cast<const float4*>(ly.scale + col + j));
            const float4 sf = __ldg(reinterpret_cast<const float4*>(ly.shift + col + j));
            const float4 aa = __ldg(reinterpret_cast<const float4*>(ly.a2 + col + j));
            const float4 bb = __ldg(reinterpret_cast<const float4*>(ly.b2 + col + j));
            const float scs[4] = {sc.x, sc.y, sc.z, sc.w}, sfs[4] = {sf.x, sf.y, sf.z, sf.w};
            const float as[4] = {aa.x, aa.y, aa.z, aa.w}, bs[4] = {bb.x, bb.y, bb.z, bb.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
              d[j + k] = fmaf(scs[k], __uint_as_float(v[j + k]) + bias[j + k], sfs[k]);
              a[j + k] = fmaf(as[k], d[j + k], bs[k]);
            }
          }
        } else {
          fwd_act16(ca.act, v, bias, has_prev, a, d);
        }
        if (lane == 0) tcx::bulk_wait_read0();   // previous chunk's stores have read their staging
        __syncwarp();
        issue(ci + RING - 1);
        if (has_D) row_put(Dst, lane, d);
        if (has_split) row_put_split(sh, sl, lane, a);
        tcx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if (has_D) tcx::tma_store_2d(&ca.dmap[l], Dst, col, r0);
          if (has_split) tcx::tma_store_3d(&ca.smap[l], sh, col, r0, 0);
          tcx::bulk_commit();
        }
      }
      jt += nch;
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (ly.fout) {                              // this warp's part of the row block is written: tell the publisher
        __syncwarp();
        if (lane == 0) {
          tcx::bulk_wait0();
          tcx::fence_proxy_async_global();
          tcx::red_release_cta_smem(&pubc[ti & 3], 1u);
        }
      }
      if (warp == 4 && lane == 0) chain_stamp(ti, 5);
      ++ti;
    }
    if (lane == 0) tcx::bulk_wait0();
  }
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();
  if (warp == 2) {
    tcx::fence_after();
    if constexpr (CG == 1) tcx::tmem_dealloc(tmem, 2 * BN);
    else tcx::tmem_dealloc_pair(tmem, 2 * BN);
  }
}

// Persistent reverse chain: the dense sweep's chain steps (every reverse
// GEMM but the last, summing one) in ONE launch, the forward chain's scheme
// with the reverse ring epilogue: per chunk the residual gradient G and the
// act' tile are TMA-loaded RING-1 chunks ahead into one 4-KB slot, g = acc
// [+ G], u = D g, G written back in place (same rows, same columns: the tile
// that reads a G element is the one that rewrites it) and u's split stored
// as the next step's A operand.  Layer l-1 overwrites the split that layer l
// read only on rows whose layer-l outputs are published (row-block flags).
struct BwdChainLayer {
  const int* fin;
  int* fout;
  int K, has_resid, has_G;
  int N, nt;
};
struct BwdChainArgs {
  int L, N, n_tiles, m_tiles;
  int lstart[SDN_CHAIN_MAX + 1];
  int64_t M;
  BwdChainLayer ly[SDN_CHAIN_MAX];
  CUtensorMap a[SDN_CHAIN_MAX], b[SDN_CHAIN_MAX];          // mainloop operands
  CUtensorMap rmap[SDN_CHAIN_MAX], dmap[SDN_CHAIN_MAX];    // residual gradient, act' inputs
  CUtensorMap gmap[SDN_CHAIN_MAX], smap[SDN_CHAIN_MAX];    // G and split(u) outputs
};
template <int BN, int RING, int CG, int EW, int BK = TC_BK>
struct BwdChainCfg {
  static_assert(EW % 4 == 0 && EW >= 4, "epilogue warps come in lane-quarter groups of four");
  using C = TcCfg<BN, RING, true, CG, BK>;
  static constexpr uint32_t WB = (uint32_t)RING * 4096u;
  static constexpr uint32_t EPI_BYTES = EW * WB;
  static constexpr int FIT = (int)((TC_SMEM_MAX - EPI_BYTES - 1024 - TC_BAR_BYTES) / C::STAGE_BYTES);
  static constexpr int STAGES = FIT > 4 ? 4 : FIT;
  static constexpr uint32_t SMEM = STAGES * C::STAGE_BYTES + EPI_BYTES + 1024 + TC_BAR_BYTES;
  static constexpr int THREADS = 32 * (4 + EW);
};

template <int BN, int RING, int CG, int EW, int BK = TC_BK>
__global__ void __launch_bounds__(BwdChainCfg<BN, RING, CG, EW, BK>::THREADS, 1)
tc_bwd_chain_kernel(const __grid_constant__ BwdChainArgs ca) {
  using CC = BwdChainCfg<BN, RING, CG, EW, BK>;
  using C = typename CC::C;
  constexpr int STAGES = CC::STAGES;
  constexpr int CS = 16 * (EW / 4);
  constexpr uint32_t WB = CC::WB;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (tcx::smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* epi_base = smem + STAGES * C::STAGE_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(epi_base + CC::EPI_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rbar_all = tempty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rbar_all + RING * EW);
  uint32_t* pubc = tmem_slot + 2;                 // 4 rotating tile-done counters (publisher hand-off)
  const int warp = __shfl_sync(0xffffffffu, (int)(threadIdx.x >> 5), 0), lane = threadIdx.x & 31;
  const int rank = CG == 1 ? 0 : (int)tcx::cluster_rank();
  if (threadIdx.x == 0) {
    for (int l = 0; l < ca.L; ++l) {
      tcx::prefetch_tmap(&ca.a[l]);
      tcx::prefetch_tmap(&ca.b[l]);
    }
    for (int s2 = 0; s2 < STAGES; ++s2) { tcx::mbar_init(&full[s2], 1); tcx::mbar_init(&empty[s2], 1); }
    for (int a = 0; a < 2; ++a) { tcx::mbar_init(&tfull[a], 1); tcx::mbar_init(&tempty[a], CG * EW); }
    for (int i = 0; i < RING * EW; ++i) tcx::mbar_init(&rbar_all[i], 1);
    for (int i = 0; i < 4; ++i) pubc[i] = 0;
    tcx::fence_barrier_init();
  }
  if (warp == 2) {
    if constexpr (CG == 1) {
      tcx::tmem_alloc(tmem_slot, 2 * BN);
      tcx::tmem_relinquish();
    } else {
      tcx::tmem_alloc_pair(tmem_slot, 2 * BN);
      tcx::tmem_relinquish_pair();
    }
  }
  tcx::fence_before();
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();
  tcx::fence_after();
  const uint32_t tmem = *tmem_slot;
  asm volatile("griddepcontrol.wait;" ::: "memory");      // the seeds' split (forward output layer)
  asm volatile("griddepcontrol.launch_dependents;");
  const int n_tiles = ca.n_tiles, tpl = ca.m_tiles * n_tiles, total = ca.lstart[ca.L];
  const int t0 = (int)blockIdx.x / CG, ts = (int)gridDim.x / CG;

  if (warp == 0) {
    if (lane == 0) chain_produce<BN, CG, STAGES, C>(ca, smem, full, empty, rank, t0, ts, tpl, total, n_tiles);
  } else if (warp == 1) {
    if (lane == 0 && rank == 0) chain_mma<BN, CG, STAGES, C>(ca, smem, full, empty, tfull, tempty, tmem, t0, ts, tpl, total);
  } else if (warp == 3) {
    if (lane == 0) chain_publish<BN, CG, EW>(ca, pubc, rank, t0, ts, total);
  } else if (warp >= 4) {
    const int w = warp - 4, q = warp & 3, first_c = 16 * (w >> 2);
    uint8_t* wb = epi_base + w * WB;
    uint64_t* rbar = rbar_all + w * RING;
    int acc = 0, jt = 0, ti = 0;
    uint32_t acc_phase = 0, rphase = 0;
    for (int g = t0; g < total; g += ts, ++ti) {
      int l, mbt, nb;
      chain_tile(ca, g, l, mbt, nb);
      const int mbl = mbt * CG + rank;
      const BwdChainLayer& ly = ca.ly[l];
      const int N = ly.N;
      const bool has_resid = ly.has_resid, has_G = ly.has_G;
      const int r0 = mbl * TC_BM + q * 32;
      int nch = 0;
      for (int c = first_c; c < BN && nb * BN + c < N; c += CS) ++nch;
      if (lane == 0 && nch > 0 && ly.fin) {       // this step's inputs (G rows) published
        while (tcx::ld_acquire(ly.fin + mbl) < TC_BM * ly.K) __nanosleep(64);
        tcx::fence_proxy_async_global();
      }
      auto issue = [&](int ci) {
        if (ci < nch && lane == 0) {
          const int s2 = (jt + ci) % RING;
          const int x = nb * BN + first_c + CS * ci;
          tcx::mbar_expect_tx(&rbar[s2], has_resid ? 4096u : 2048u);
          if (has_resid) tcx::tma_load_2d(wb + s2 * 4096, &ca.rmap[l], &rbar[s2], x, r0);
          tcx::tma_load_2d(wb + s2 * 4096 + 2048, &ca.dmap[l], &rbar[s2], x, r0);
        }
      };
      for (int k = 0; k < RING - 1; ++k) issue(k);
      tcx::mbar_wait(&tfull[acc], acc_phase);
      tcx::fence_after();
      const uint32_t tbase = tmem + ((uint32_t)(q * 32) << 16) + acc * BN;
      if (nch == 0) {
        tcx::fence_before();
        __syncwarp();
        if (lane == 0) tmem_release<CG>(&tempty[acc]);
      }
#pragma unroll 1
      for (int ci = 0; ci < nch; ++ci) {
        const int c0 = first_c + CS * ci, col = nb * BN + c0, s2 = (jt + ci) % RING;
        float* Rs = reinterpret_cast<float*>(wb + s2 * 4096);
        float* Ds = Rs + 512;
        uint32_t v[16];
        tcx::tmem_ld16(tbase + c0, v);
        tcx::mbar_wait(&rbar[s2], (rphase >> s2) & 1u);
        rphase ^= 1u << s2;
        tcx::tmem_ld_wait();
        if (ci == nch - 1) {
          tcx::fence_before();
          __syncwarp();
          if (lane == 0) tmem_release<CG>(&tempty[acc]);
        }
        float gv[16], dd[16];
#pragma unroll
        for (int j = 0; j < 16; ++j) gv[j] = __uint_as_float(v[j]);
        if (has_resid) {
          float r[16];
          row_get(Rs, lane, r);
#pragma unroll
          for (int j = 0; j < 16; ++j) gv[j] += r[j];
        }
        row_get(Ds, lane, dd);
#pragma unroll
        for (int j = 0; j < 16; ++j) dd[j] *= gv[j];
        if (lane == 0) tcx::bulk_wait_read0();   // previous chunk's stores have read their slot
        __syncwarp();
        issue(ci + RING - 1);
        if (has_G) row_put(Rs, lane, gv);
        uint32_t* sh = reinterpret_cast<uint32_t*>(Ds);
        row_put_split(sh, sh + 256, lane, dd);
        tcx::fence_proxy_async();
        __syncwarp();
        if (lane == 0) {
          if (has_G) tcx::tma_store_2d(&ca.gmap[l], Rs, col, r0);
          tcx::tma_store_3d(&ca.smap[l], sh, col, r0, 0);      // hi, lo (+1 KB)
          tcx::bulk_commit();
        }
      }
      jt += nch;
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      if (ly.fout) {                              // this warp's stores of the tile are complete: tell the publisher
        __syncwarp();
        if (lane == 0) {
          tcx::bulk_wait0();
          tcx::fence_proxy_async_global();
          tcx::red_release_cta_smem(&pubc[ti & 3], 1u);
        }
      }
    }
    if (lane == 0) tcx::bulk_wait0();
  }
  if constexpr (CG == 1) __syncthreads();
  else tcx::cluster_sync();
  if (warp == 2) {
    tcx::fence_after();
    if constexpr (CG == 1) tcx::tmem_dealloc(tmem, 2 * BN);
    else tcx::tmem_dealloc_pair(tmem, 2 * BN);
  }
}

// ---------------------------------------------------------------------------
// host side

static PFN_cuTensorMapEncodeTiled_v12000 tc_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 3-D bf16 pair map over a split operand: (cols x rows x {hi, lo}) with row
// pitch ld elements and lo at a fixed offset from hi; box = 32 x box_rows x 2
// (64 B swizzle): one TMA load brings a k-block's hi and lo tiles
static int tc_map(TcWeights& t, const TcOperand& op, int64_t rows, int cols, int box_rows, CUtensorMap* out,
                  int bk = TC_BK) {
  const __nv_bfloat16* base = op.hi;
  const int ld = op.ld;
  const int64_t pair = (int64_t)((const char*)op.lo - (const char*)op.hi);
  auto key = std::make_tuple((const void*)base, rows, cols * 65536 + box_rows + (bk == TC_BK ? 0 : 32768), (int)ld);
  auto it = t.maps.find(key);
  if (it != t.maps.end()) { *out = it->second; return 0; }
  auto fn = tc_encode_fn();
  if (!fn) return -1;
  if (pair <= 0 || pair % 16) return -4;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)rows, 2};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)pair};
  cuuint32_t box[3] = {(cuuint32_t)bk, (cuuint32_t)box_rows, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(base), dims, strides, box,
                  estr, CU_TENSOR_MAP_INTERLEAVE_NONE, bk == 64 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -2;
  t.maps[key] = m;
  *out = m;
  return 0;
}

// output map for the TMA-store epilogue: (rows x cols) of fp32 or bf16 with
// row pitch ld; box = 32 rows x 16 columns, swizzle matching the staging
// layout (sw_f = 64B for fp32 rows of 64 B, sw_h = 32B for bf16 rows of 32 B)
static int tc_out_map(TcWeights& t, const void* base, bool bf16, int64_t rows, int cols, int64_t ld,
                      CUtensorMap* out) {
  auto key = std::make_tuple(base, rows, (int64_t)cols * 2 + (bf16 ? 1 : 0), ld);
  auto it = t.omaps.find(key);
  if (it != t.omaps.end()) { *out = it->second; return 0; }
  auto fn = tc_encode_fn();
  if (!fn) return -1;
  const int es = bf16 ? 2 : 4;
  if (((uintptr_t)base & 15) || (ld * es) % 16) return -2;
  CUtensorMap m;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)std::max<int64_t>(rows, 1)};
  cuuint64_t strides[1] = {(cuuint64_t)ld * es};
  cuuint32_t box[2] = {16, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(&m, bf16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                  const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  bf16 ? CU_TENSOR_MAP_SWIZZLE_32B : CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -3;
  t.omaps[key] = m;
  *out = m;
  return 0;
}

// epilogue pair map of a split operand (hi, lo at a fixed offset): box
// 16 columns x 32 rows x 2, 32 B swizzle (the sw_h staging of hi, then lo +1 KB)
static int tc_out_map_pair(TcWeights& t, const __nv_bfloat16* hi, const __nv_bfloat16* lo, int64_t rows, int cols,
                           int64_t ld, CUtensorMap* out) {
  const int64_t pair = (int64_t)((const char*)lo - (const char*)hi);
  auto key = std::make_tuple((const void*)hi, rows, (int64_t)cols * 2 + 1 + (pair << 20), ld + (1ll << 40));
  auto it = t.omaps.find(key);
  if (it != t.omaps.end()) { *out = it->second; return 0; }
  auto fn = tc_encode_fn();
  if (!fn) return -1;
  if (((uintptr_t)hi & 15) || (ld * 2) % 16 || pair <= 0 || pair % 16) return -2;
  CUtensorMap m;
  cuuint64_t dims[3] = {(cuuint64_t)cols, (cuuint64_t)std::max<int64_t>(rows, 1), 2};
  cuuint64_t strides[2] = {(cuuint64_t)ld * 2, (cuuint64_t)pair};
  cuuint32_t box[3] = {16, 32, 2};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<__nv_bfloat16*>(hi), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return -3;
  t.omaps[key] = m;
  *out = m;
  return 0;
}

// which epilogues store through TMA, and their output maps (slot order as in
// TcOutMaps); returns bit 1 when every output got a map, bit 2 when the
// ring epilogue's input maps (m[4], m[5]) were built too
template <class Epi>
struct EpiOut {
  static int build(TcWeights&, const Epi&, int64_t, int, TcOutMaps&) { return 0; }
};
template <>
struct EpiOut<EpiAffine> {
  static int build(TcWeights& t, const EpiAffine& e, int64_t M, int N, TcOutMaps& om) {
    return tc_out_map(t, e.C, false, M, N, e.ldc, &om.m[0]) == 0 ? 1 : 0;
  }
};
template <>
struct EpiOut<EpiAffineSeed> {
  static int build(TcWeights& t, const EpiAffineSeed& e, int64_t M, int N, TcOutMaps& om) {
    if (tc_out_map(t, e.base.C, false, M, N, e.base.ldc, &om.m[0])) return 0;
    if (tc_out_map_pair(t, e.seed.hi, e.seed.lo, M, N, e.seed.ld, &om.m[2])) return 0;
    return 1;
  }
};
template <>
struct EpiOut<TcChain<EpiFwdHidden>> {
  static int build(TcWeights& t, const TcChain<EpiFwdHidden>& ch, int64_t M, int N, TcOutMaps& om) {
    const EpiFwdHidden& e = ch.base;
    if (e.H && tc_out_map(t, e.H, false, M, N, e.ld, &om.m[0])) return 0;
    if (e.D && tc_out_map(t, e.D, false, M, N, e.ld, &om.m[1])) return 0;
    if (ch.split.hi && tc_out_map_pair(t, ch.split.hi, ch.split.lo, M, N, ch.split.ld, &om.m[2])) return 0;
    // residual input tiles for the ring epilogue (same 32 x 16 boxes, loaded): bit 2
    if (ch.prev.hi && tc_out_map_pair(t, ch.prev.hi, ch.prev.lo, M, N, ch.prev.ld, &om.m[4])) return 1;
    return 3;
  }
};
template <>
struct EpiOut<TcChain<EpiBwd>> {
  static int build(TcWeights& t, const TcChain<EpiBwd>& ch, int64_t M, int N, TcOutMaps& om) {
    const EpiBwd& e = ch.base;
    if (e.G && tc_out_map(t, e.G, false, M, N, e.ld, &om.m[0])) return 0;
    if (e.U && tc_out_map(t, e.U, false, M, N, e.ld, &om.m[1])) return 0;
    if (ch.split.hi && tc_out_map_pair(t, ch.split.hi, ch.split.lo, M, N, ch.split.ld, &om.m[2])) return 0;
    // ring-epilogue input tiles (dense sweeps only: no row gather): bit 2
    if (e.rowidx || !e.D) return 1;
    if (e.resid && tc_out_map(t, e.resid, false, M, N, e.ld, &om.m[4])) return 1;
    if (tc_out_map(t, e.D, false, M, N, e.ldD, &om.m[5])) return 1;
    return 3;
  }
};
template <>
struct EpiOut<TcChain<EpiTanTc>> {
  static int build(TcWeights& t, const TcChain<EpiTanTc>& ch, int64_t M, int N, TcOutMaps& om) {
    return tc_out_map_pair(t, ch.split.hi, ch.split.lo, M, N, ch.split.ld, &om.m[2]) == 0 ? 1 : 0;
  }
};
template <>
struct EpiOut<EpiScaleSplit> {
  static int build(TcWeights& t, const EpiScaleSplit& e, int64_t M, int N, TcOutMaps& om) {
    return tc_out_map_pair(t, e.split.hi, e.split.lo, M, N, e.split.ld, &om.m[2]) == 0 ? 1 : 0;
  }
};
// the summing reverse step stores nothing through TMA: its maps are the
// ring-epilogue inputs only (bit 2)
template <>
struct EpiOut<EpiBwdSum> {
  static int build(TcWeights& t, const EpiBwdSum& e, int64_t M, int N, TcOutMaps& om) {
    if (e.rowidx || !e.D) return 0;
    if (e.resid && tc_out_map(t, e.resid, false, M, N, e.ld, &om.m[4])) return 0;
    if (tc_out_map(t, e.D, false, M, N, e.ldD, &om.m[5])) return 0;
    if (e.U0 && tc_out_map(t, e.U0, false, M, N, e.ld, &om.m[1])) return 0;
    return 2;
  }
};

inline bool tc_gemm_supported(int64_t M, int N, int K) {
  return M >= 1 && K >= 8 && K % 8 == 0 && N >= 16 && N % 16 == 0 && tc_encode_fn() != nullptr;
}

// ring epilogue depth for the forward chain (0 = register-prefetch epilogue);
// SDN_EPI_RING=0/2/3 overrides
static int g_tc_ring = getenv("SDN_EPI_RING") ? atoi(getenv("SDN_EPI_RING")) : 2;

template <class Epi>
struct RingOk {
  static bool ok(const Epi&, int) { return false; }
};
template <>
struct RingOk<TcChain<EpiFwdHidden>> {
  static bool ok(const TcChain<EpiFwdHidden>& ch, int) { return !ch.base.H && !ch.base.prev; }
};
template <>
struct RingOk<TcChain<EpiBwd>> {
  static bool ok(const TcChain<EpiBwd>& ch, int) { return !ch.base.rowidx && ch.base.D && !ch.base.U; }
};
template <>
struct RingOk<EpiBwdSum> {
  static bool ok(const EpiBwdSum& e, int) { return !e.rowidx && e.D; }
};
// reverse-sweep ring depth (0 = register-prefetch epilogue); SDN_BWD_RING overrides.
// 3 on the 128-column reverse tiles: with 8 epilogue warps (TC_RING_EW_BWD) depths 2
// and 3 both keep four mainloop stages; depth 3 wins on the epilogue's prefetch
// distance (reverse GEMMs 0.185 -> 0.171 ms per c2 step)
static int g_tc_bwd_ring = getenv("SDN_BWD_RING") ? atoi(getenv("SDN_BWD_RING")) : 3;

template <int BN, class Epi, int RING, int CG = 1>
static int tc_launch_k(cudaStream_t st, int grid, int64_t M, const int* Mdev, int N, int K, const CUtensorMap& am,
                       const CUtensorMap& bm, const Epi& epi, const TcOutMaps& om, int use_om, TcFlags fl) {
  using C = TcCfg<BN, RING, RingKind<Epi>::BWD, CG>;
  static_assert(C::STAGES >= 2 && C::SMEM <= TC_SMEM_MAX, "shared memory budget");
  static unsigned attr_set = 0;                    // per device: the attribute is a per-context setting
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set & (1u << (dev & 31)))) {
    cudaFuncSetAttribute(tc_gemm_kernel<BN, Epi, RING, CG>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)C::SMEM);
    attr_set |= 1u << (dev & 31);
  }
  // programmatic stream serialization (PDL): the kernel may start while the
  // previous one drains; griddepcontrol.wait orders it
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(EpiWarps<RING, RingKind<Epi>::BWD>::THREADS);
  cfg.dynamicSmemBytes = C::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (g_tc_pdl && g_tc_pdl_now) ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;   // CTA pairs on one TPC
  attr[1].val.clusterDim.x = CG;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CG > 1 ? 2 : 1;
  if (!(g_tc_pdl && g_tc_pdl_now)) fl.in = nullptr;   // row flags only pay off with early (PDL) launch
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_gemm_kernel<BN, Epi, RING, CG>, am, bm, M, Mdev, N, K, epi, om,
                                           use_om, g_tc_trace, fl);
  return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? 0 : -3;
}

// CTA pairs (cta_group::2, 256-row tiles) for the ring GEMMs with a host-
// known row count: each SM then loads half of every weight k-block.  Measured
// neutral at c2 (forward 182.7 vs 180.9, reverse 168.7 vs 172.2 us per step:
// the epilogue, not the mainloop's L2 traffic, paces these GEMMs), so off by
// default; SDN_TC_PAIRS=1 enables them
static bool g_tc_pairs = getenv("SDN_TC_PAIRS") && getenv("SDN_TC_PAIRS")[0] == '1';

template <int BN, class Epi>
static int tc_launch_pairs(TcWeights& t, cudaStream_t st, int num_sms, int64_t M, int N, int K, const TcOperand& A,
                           const TcOperand& B, const Epi& epi, const TcOutMaps& om, int use_om, TcFlags fl) {
  constexpr bool BWD = RingKind<Epi>::BWD;
  constexpr int RING_BWD = 3;
  CUtensorMap am, bm;
  if (tc_map(t, A, std::max<int64_t>(M, 1), K, TC_BM, &am) || tc_map(t, B, N, K, BN / 2, &bm)) return -1;
  const int64_t tiles = ((M + 2 * TC_BM - 1) / (2 * TC_BM)) * ((N + BN - 1) / BN);
  const int grid = 2 * (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms / 2));
  if constexpr (BWD) {
    if constexpr (TcCfg<BN, RING_BWD, true, 2>::STAGES_FIT >= 2)
      return tc_launch_k<BN, Epi, RING_BWD, 2>(st, grid, M, nullptr, N, K, am, bm, epi, om, use_om, fl);
    return -5;
  } else {
    return tc_launch_k<BN, Epi, 2, 2>(st, grid, M, nullptr, N, K, am, bm, epi, om, use_om, fl);
  }
}

template <int BN, class Epi>
static int tc_launch(TcWeights& t, cudaStream_t st, int num_sms, int64_t M, const int* Mdev, int N, int K,
                     const TcOperand& A, const TcOperand& B, Epi epi, TcFlags fl = TcFlags{}) {
  TcOutMaps om;
  memset(&om, 0, sizeof(om));
  const int ob = g_tc_thread_stores ? 0 : EpiOut<Epi>::build(t, epi, std::max<int64_t>(M, 1), N, om);
  const int use_om = ob & 1;
  if constexpr (BN == 256 && (std::is_same<Epi, TcChain<EpiFwdHidden>>::value || RingKind<Epi>::BWD)) {
    const bool ring = std::is_same<Epi, TcChain<EpiFwdHidden>>::value ? g_tc_ring > 0 : g_tc_bwd_ring > 0;
    if (g_tc_pairs && !Mdev && (ob & 2) && ring && !g_tc_trace && RingOk<Epi>::ok(epi, N) && num_sms >= 2)
      return tc_launch_pairs<BN>(t, st, num_sms, M, N, K, A, B, epi, om, use_om, fl);
  }
  CUtensorMap am, bm;
  if (tc_map(t, A, std::max<int64_t>(M, 1), K, TC_BM, &am) || tc_map(t, B, N, K, BN, &bm)) return -1;
  const int64_t tiles = ((M + TC_BM - 1) / TC_BM) * ((N + BN - 1) / BN);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(tiles, num_sms));
  if constexpr (std::is_same<Epi, TcChain<EpiFwdHidden>>::value) {
    if ((ob & 2) && g_tc_ring > 0 && !g_tc_trace && RingOk<Epi>::ok(epi, N)) {
      if constexpr (TcCfg<BN, 3, false>::STAGES_FIT >= 2)
        if (g_tc_ring == 3) return tc_launch_k<BN, Epi, 3>(st, grid, M, Mdev, N, K, am, bm, epi, om, use_om, fl);
      return tc_launch_k<BN, Epi, 2>(st, grid, M, Mdev, N, K, am, bm, epi, om, use_om, fl);
    }
  }
  if constexpr (RingKind<Epi>::BWD) {
    if ((ob & 2) && !Mdev && g_tc_bwd_ring > 0 && !g_tc_trace && RingOk<Epi>::ok(epi, N)) {
      if constexpr (TcCfg<BN, 3, true>::STAGES_FIT >= 2)
        if (g_tc_bwd_ring == 3) return tc_launch_k<BN, Epi, 3>(st, grid, M, Mdev, N, K, am, bm, epi, om, use_om, fl);
      return tc_launch_k<BN, Epi, 2>(st, grid, M, Mdev, N, K, am, bm, epi, om, use_om, fl);
    }
  }
  return tc_launch_k<BN, Epi, 0>(st, grid, M, Mdev, N, K, am, bm, epi, om, use_om, fl);
}


template <class Epi>
static int tc_gemm(TcWeights& t, cudaStream_t st, int num_sms, int64_t M, const int* Mdev, int N, int K,
                   const TcOperand& A, const TcOperand& B, Epi epi, int64_t rows_est = -1, TcFlags fl = TcFlags{}) {
  // widest N tile that still gives every SM work; narrower tiles for the
  // short compacted sweeps (CVaR tails) and small shards
  const int64_t mt = ((rows_est > 0 ? rows_est : M) + TC_BM - 1) / TC_BM;
  static const int bn_force = getenv("SDN_TC_BN") ? atoi(getenv("SDN_TC_BN")) : 0;   // tuning override
  if (bn_force == 64) return tc_launch<64>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
  if (bn_force == 128) return tc_launch<128>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
  // dense reverse-sweep ring GEMMs: 128-column tiles leave the mainloop four
  // stages next to the 4-KB-slot epilogue ring (256: two); measured faster at c2
  if constexpr (RingKind<Epi>::BWD)
    if (!Mdev && !bn_force && N > 128 && mt * ((N + 127) / 128) >= num_sms && g_tc_bwd_ring > 0 && !g_tc_pairs)
      return tc_launch<128>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
  if (N > 128 && mt * ((N + 255) / 256) >= num_sms / 2)
    return tc_launch<256>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
  if (N > 64 && mt * ((N + 127) / 128) >= num_sms / 4)
    return tc_launch<128>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
  return tc_launch<64>(t, st, num_sms, M, Mdev, N, K, A, B, epi, fl);
}

// persistent forward chain launch (see tc_fwd_chain_kernel).  Layer l reads
// A[l] and writes its split to S[l] (the next layer's A) and act' to D[l];
// P[l] (may be null) is its residual input.  Returns 0 on launch.
// CTA (pair) slots of a persistent chain.  Slot c walks the layer-major tile
// list with stride S; a layer-(l+1) tile depends on the layer-l tiles of its
// rows, T = tiles per layer earlier in the list, i.e. T/S rounds back.  With
// T >= 2 S every dependency was published at least two rounds ago, so a tile's
// MMAs always run under the previous tile's epilogue.  With T < 2 S the slots
// c >= T - S depend on tiles of the round just before theirs: their MMAs cannot
// start until that round's epilogues are done, every round -- the c2 forward
// chain on 74 pair slots (T = 128) ran 7 rounds of epilogue + exposed MMA
// (122 us) where 64 slots run 8 rounds of epilogue alone.  Cost model:
// epilogue 2, exposed MMA 1 per round (SDN_CHAIN_SLOTS=n overrides).
static int chain_slots(int slots_max, int T, int total) {
  static const int forced = getenv("SDN_CHAIN_SLOTS") ? atoi(getenv("SDN_CHAIN_SLOTS")) : 0;
  if (forced > 0) return std::min(forced, slots_max);
  const int alt = T / 2;
  if (alt < 1 || alt >= slots_max) return slots_max;
  auto cost = [&](int S) { return ((total + S - 1) / S) * (2 + (T < 2 * S ? 1 : 0)) + 1; };
  return cost(alt) < cost(slots_max) ? alt : slots_max;
}

struct FwdChainLayerHost {
  const TcOperand* A;
  const TcOperand* B;
  const TcOperand* S;
  const TcOperand* P;
  float* D;
  const float* bias;
  int K;
  TcFlags fl;
  int N = 0;           // 0: the chain's N
  int kind = 0;        // 1: output layer (phi to D, seeds to S)
  const float* scale = nullptr;
  const float* shift = nullptr;
  const float* a2 = nullptr;
  const float* b2 = nullptr;
};
static bool g_tc_chain = !(getenv("SDN_NO_CHAIN") && getenv("SDN_NO_CHAIN")[0] == '1');
template <int CG, int EW, int BK = TC_BK>
static int tc_fwd_chain_k(TcWeights& t, cudaStream_t st, int grid, int64_t M, int N, int act,
                          const std::vector<FwdChainLayerHost>& ls) {
  constexpr int BN = 256, RING = 2;
  using CC = ChainCfg<BN, RING, CG, EW, BK>;
  constexpr uint32_t SMEM = CC::SMEM;
  static_assert(CC::STAGES >= 2 && SMEM <= TC_SMEM_MAX, "chain shared memory budget");
  grid = CG * std::max(1, grid / CG);
  const int L = (int)ls.size();
  if (L < 1 || L > SDN_CHAIN_MAX || N % 16) return -1;
  FwdChainArgs ca;
  memset(&ca, 0, sizeof(ca));
  ca.L = L; ca.N = N; ca.M = M; ca.act = act;
  ca.n_tiles = (N + BN - 1) / BN;
  ca.m_tiles = (int)((M + TC_BM * CG - 1) / (TC_BM * CG));
  int boff = 0, tiles = 0;
  for (int l = 0; l < L; ++l) {
    const FwdChainLayerHost& x = ls[l];
    FwdChainLayer& y = ca.ly[l];
    const int Nl = x.N ? x.N : N;
    if (Nl % 16) return -1;
    if (tc_map(t, *x.A, std::max<int64_t>(M, 1), x.K, TC_BM, &ca.a[l], BK) ||
        tc_map(t, *x.B, Nl, x.K, BN / CG, &ca.b[l], BK))
      return -2;
    if (x.D && tc_out_map(t, x.D, false, M, Nl, Nl, &ca.dmap[l])) return -3;
    if (x.S && tc_out_map_pair(t, x.S->hi, x.S->lo, M, Nl, x.S->ld, &ca.smap[l])) return -3;
    if (x.P && tc_out_map_pair(t, x.P->hi, x.P->lo, M, Nl, x.P->ld, &ca.pmap[l])) return -3;
    y.bias = x.bias; y.K = x.K; y.fin = x.fl.in; y.fout = x.fl.out;
    y.has_prev = x.P != nullptr; y.has_D = x.D != nullptr; y.has_split = x.S != nullptr;
    y.N = Nl; y.nt = (Nl + BN - 1) / BN; y.boff = boff; boff += Nl;
    y.kind = x.kind; y.scale = x.scale; y.shift = x.shift; y.a2 = x.a2; y.b2 = x.b2;
    ca.lstart[l] = tiles;
    tiles += ca.m_tiles * y.nt;
  }
  ca.lstart[L] = tiles;
  ca.bias_smem = (uint32_t)boff * 4 <= CC::BIAS_BYTES ? 1 : 0;
  if (L > 1) {
    int T = tiles;
    for (int l = 0; l + 1 < L; ++l) T = std::min(T, ca.m_tiles * ca.ly[l].nt);
    grid = CG * chain_slots(grid / CG, T, tiles);
  }

  static unsigned attr_set = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set & (1u << (dev & 31)))) {
    cudaFuncSetAttribute(tc_fwd_chain_kernel<BN, RING, CG, EW, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)SMEM);
    attr_set |= 1u << (dev & 31);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CC::THREADS);
  cfg.dynamicSmemBytes = SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (g_tc_pdl && g_tc_pdl_now) ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CG;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CG > 1 ? 2 : 1;
  static const bool trace = getenv("SDN_CHAIN_TRACE") != nullptr;
  static unsigned long long* tbuf = nullptr;
  const size_t tn = (size_t)grid * CHAIN_TR_TILES * 8;
  if (trace) {
    if (!tbuf) cudaMalloc(&tbuf, sizeof(unsigned long long) * 148 * 2 * CHAIN_TR_TILES * 8);
    cudaMemsetAsync(tbuf, 0, sizeof(unsigned long long) * tn, st);
    cudaMemcpyToSymbolAsync(g_chain_trace, &tbuf, sizeof(tbuf), 0, cudaMemcpyHostToDevice, st);
  }
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_fwd_chain_kernel<BN, RING, CG, EW, BK>, ca);
  if (trace) {                                    // dump: grid, tiles per layer, then stamps
    std::vector<unsigned long long> hb(tn);
    cudaMemcpyAsync(hb.data(), tbuf, sizeof(unsigned long long) * tn, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    unsigned long long* z = nullptr;
    cudaMemcpyToSymbol(g_chain_trace, &z, sizeof(z));
    FILE* f = fopen(getenv("SDN_CHAIN_TRACE"), "ab");
    if (f) {
      const long long hdr[3] = {grid, (long long)ca.m_tiles * ca.n_tiles, L};
      fwrite(hdr, sizeof(hdr), 1, f);
      fwrite(hb.data(), sizeof(unsigned long long), tn, f);
      fclose(f);
    }
  }
  return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? 0 : -4;
}
// CTA pairs for the persistent chain (SDN_CHAIN_PAIRS=0 disables)
static bool g_chain_pairs = !(getenv("SDN_CHAIN_PAIRS") && getenv("SDN_CHAIN_PAIRS")[0] == '0');
// epilogue warps of the chain (SDN_CHAIN_EW=12 / 16): 12 measured faster at
// c2 (forward GEMMs 148 vs 153 us per step), though 16 split a 256-column tile
// into four chunks per warp exactly (12: five or six)
static int g_chain_ew = getenv("SDN_CHAIN_EW") ? atoi(getenv("SDN_CHAIN_EW")) : 12;
static int tc_fwd_chain(TcWeights& t, cudaStream_t st, int grid, int64_t M, int N, int act,
                        const std::vector<FwdChainLayerHost>& ls) {
  // 128-byte swizzle rows, 64 K columns per stage (two 64-KB stages instead of four 32-KB ones): the
  // forward chain's TMA row requests halve -- c2 0.3081 -> 0.3024 ms, c3 +1-2% (SDN_CHAIN_BK=32: the old
  // stages; the reverse chain measured slower with 64, SDN_BWD_CHAIN_BK=64)
  static const bool bk64 = !(getenv("SDN_CHAIN_BK") && atoi(getenv("SDN_CHAIN_BK")) == 32);
  if (g_chain_pairs && grid >= 2) {
    if (g_chain_ew == 12 && bk64) return tc_fwd_chain_k<2, 12, 64>(t, st, grid, M, N, act, ls);
    if (g_chain_ew == 12) return tc_fwd_chain_k<2, 12>(t, st, grid, M, N, act, ls);
    return tc_fwd_chain_k<2, 16>(t, st, grid, M, N, act, ls);
  }
  if (g_chain_ew == 16) return tc_fwd_chain_k<1, 16>(t, st, grid, M, N, act, ls);
  return tc_fwd_chain_k<1, 12>(t, st, grid, M, N, act, ls);
}

// persistent reverse chain launch (see tc_bwd_chain_kernel).  Step l reads
// A[l] (the previous step's split of u), the residual gradient R[l] (may be
// null) and act' D[l]; writes G[l] (may be null; in place of R) and split(u).
struct BwdChainLayerHost {
  const TcOperand* A;
  const TcOperand* B;
  const TcOperand* S;
  const float* R;
  float* G;
  const float* D;
  int64_t ldD;
  int K;
  TcFlags fl;
};
template <int CG, int BK = TC_BK>
static int tc_bwd_chain_k(TcWeights& t, cudaStream_t st, int grid, int64_t M, int N,
                          const std::vector<BwdChainLayerHost>& ls) {
  constexpr int BN = 256, RING = 3, EW = 8;
  using CC = BwdChainCfg<BN, RING, CG, EW, BK>;
  static_assert(CC::STAGES >= 2 && CC::SMEM <= TC_SMEM_MAX, "reverse chain shared memory budget");
  grid = CG * std::max(1, grid / CG);
  const int L = (int)ls.size();
  if (L < 1 || L > SDN_CHAIN_MAX || N % 16) return -1;
  BwdChainArgs ca;
  memset(&ca, 0, sizeof(ca));
  ca.L = L; ca.N = N; ca.M = M;
  ca.n_tiles = (N + BN - 1) / BN;
  ca.m_tiles = (int)((M + TC_BM * CG - 1) / (TC_BM * CG));
  for (int l = 0; l < L; ++l) {
    const BwdChainLayerHost& x = ls[l];
    BwdChainLayer& y = ca.ly[l];
    if (tc_map(t, *x.A, std::max<int64_t>(M, 1), x.K, TC_BM, &ca.a[l], BK) ||
        tc_map(t, *x.B, N, x.K, BN / CG, &ca.b[l], BK))
      return -2;
    if (x.R && tc_out_map(t, x.R, false, M, N, N, &ca.rmap[l])) return -3;
    if (tc_out_map(t, x.D, false, M, N, x.ldD, &ca.dmap[l])) return -3;
    if (x.G && tc_out_map(t, x.G, false, M, N, N, &ca.gmap[l])) return -3;
    if (tc_out_map_pair(t, x.S->hi, x.S->lo, M, N, x.S->ld, &ca.smap[l])) return -3;
    y.K = x.K; y.fin = x.fl.in; y.fout = x.fl.out;
    y.has_resid = x.R != nullptr; y.has_G = x.G != nullptr;
    y.N = N; y.nt = ca.n_tiles;
    ca.lstart[l] = l * ca.m_tiles * ca.n_tiles;
  }
  ca.lstart[L] = L * ca.m_tiles * ca.n_tiles;
  if (L > 1) grid = CG * chain_slots(grid / CG, ca.m_tiles * ca.n_tiles, ca.lstart[L]);
  static unsigned attr_set = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (!(attr_set & (1u << (dev & 31)))) {
    cudaFuncSetAttribute(tc_bwd_chain_kernel<BN, RING, CG, EW, BK>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)CC::SMEM);
    attr_set |= 1u << (dev & 31);
  }
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(CC::THREADS);
  cfg.dynamicSmemBytes = CC::SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = (g_tc_pdl && g_tc_pdl_now) ? 1 : 0;
  attr[1].id = cudaLaunchAttributeClusterDimension;
  attr[1].val.clusterDim.x = CG;
  attr[1].val.clusterDim.y = 1;
  attr[1].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = CG > 1 ? 2 : 1;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, tc_bwd_chain_kernel<BN, RING, CG, EW, BK>, ca);
  return (e == cudaSuccess && cudaGetLastError() == cudaSuccess) ? 0 : -4;
}
static bool g_bwd_chain = !(getenv("SDN_NO_BWD_CHAIN") && getenv("SDN_NO_BWD_CHAIN")[0] == '1');
static int tc_bwd_chain(TcWeights& t, cudaStream_t st, int grid, int64_t M, int N,
                        const std::vector<BwdChainLayerHost>& ls) {
  static const bool bk64 = getenv("SDN_BWD_CHAIN_BK") && atoi(getenv("SDN_BWD_CHAIN_BK")) == 64;   // study switch
  if (g_chain_pairs && grid >= 2 && bk64) return tc_bwd_chain_k<2, 64>(t, st, grid, M, N, ls);
  if (g_chain_pairs && grid >= 2) return tc_bwd_chain_k<2>(t, st, grid, M, N, ls);
  return tc_bwd_chain_k<1>(t, st, grid, M, N, ls);
}

// allocation / refresh of the split operands -------------------------------

template <class H>
static int tc_buf(H* h, TcWeights& t, TcOperand& op, int64_t rows, int ld) {
  op.rows = rows;
  op.ld = ld;
  size_t n = (size_t)std::max<int64_t>(rows, 1) * ld;
  // hi and lo in one allocation, lo at +n elements: the TMA pair maps move both
  // halves of a tile with one instruction
  if (cudaMalloc(&op.hi, n * 4) != cudaSuccess) return -1;
  op.lo = op.hi + n;
  cudaMemset(op.hi, 0, n * 4);
  t.allocs.push_back(op.hi);
  return 0;
}

template <class H>
static int tc_alloc(H* h, TcWeights& t) {
  t.enabled = false;
  if (!tc_encode_fn()) return 0;                       // no driver entry point: SIMT only
  int dev = 0, major = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  if (major != 10) return 0;                           // tcgen05 needs sm_100
  t.fwd.assign(h->L, TcOperand{});
  t.bwd.assign(h->L, TcOperand{});
  for (int l = 0; l < h->L; ++l) {
    const int n_in = (l == 0) ? h->r_m : h->w[l];
    if (tc_buf(h, t, t.fwd[l], h->w[l + 1], n_in)) return -1;
    if (l >= 1 && tc_buf(h, t, t.bwd[l], n_in, h->w[l + 1])) return -1;
  }
  for (int i = 0; i < 2; ++i)
    if (tc_buf(h, t, t.act[i], h->cap, h->maxw)) return -1;
  if (tc_buf(h, t, t.seed, h->cap, h->r_u)) return -1;
  if (tc_buf(h, t, t.mr, h->cap, h->r_m)) return -1;
  t.enabled = true;
  return 0;
}

static void tc_free(TcWeights& t) {
  for (void* p : t.allocs) cudaFree(p);
  t.allocs.clear();
  t.maps.clear();
  t.omaps.clear();
  t.enabled = false;
}

template <class H>
static int tc_set_weights(H* h, TcWeights& t) {
  for (int l = 0; l < h->L; ++l) {
    const int n_out = h->w[l + 1], n_in = (l == 0) ? h->r_m : h->w[l];
    k_split<<<256, 256, 0, h->stream>>>(n_out, nullptr, n_in, n_in, h->W[l], n_in, t.fwd[l].hi, t.fwd[l].lo);
    if (l >= 1) k_split_transpose<<<256, 256, 0, h->stream>>>(n_out, n_in, h->W[l], t.bwd[l].hi, t.bwd[l].lo);
  }
  return cudaStreamSynchronize(h->stream) == cudaSuccess ? 0 : -1;
}

template <class H>
static int tc_set_samples(H* h, TcWeights& t, const float* mr, int64_t n) {
  if (n > 0)
    k_split<<<(unsigned)std::min<int64_t>((n * h->r_m + 255) / 256, 4096), 256, 0, h->stream>>>(
        n, nullptr, h->r_m, h->r_m, mr, h->r_m, t.mr.hi, t.mr.lo);
  t.mr.rows = n;
  return cudaStreamSynchronize(h->stream) == cudaSuccess ? 0 : -1;
}

template <class H>
static int tc_split_seed(H* h, TcWeights& t, const float* E, int64_t nmax, const int* n_act_dev) {
  if (nmax > 0)
    k_split<<<(unsigned)std::min<int64_t>((nmax * h->r_u + 255) / 256, 8192), 256, 0, h->stream>>>(
        nmax, n_act_dev, h->r_u, h->r_u, E, h->r_u, t.seed.hi, t.seed.lo);
  return cudaGetLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace sdn
