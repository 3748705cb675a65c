// Plan executor for sm_100a: communicator (CUDA IPC peer maps + flag pages), lowering of a
// plan to per-rank device step tables, and the persistent step-table kernel.
//
// Hot path:
//   a1  entry flags — each CTA posts the call's epoch into its slot of every consumer's
//       flag page (st.release.sys over NVLink) and waits for its paired producers;
//   a2  ReduceScatter step — k-way pull reduction: k 16-byte loads per vector from local
//       HBM / peer HBM (NVLink, IPC-mapped), fp32 left-to-right sum in the plan's order
//       (reading Q1), one RNE rounding for bf16 (Q2);
//   a3  inter-step flags — full producer->consumer waits between dependent steps;
//   a4  AllGather — P2P 16-byte stores of the reduced vector; the last RS level is fused
//       with the first AG level so the owner writes its block straight from registers to
//       every destination (one read and one write per element, the δ saving of P:402);
//   a5  exit flags — paired waits on every rank that accessed this rank's buffer.
// The same kernel runs an emulated communicator (all ranks on one GPU) as one cooperative
// launch with blockIdx.y = rank.
#include <cuda.h>
#include <cuda_runtime.h>
#include <unistd.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <set>
#include <string>
#include <vector>

#include "../../include/gentree_ar.h"
#include "internal.hpp"

using namespace gtar;

namespace {

constexpr int kThreads = 512;
constexpr int kMaxSlots = 256;        // plan steps + entry (slot 0)
constexpr int kCtaCapMulti = 256;     // flag page CTA dimension, multi-process comms
constexpr uint32_t kBlobMagic = 0x47544152u;  // "GTAR"
constexpr int kTraceSteps = 64;       // steps traced per CTA
constexpr int kTraceSlots = 2 + 3 * kTraceSteps;

// ------------------------------------------------------------------ device tables
struct DevOp {
  long long off, len;        // elements
  int nsrc, ndst;
  int src_begin, dst_begin;  // into the rank list
  int fin;                   // 1 = the last RS op writing this region (AVG divides here)
  int pad;
};
struct DevStep {
  int slot;                  // flag slot written after this step (0 = entry)
  int op_begin, op_count;
  int wait_begin, wait_count;
  int notify_begin, notify_count;
  int pad;
};
constexpr int kWaitPaired = 0;   // wait for the producer's same-index CTA
constexpr int kWaitFull = 1;     // wait for every producer CTA
constexpr int kWaitRange = 2;    // wait for the producer CTAs whose slice of [p_off, p_len) meets ours of [c_off, c_len)
struct DevWait {
  int rank, slot, kind, pad;
  long long p_off, p_len;    // producer op range (elements)
  long long c_off, c_len;    // consumer op range (elements)
};
struct ExecArgs {
  const DevStep *steps;
  const DevOp *ops;
  const DevWait *waits;
  const int *ranks;          // op src/dst rank lists and notify lists
  const int *prog_begin;     // per local rank
  const int *prog_len;
  char *bufs[AR_MAX_RANKS];            // rank -> data buffer base (as seen here)
  unsigned long long *sigs[AR_MAX_RANKS];  // rank -> flag page base (as seen here)
  unsigned long long *err;
  unsigned long long *epoch_dev;   // last completed call's epoch (device-resident: graph-capturable)
  unsigned int *done_ctr;          // CTAs finished in the current call
  unsigned long long timeout_ns;
  int rank0, world, cta_cap, esize;
  int bulk;                  // 1 = cp.async.bulk-staged body, 0 = register body
  unsigned long long *trace; // optional globaltimer stamps (kTraceSlots per CTA), nullptr = off
  int fence_mode;            // notify ordering: 0 membar.sys/thread, 1 release.sys, 2 fence+relaxed, 3 gpu scope
  int store_tma;             // 1 = results leave through cp.async.bulk stores (body_bulk_st)
  int stages, stage_bytes;   // bulk-copy ring geometry
  unsigned int jitter_ns;    // stress mode: random delay before each notify (AR_JITTER_NS), 0 = off
  int avg_n;                 // AR_OP_AVG: divide final reduces by avg_n (IEEE fp32 division); 0 = SUM
  // push protocol (lower_push): rank -> its push scratch as seen here; [parity][src][slot]
  char *scr[AR_MAX_RANKS];
  long long scr_plane, scr_slot;
  // dynamic tile scheduling (CPS-shaped plans, one rank per process): op i's tiles are handed
  // out by atomicAdd on dyn_ctr[i]; the last CTA of the launch zeroes the dyn_nops counters
  unsigned int *dyn_ctr;     // nullptr = static per-CTA slices
  int dyn_nops;
  int entry_fence;           // 1 = fence.acq_rel.sys before the relaxed entry flags (AR_ENTRY_FENCE)
};

// Buffer references in op rank lists: r < kScrRef is rank r's data buffer; kScrRef + o·64 + s
// is the push scratch slot on owner o for source s (parity = the call's epoch & 1).
constexpr int kScrRef = 1 << 12;
__device__ __forceinline__ char *ref_base(const ExecArgs &a, int id, long long off, unsigned long long epoch) {
  if (id < kScrRef) return a.bufs[id];
  const int o = (id - kScrRef) / AR_MAX_RANKS, src = (id - kScrRef) % AR_MAX_RANKS;
  const long long ob = off * a.esize;   // slot keeps the buffer's 16-byte phase of element `off`
  return a.scr[o] + (long long)(epoch & 1ull) * a.scr_plane + (long long)src * a.scr_slot + (ob & 15) - ob;
}

// ------------------------------------------------------------------ PTX helpers
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ uint4 ld_cg(const uint4 *p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}
__device__ __forceinline__ void st_v4(uint4 *p, const uint4 &v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w)
               : "memory");
}

// bf16 <-> fp32.  Widening is exact; narrowing is round-to-nearest-even with NaN mapped to
// a quiet NaN that keeps the sign (reading Q2).
__device__ __forceinline__ float bf_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }
__device__ __forceinline__ uint32_t f2bf(float f) {
  uint32_t u = __float_as_uint(f);
  if ((u & 0x7FFFFFFFu) > 0x7F800000u) return 0x7FC0u | ((u >> 16) & 0x8000u);
  return (u + 0x7FFFu + ((u >> 16) & 1u)) >> 16;
}
// Two fp32 values to a bf16 pair (lo in the low half), round-to-nearest-even in one
// instruction: the same bits as f2bf for every non-NaN input (finite, subnormal, overflow to
// inf); a NaN becomes the canonical NaN (payload and sign are not part of the contract: Q2,
// the tests compare NaNs by isnan)
__device__ __forceinline__ uint32_t f2bf2(float lo, float hi) {
  uint32_t r;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
  return r;
}

// ------------------------------------------------------------------ reduction core
// Accumulate one 16-byte vector of source s into acc (fp32).  First source initialises.
template <bool BF16>
__device__ __forceinline__ void acc_first(float (&acc)[8], const uint4 &v) {
  if (BF16) {
    acc[0] = bf_lo(v.x); acc[1] = bf_hi(v.x); acc[2] = bf_lo(v.y); acc[3] = bf_hi(v.y);
    acc[4] = bf_lo(v.z); acc[5] = bf_hi(v.z); acc[6] = bf_lo(v.w); acc[7] = bf_hi(v.w);
  } else {
    acc[0] = __uint_as_float(v.x); acc[1] = __uint_as_float(v.y);
    acc[2] = __uint_as_float(v.z); acc[3] = __uint_as_float(v.w);
  }
}
template <bool BF16>
__device__ __forceinline__ void acc_add(float (&acc)[8], const uint4 &v) {
  if (BF16) {
    acc[0] = __fadd_rn(acc[0], bf_lo(v.x)); acc[1] = __fadd_rn(acc[1], bf_hi(v.x));
    acc[2] = __fadd_rn(acc[2], bf_lo(v.y)); acc[3] = __fadd_rn(acc[3], bf_hi(v.y));
    acc[4] = __fadd_rn(acc[4], bf_lo(v.z)); acc[5] = __fadd_rn(acc[5], bf_hi(v.z));
    acc[6] = __fadd_rn(acc[6], bf_lo(v.w)); acc[7] = __fadd_rn(acc[7], bf_hi(v.w));
  } else {
    acc[0] = __fadd_rn(acc[0], __uint_as_float(v.x)); acc[1] = __fadd_rn(acc[1], __uint_as_float(v.y));
    acc[2] = __fadd_rn(acc[2], __uint_as_float(v.z)); acc[3] = __fadd_rn(acc[3], __uint_as_float(v.w));
  }
}
template <bool BF16>
__device__ __forceinline__ uint4 acc_pack(const float (&acc)[8]) {
  uint4 o;
  if (BF16) {
    o.x = f2bf2(acc[0], acc[1]);
    o.y = f2bf2(acc[2], acc[3]);
    o.z = f2bf2(acc[4], acc[5]);
    o.w = f2bf2(acc[6], acc[7]);
  } else {
    o.x = __float_as_uint(acc[0]); o.y = __float_as_uint(acc[1]);
    o.z = __float_as_uint(acc[2]); o.w = __float_as_uint(acc[3]);
  }
  return o;
}

struct OpShared {
  const uint4 *src[AR_MAX_RANKS];
  uint4 *dst[AR_MAX_RANKS];
  int nsrc, ndst;
  int div;                   // > 0: this op's result is divided by div (AVG, reading AV1)
};

// AVG (reading AV1): the fp32 sum of a final reduce is divided by N with one correctly
// rounded IEEE division before the store's rounding.
__device__ __forceinline__ void acc_div(float (&acc)[8], float d) {
#pragma unroll
  for (int i = 0; i < 8; i++) acc[i] = __fdiv_rn(acc[i], d);
}

// Vector body, NSRC sources known at compile time (1 = copy).  UNROLL vectors per thread
// per iteration, all loads issued before any add (memory-level parallelism).
template <int NSRC, int UNROLL, bool BF16>
__device__ __noinline__ void body_fixed(const OpShared &s, size_t v0, size_t v1) {
  const size_t stride = (size_t)blockDim.x * UNROLL;
  const int ndst = s.ndst;
  for (size_t base = v0 + threadIdx.x; base < v1; base += stride) {
    uint4 x[UNROLL][NSRC];
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      size_t v = base + (size_t)u * blockDim.x;
      if (v < v1) {
#pragma unroll
        for (int k = 0; k < NSRC; k++) x[u][k] = ld_cg(s.src[k] + v);
      }
    }
#pragma unroll
    for (int u = 0; u < UNROLL; u++) {
      size_t v = base + (size_t)u * blockDim.x;
      if (v < v1) {
        uint4 o;
        if (NSRC == 1) {
          o = x[u][0];
        } else {
          float acc[8];
          acc_first<BF16>(acc, x[u][0]);
#pragma unroll
          for (int k = 1; k < NSRC; k++) acc_add<BF16>(acc, x[u][k]);
          if (s.div) acc_div(acc, (float)s.div);
          o = acc_pack<BF16>(acc);
        }
        for (int d = 0; d < ndst; d++) st_v4(s.dst[d] + v, o);
      }
    }
  }
}

// Any number of sources (> 8): groups of 8 loads, accumulation order unchanged.
template <bool BF16>
__device__ __noinline__ void body_generic(const OpShared &s, size_t v0, size_t v1) {
  for (size_t v = v0 + threadIdx.x; v < v1; v += blockDim.x) {
    float acc[8];
    for (int k0 = 0; k0 < s.nsrc; k0 += 8) {
      uint4 x[8];
      const int kn = min(8, s.nsrc - k0);
#pragma unroll
      for (int k = 0; k < 8; k++)
        if (k < kn) x[k] = ld_cg(s.src[k0 + k] + v);
#pragma unroll
      for (int k = 0; k < 8; k++) {
        if (k >= kn) break;
        if (k0 + k == 0) acc_first<BF16>(acc, x[k]);
        else acc_add<BF16>(acc, x[k]);
      }
    }
    if (s.div) acc_div(acc, (float)s.div);
    uint4 o = acc_pack<BF16>(acc);
    for (int d = 0; d < s.ndst; d++) st_v4(s.dst[d] + v, o);
  }
}

template <bool BF16>
__device__ void body_dispatch(const OpShared &s, size_t v0, size_t v1) {
  if (s.div && s.nsrc == 1) {
    body_generic<BF16>(s, v0, v1);
    return;
  }
  switch (s.nsrc) {
    case 1: body_fixed<1, 4, BF16>(s, v0, v1); break;
    case 2: body_fixed<2, 2, BF16>(s, v0, v1); break;
    case 3: body_fixed<3, 2, BF16>(s, v0, v1); break;
    case 4: body_fixed<4, 1, BF16>(s, v0, v1); break;
    case 5: body_fixed<5, 1, BF16>(s, v0, v1); break;
    case 6: body_fixed<6, 1, BF16>(s, v0, v1); break;
    case 7: body_fixed<7, 1, BF16>(s, v0, v1); break;
    case 8: body_fixed<8, 1, BF16>(s, v0, v1); break;
    default: body_generic<BF16>(s, v0, v1); break;
  }
}

// ------------------------------------------------------------------ bulk-staged body
// Warp-specialised pipeline: warp 0 (one lane) streams tiles of every source into shared
// memory with cp.async.bulk (the TMA bulk-copy engine; works on local and NVLink-peer
// addresses alike) completing on a per-stage mbarrier; warps 1.. wait, sum the NSRC tiles
// in plan order from shared memory and store the result to every destination, then release
// the stage.  kStages x kStageBytes of loads stay in flight per CTA without tying up
// registers — the memory-level parallelism the NVLink round trip (~2 us) needs.
constexpr int kMaxStages = 8;
constexpr int kDefStages = 4;
constexpr int kDefStageBytes = 40 * 1024;
constexpr int kMaxDynSmem = 224 * 1024;   // 227 KB per block minus the static shared state
// dynamic smem: stages x stage_bytes input ring + 2 output tiles of stage_bytes / 2
inline int dyn_smem_bytes(int stages, int stage_bytes) { return (stages + 1) * stage_bytes; }

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
// Bounded: a pipeline that never completes (a bug) must not hang the GPU — after ~20 s the
// wait gives up and raises the device error word (reported by ar_comm_get_async_error).
__device__ unsigned long long g_pipe_err = 0;
__device__ __forceinline__ void mbar_wait(unsigned long long *b, uint32_t parity) {
  uint32_t ok = 0;
  unsigned int spins = 0;
  unsigned long long t0 = 0;
  while (!ok) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(smem_u32(b)), "r"(parity)
        : "memory");
    if (!ok && (++spins & 4095u) == 0) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t0 == 0) t0 = t;
      else if (t - t0 > 20000000000ull) {
        atomicExch(&g_pipe_err, 2ull);
        return;
      }
    }
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst_smem, const void *src, uint32_t bytes, unsigned long long *bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst_smem)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct Pipe {
  unsigned long long full[kMaxStages];
  unsigned long long empty[kMaxStages];
  int stages, stage_bytes;   // runtime ring geometry (AR_STAGES, AR_STAGE_KB)
  uint32_t tile[kMaxStages]; // dynamic scheduling: the op tile in each stage (kNoTile = op done)
};
constexpr uint32_t kNoTile = 0xFFFFFFFFu;

template <int NSRC, bool BF16>
__device__ __noinline__ void body_bulk(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem,
                                       Pipe &pp) {
  const int kStages = pp.stages, kStageBytes = pp.stage_bytes;
  const int T = (kStageBytes / NSRC) / 16 * 16;   // bytes per source per tile
  const int TV = T / 16;                           // 16-byte vectors per source per tile
  const size_t nv = v1 - v0;
  const uint32_t ntiles = (uint32_t)((nv + TV - 1) / TV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < ntiles; i++) {
        const uint32_t gi = g + i, st = gi % kStages, use = gi / kStages;
        if (use > 0) mbar_wait(&pp.empty[st], (use - 1) & 1);
        const size_t t0 = v0 + (size_t)i * TV;
        const uint32_t bytes = (uint32_t)min((size_t)TV, v1 - t0) * 16;
        mbar_expect_tx(&pp.full[st], bytes * NSRC);
        uint8_t *base = smem + st * kStageBytes;
#pragma unroll
        for (int k = 0; k < NSRC; k++) bulk_g2s(base + k * T, s.src[k] + t0, bytes, &pp.full[st]);
      }
    }
  } else {
    const int ndst = s.ndst;
    const int nthr = blockDim.x - 32;
    for (uint32_t i = 0; i < ntiles; i++) {
      const uint32_t gi = g + i, st = gi % kStages, use = gi / kStages;
      mbar_wait(&pp.full[st], use & 1);
      const size_t t0 = v0 + (size_t)i * TV;
      const int nvt = (int)min((size_t)TV, v1 - t0);
      const uint4 *base = (const uint4 *)(smem + st * kStageBytes);
      for (int v = threadIdx.x - 32; v < nvt; v += nthr) {
        uint4 x[NSRC];
#pragma unroll
        for (int k = 0; k < NSRC; k++) x[k] = base[k * TV + v];
        uint4 o;
        if (NSRC == 1) {
          o = x[0];
        } else {
          float acc[8];
          acc_first<BF16>(acc, x[0]);
#pragma unroll
          for (int k = 1; k < NSRC; k++) acc_add<BF16>(acc, x[k]);
          if (s.div) acc_div(acc, (float)s.div);
          o = acc_pack<BF16>(acc);
        }
        for (int d = 0; d < ndst; d++) st_v4(s.dst[d] + t0 + v, o);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&pp.empty[st]);
    }
  }
  g += ntiles;
}

// Same pipeline, but the results go out through the bulk-copy engine as well: consumer warps
// sum into a shared-memory output tile and one thread issues cp.async.bulk stores of it to
// every destination (local and NVLink peers), so the SM issues 16-byte smem stores instead of
// ndst global stores per vector.  Two output tiles alternate; a copy op (NSRC = 1) stores
// straight from the input stage.  The stage's empty barrier has a single arrival (the storer).
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src_smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(src_smem)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void consumer_bar(int nthr) {
  asm volatile("bar.sync 1, %0;" ::"r"(nthr) : "memory");
}

template <int NSRC, bool BF16>
__device__ __noinline__ void body_bulk_st(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem,
                                          Pipe &pp) {
  const int kStages = pp.stages, kStageBytes = pp.stage_bytes, kOutTile = pp.stage_bytes / 2;
  const int T = (kStageBytes / NSRC) / 16 * 16;
  const int TV = T / 16;
  const size_t nv = v1 - v0;
  const uint32_t ntiles = (uint32_t)((nv + TV - 1) / TV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp == 0) {
    if (lane == 0) {
      for (uint32_t i = 0; i < ntiles; i++) {
        const uint32_t gi = g + i, st = gi % kStages, use = gi / kStages;
        if (use > 0) mbar_wait(&pp.empty[st], (use - 1) & 1);
        const size_t t0 = v0 + (size_t)i * TV;
        const uint32_t bytes = (uint32_t)min((size_t)TV, v1 - t0) * 16;
        mbar_expect_tx(&pp.full[st], bytes * NSRC);
        uint8_t *base = smem + st * kStageBytes;
#pragma unroll
        for (int k = 0; k < NSRC; k++) bulk_g2s(base + k * T, s.src[k] + t0, bytes, &pp.full[st]);
      }
    }
  } else {
    const int ndst = s.ndst;
    const int nthr = blockDim.x - 32;
    const bool storer = threadIdx.x == 32;
    uint4 *outb = (uint4 *)(smem + kStages * kStageBytes);   // 2 x kOutTile bytes
    // A copy (NSRC = 1) is done by the storer alone: the other threads must not wait on the
    // full barriers, since nothing would keep them within one phase of the storer (a thread
    // that falls two phases behind sees the parity flip twice and waits forever).
    for (uint32_t i = 0; i < ntiles && (NSRC > 1 || storer); i++) {
      const uint32_t gi = g + i, st = gi % kStages, use = gi / kStages;
      mbar_wait(&pp.full[st], use & 1);
      const size_t t0 = v0 + (size_t)i * TV;
      const int nvt = (int)min((size_t)TV, v1 - t0);
      const uint4 *base = (const uint4 *)(smem + st * kStageBytes);
      const void *src_tile = base;
      if (NSRC > 1) {
        uint4 *o = outb + (gi & 1) * (kOutTile / 16);
        consumer_bar(nthr);     // the storer has drained reads of this output tile (tile i-2)
        for (int v = threadIdx.x - 32; v < nvt; v += nthr) {
          uint4 x[NSRC];
#pragma unroll
          for (int k = 0; k < NSRC; k++) x[k] = base[k * TV + v];
          float acc[8];
          acc_first<BF16>(acc, x[0]);
#pragma unroll
          for (int k = 1; k < NSRC; k++) acc_add<BF16>(acc, x[k]);
          if (s.div) acc_div(acc, (float)s.div);
          o[v] = acc_pack<BF16>(acc);
        }
        consumer_bar(nthr);     // output tile complete, input stage fully read
        src_tile = o;
        if (storer) mbar_arrive(&pp.empty[st]);
      }
      if (storer) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int d = 0; d < ndst; d++) bulk_s2g(s.dst[d] + t0, src_tile, (uint32_t)nvt * 16);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (NSRC == 1) {
          asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          mbar_arrive(&pp.empty[st]);
        } else {
          asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        }
      }
    }
    // no drain here: the caller completes this CTA's bulk stores (bulk_store_drain) once per
    // step, before its flags are released — consecutive ops of a step then overlap their
    // store completion with the next op's loads
  }
  g += ntiles;
}

// Dynamic-tile variant of body_bulk_st for NSRC > 1 (CPS-shaped plans).  [v0, v1) is the WHOLE
// op; the producer thread takes tile indices from the op's global counter (atomicAdd), so CTAs
// that get more NVLink/HBM bandwidth take more tiles and all CTAs finish together (static
// slices finished between 0.67x and 1.0x of the slowest CTA's time: harness mtrace, 256 MiB,
// 2 x B200).  The tile index travels to the consumers through the stage's smem slot, released
// by the full barrier; when the counter runs out the producer publishes kNoTile with a plain
// arrive.  Per element the reduction is unchanged (same sources, same order): same bits.
template <int NSRC, bool BF16>
__device__ __noinline__ void body_bulk_st_dyn(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem,
                                              Pipe &pp, unsigned int *ctr) {
  const int kStages = pp.stages, kStageBytes = pp.stage_bytes, kOutTile = pp.stage_bytes / 2;
  const int T = (kStageBytes / NSRC) / 16 * 16;
  const int TV = T / 16;
  const uint32_t ntiles = (uint32_t)((v1 - v0 + TV - 1) / TV);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t used = 0;   // stage uses of this op (tiles + the closing kNoTile), identical in every thread
  if (warp == 0) {
    if (lane == 0) {
      for (;; used++) {
        const uint32_t gi = g + used, st = gi % kStages, use = gi / kStages;
        if (use > 0) mbar_wait(&pp.empty[st], (use - 1) & 1);
        const uint32_t tile = atomicAdd(ctr, 1u);
        if (tile >= ntiles) {
          pp.tile[st] = kNoTile;
          mbar_arrive(&pp.full[st]);
          used++;
          break;
        }
        pp.tile[st] = tile;
        const size_t t0 = v0 + (size_t)tile * TV;
        const uint32_t bytes = (uint32_t)min((size_t)TV, v1 - t0) * 16;
        mbar_expect_tx(&pp.full[st], bytes * NSRC);
        uint8_t *base = smem + st * kStageBytes;
#pragma unroll
        for (int k = 0; k < NSRC; k++) bulk_g2s(base + k * T, s.src[k] + t0, bytes, &pp.full[st]);
      }
    }
    used = __shfl_sync(0xffffffffu, used, 0);
  } else {
    const int ndst = s.ndst;
    const int nthr = blockDim.x - 32;
    const bool storer = threadIdx.x == 32;
    uint4 *outb = (uint4 *)(smem + kStages * kStageBytes);
    for (;; used++) {
      const uint32_t gi = g + used, st = gi % kStages, use = gi / kStages;
      mbar_wait(&pp.full[st], use & 1);
      const uint32_t tile = pp.tile[st];
      if (tile == kNoTile) {
        consumer_bar(nthr);   // every consumer has read the slot before the stage is released
        if (storer) mbar_arrive(&pp.empty[st]);
        used++;
        break;
      }
      const size_t t0 = v0 + (size_t)tile * TV;
      const int nvt = (int)min((size_t)TV, v1 - t0);
      const uint4 *base = (const uint4 *)(smem + st * kStageBytes);
      uint4 *o = outb + (gi & 1) * (kOutTile / 16);
      consumer_bar(nthr);     // the storer has drained reads of this output tile (use i-2)
      for (int v = threadIdx.x - 32; v < nvt; v += nthr) {
        uint4 x[NSRC];
#pragma unroll
        for (int k = 0; k < NSRC; k++) x[k] = base[k * TV + v];
        float acc[8];
        acc_first<BF16>(acc, x[0]);
#pragma unroll
        for (int k = 1; k < NSRC; k++) acc_add<BF16>(acc, x[k]);
        if (s.div) acc_div(acc, (float)s.div);
        o[v] = acc_pack<BF16>(acc);
      }
      consumer_bar(nthr);     // output tile complete, input stage fully read
      if (storer) {
        mbar_arrive(&pp.empty[st]);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        for (int d = 0; d < ndst; d++) bulk_s2g(s.dst[d] + t0, o, (uint32_t)nvt * 16);
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
      }
    }
    // completed by the caller (bulk_store_drain), as in body_bulk_st
  }
  g += used;
}

// Complete every bulk store this CTA's storer thread (threadIdx.x == 32) issued and order them
// before later generic-proxy operations: called once per step before the step's flags are
// released (the bar.sync of the notify then makes it cumulative), and before a kernel exits.
__device__ __forceinline__ void bulk_store_drain() {
  if (threadIdx.x == 32) {
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
  }
}

template <bool BF16>
__device__ void body_dispatch_bulk_st_dyn(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem,
                                          Pipe &pp, unsigned int *ctr) {
  switch (s.nsrc) {
    case 2: body_bulk_st_dyn<2, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 3: body_bulk_st_dyn<3, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 4: body_bulk_st_dyn<4, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 5: body_bulk_st_dyn<5, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 6: body_bulk_st_dyn<6, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 7: body_bulk_st_dyn<7, BF16>(s, v0, v1, g, smem, pp, ctr); break;
    case 8: body_bulk_st_dyn<8, BF16>(s, v0, v1, g, smem, pp, ctr); break;
  }
}

template <bool BF16>
__device__ void body_dispatch_bulk_st(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem,
                                      Pipe &pp) {
  if (s.div && s.nsrc == 1) {
    body_generic<BF16>(s, v0, v1);
    return;
  }
  switch (s.nsrc) {
    case 1: body_bulk_st<1, BF16>(s, v0, v1, g, smem, pp); break;
    case 2: body_bulk_st<2, BF16>(s, v0, v1, g, smem, pp); break;
    case 3: body_bulk_st<3, BF16>(s, v0, v1, g, smem, pp); break;
    case 4: body_bulk_st<4, BF16>(s, v0, v1, g, smem, pp); break;
    case 5: body_bulk_st<5, BF16>(s, v0, v1, g, smem, pp); break;
    case 6: body_bulk_st<6, BF16>(s, v0, v1, g, smem, pp); break;
    case 7: body_bulk_st<7, BF16>(s, v0, v1, g, smem, pp); break;
    case 8: body_bulk_st<8, BF16>(s, v0, v1, g, smem, pp); break;
    default: body_generic<BF16>(s, v0, v1); break;
  }
}

template <bool BF16>
__device__ void body_dispatch_bulk(const OpShared &s, size_t v0, size_t v1, uint32_t &g, uint8_t *smem, Pipe &pp) {
  if (s.div && s.nsrc == 1) {
    body_generic<BF16>(s, v0, v1);
    return;
  }
  switch (s.nsrc) {
    case 1: body_bulk<1, BF16>(s, v0, v1, g, smem, pp); break;
    case 2: body_bulk<2, BF16>(s, v0, v1, g, smem, pp); break;
    case 3: body_bulk<3, BF16>(s, v0, v1, g, smem, pp); break;
    case 4: body_bulk<4, BF16>(s, v0, v1, g, smem, pp); break;
    case 5: body_bulk<5, BF16>(s, v0, v1, g, smem, pp); break;
    case 6: body_bulk<6, BF16>(s, v0, v1, g, smem, pp); break;
    case 7: body_bulk<7, BF16>(s, v0, v1, g, smem, pp); break;
    case 8: body_bulk<8, BF16>(s, v0, v1, g, smem, pp); break;
    default: body_generic<BF16>(s, v0, v1); break;
  }
}

// Scalar elements [e0, e1) (unaligned head / tail), same summation order.
__device__ __noinline__ void scalar_elems(const OpShared &s, long long e0, long long e1, bool bf16) {
  for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
    if (bf16) {
      const unsigned short *p0 = (const unsigned short *)(s.src[0]) + e;
      unsigned short out;
      if (s.nsrc == 1 && !s.div) {
        out = *(volatile const unsigned short *)p0;
      } else {
        float acc = __uint_as_float((uint32_t)(*(volatile const unsigned short *)p0) << 16);
        for (int k = 1; k < s.nsrc; k++) {
          const unsigned short *pk = (const unsigned short *)(s.src[k]) + e;
          acc = __fadd_rn(acc, __uint_as_float((uint32_t)(*(volatile const unsigned short *)pk) << 16));
        }
        if (s.div) acc = __fdiv_rn(acc, (float)s.div);
        out = (unsigned short)f2bf(acc);
      }
      for (int d = 0; d < s.ndst; d++) ((unsigned short *)(s.dst[d]))[e] = out;
    } else {
      const uint32_t *p0 = (const uint32_t *)(s.src[0]) + e;
      uint32_t out;
      if (s.nsrc == 1 && !s.div) {
        out = *(volatile const uint32_t *)p0;
      } else {
        float acc = __uint_as_float(*(volatile const uint32_t *)p0);
        for (int k = 1; k < s.nsrc; k++) {
          const uint32_t *pk = (const uint32_t *)(s.src[k]) + e;
          acc = __fadd_rn(acc, __uint_as_float(*(volatile const uint32_t *)pk));
        }
        if (s.div) acc = __fdiv_rn(acc, (float)s.div);
        out = __float_as_uint(acc);
      }
      for (int d = 0; d < s.ndst; d++) ((uint32_t *)(s.dst[d]))[e] = out;
    }
  }
}

// Elements [e0, e1) of op [off, off+len) handled by CTA k of C: whole 16-byte vectors are split
// evenly and contiguously; CTA 0 also takes the unaligned head and CTA C-1 the tail (if the
// op has no whole vector, CTA 0 takes everything).  The ops loop below uses the same rule.
__device__ __forceinline__ void cta_elems(long long off, long long len, int esize, int k, int C, long long &e0,
                                          long long &e1) {
  const long long E = 16 / esize;
  const long long vb = (off * esize + 15) / 16, ve = (off + len) * esize / 16;
  if (vb >= ve) {
    e0 = k == 0 ? off : 0;
    e1 = k == 0 ? off + len : 0;
    return;
  }
  const long long nv = ve - vb;
  e0 = (vb + nv * k / C) * E;
  e1 = (vb + nv * (k + 1) / C) * E;
  if (k == 0) e0 = off;
  if (k == C - 1) e1 = off + len;
}

__device__ __forceinline__ unsigned long long *flag_ptr(const ExecArgs &a, int page_rank, int slot, int producer,
                                                        int cta) {
  return a.sigs[page_rank] + ((size_t)(slot * a.world + producer) * a.cta_cap + cta);
}

__global__ void __launch_bounds__(kThreads, 1) ar_exec_kernel(const __grid_constant__ ExecArgs a) {
  __shared__ OpShared sh;
  __shared__ Pipe pp;
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  const int lr = blockIdx.y;
  const int me = a.rank0 + lr;
  const int cta = blockIdx.x;
  const int nctas = gridDim.x;
  const bool bf16 = a.esize == 2;
  const int vec_elems = 16 / a.esize;
  const DevStep *prog = a.steps + a.prog_begin[lr];
  const int nst = a.prog_len[lr];
  const unsigned long long t_start = globaltimer();
  unsigned long long *tr = a.trace ? a.trace + (size_t)(lr * gridDim.x + cta) * kTraceSlots : nullptr;
#define AR_TRACE(i) \
  if (tr && threadIdx.x == 0 && (i) < kTraceSlots) tr[i] = globaltimer()
  AR_TRACE(0);
  uint32_t g = 0;   // bulk-pipeline tile counter (identical in every thread)
  // this call's epoch = last completed + 1; the last CTA to finish publishes it (below), so
  // every CTA reads the same value and the launch carries no per-call host argument
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = *(volatile unsigned long long *)a.epoch_dev + 1;
  if (a.bulk && threadIdx.x == 0) {
    pp.stages = a.stages;
    pp.stage_bytes = a.stage_bytes;
    for (int s = 0; s < a.stages; s++) {
      mbar_init(&pp.full[s], 1);
      mbar_init(&pp.empty[s], a.store_tma ? 1 : blockDim.x / 32 - 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const unsigned long long epoch = s_epoch;

  for (int si = 0; si < nst; si++) {
    const DevStep st = prog[si];
    // ---- waits (a1 / a3 / a5)
    if (st.wait_count > 0) {
      const int tot = st.wait_count * nctas;  // (wait, producer CTA) pairs over the threads
      for (int i = threadIdx.x; i < tot; i += blockDim.x) {
        const DevWait &w = a.waits[st.wait_begin + i / nctas];
        const int c = i % nctas;
        if (w.kind == kWaitPaired && c != cta) continue;
        if (w.kind == kWaitRange) {
          long long m0, m1, p0, p1;
          cta_elems(w.c_off, w.c_len, a.esize, cta, nctas, m0, m1);
          cta_elems(w.p_off, w.p_len, a.esize, c, nctas, p0, p1);
          if (!(m0 < m1 && p0 < p1 && m0 < p1 && p0 < m1)) continue;
        }
        const unsigned long long *f = flag_ptr(a, me, w.slot, w.rank, c);
        unsigned int spins = 0;
        while (ld_acquire_sys(f) < epoch) {
          if ((++spins & 1023u) == 0 && globaltimer() - t_start > a.timeout_ns) {
            atomicExch(a.err, 1ull);
            break;
          }
        }
      }
      __syncthreads();
      // the bulk loads below run in the async proxy: order them after the generic-proxy
      // writes this acquire made visible.  Only their issuer (thread 0, the bulk producer)
      // needs the proxy fence — executed by all 512 threads it was the kernel's top stall
      // (ncu, RHD on 8 emulated ranks: 12 % of the warp samples)
      if (!a.bulk || threadIdx.x == 0) asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    AR_TRACE(1 + 3 * si);
    // ---- ops (a2 / a4)
    for (int oi = 0; oi < st.op_count; oi++) {
      const DevOp op = a.ops[st.op_begin + oi];
      const int *sr = a.ranks + op.src_begin;
      const int *dr = a.ranks + op.dst_begin;
      const long long b0 = op.off * a.esize, b1 = (op.off + op.len) * a.esize;
      const long long vb = (b0 + 15) / 16, ve = b1 / 16;   // whole 16-byte vectors
      __syncthreads();
      if (threadIdx.x < op.nsrc) sh.src[threadIdx.x] = (const uint4 *)ref_base(a, sr[threadIdx.x], op.off, epoch);
      if (threadIdx.x < op.ndst) sh.dst[threadIdx.x] = (uint4 *)ref_base(a, dr[threadIdx.x], op.off, epoch);
      if (threadIdx.x == 0) {
        sh.nsrc = op.nsrc;
        sh.ndst = op.ndst;
        sh.div = op.fin ? a.avg_n : 0;
      }
      __syncthreads();
      if (vb >= ve) {
        if (cta == 0) scalar_elems(sh, op.off, op.off + op.len, bf16);
        continue;
      }
      const long long nv = ve - vb;
      const size_t v0 = (size_t)(vb + nv * cta / nctas), v1 = (size_t)(vb + nv * (cta + 1) / nctas);
      if (a.dyn_ctr && op.nsrc >= 2 && op.nsrc <= 8) {
        unsigned int *ctr = a.dyn_ctr + st.op_begin + oi;
        if (bf16) body_dispatch_bulk_st_dyn<true>(sh, (size_t)vb, (size_t)ve, g, dyn_smem, pp, ctr);
        else body_dispatch_bulk_st_dyn<false>(sh, (size_t)vb, (size_t)ve, g, dyn_smem, pp, ctr);
      } else if (a.bulk) {
        if (a.store_tma) {
          if (bf16) body_dispatch_bulk_st<true>(sh, v0, v1, g, dyn_smem, pp);
          else body_dispatch_bulk_st<false>(sh, v0, v1, g, dyn_smem, pp);
        } else {
          if (bf16) body_dispatch_bulk<true>(sh, v0, v1, g, dyn_smem, pp);
          else body_dispatch_bulk<false>(sh, v0, v1, g, dyn_smem, pp);
        }
      } else {
        if (bf16) body_dispatch<true>(sh, v0, v1);
        else body_dispatch<false>(sh, v0, v1);
      }
      if (cta == 0 && vb * 16 > b0) scalar_elems(sh, op.off, vb * vec_elems, bf16);
      if (cta == nctas - 1 && ve * 16 < b1) scalar_elems(sh, ve * vec_elems, op.off + op.len, bf16);
    }
    if (st.op_count > 0 && a.bulk && a.store_tma) bulk_store_drain();
    AR_TRACE(2 + 3 * si);
    // ---- notify (release our slot on every consumer's page)
    if (st.notify_count > 0) {
      if (a.jitter_ns && threadIdx.x == 0) {
        // stress mode: delay this CTA's flags by a pseudo-random amount (ordering bugs surface
        // as wrong results instead of hiding behind typical timing)
        unsigned int h = (unsigned int)(cta * 2654435761u) ^ (unsigned int)(si * 40503u) ^
                         (unsigned int)(me * 97u) ^ (unsigned int)epoch;
        h ^= h >> 13;
        h *= 0x5bd1e995u;
        __nanosleep(h % a.jitter_ns);
      }
      // Every thread's data stores of this step happen-before the barrier; the release
      // store(s) after it are cumulative over them (PTX memory model: bar.sync synchronises
      // the CTA, st.release is a release pattern).  fence_mode 0 additionally fences every
      // thread at system scope (membar.sys per thread: ~10 us on B200, measured).
      if (st.slot == 0 && st.op_count == 0 && a.fence_mode != 0) {
        // entry flag: this kernel wrote nothing yet, and the buffer it announces was made
        // final by stream order (earlier kernels) and by the previous call's exit waits, so
        // there is nothing for a release to order — a relaxed system-scope store suffices
        // (st.release.sys costs ~5 us on B200 even with no prior writes: measured with
        // `harness.py mtrace --steady`)
        if (a.entry_fence) {   // AR_ENTRY_FENCE=1: order earlier work at system scope first
          if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
          __syncthreads();
        }
        for (int i = threadIdx.x; i < st.notify_count; i += blockDim.x) {
          const int consumer = a.ranks[st.notify_begin + i];
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag_ptr(a, consumer, st.slot, me, cta)),
                       "l"(epoch)
                       : "memory");
        }
        AR_TRACE(3 + 3 * si);
        continue;
      }
      if (a.fence_mode == 0) __threadfence_system();
      __syncthreads();
      if (a.fence_mode == 2) {
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
        __syncthreads();
        for (int i = threadIdx.x; i < st.notify_count; i += blockDim.x) {
          const int consumer = a.ranks[st.notify_begin + i];
          asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(flag_ptr(a, consumer, st.slot, me, cta)),
                       "l"(epoch)
                       : "memory");
        }
      } else if (a.fence_mode == 3) {   // all ranks on this GPU (emulated comm): gpu scope
        for (int i = threadIdx.x; i < st.notify_count; i += blockDim.x) {
          const int consumer = a.ranks[st.notify_begin + i];
          asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(flag_ptr(a, consumer, st.slot, me, cta)),
                       "l"(epoch)
                       : "memory");
        }
      } else {
        for (int i = threadIdx.x; i < st.notify_count; i += blockDim.x) {
          const int consumer = a.ranks[st.notify_begin + i];
          st_release_sys(flag_ptr(a, consumer, st.slot, me, cta), epoch);
        }
      }
    }
    AR_TRACE(3 + 3 * si);
  }
  AR_TRACE(kTraceSlots - 1);
#undef AR_TRACE
  // publish the epoch once every CTA of this launch is done (they have all read it)
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned int total = gridDim.x * gridDim.y;
    if (atomicAdd(a.done_ctr, 1u) == total - 1) {
      *(volatile unsigned int *)a.done_ctr = 0;
      for (int i = 0; i < a.dyn_nops; i++) a.dyn_ctr[i] = 0u;   // every CTA is past its ops
      *(volatile unsigned long long *)a.epoch_dev = epoch;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ flat single-step path
// Emulated ranks (all buffers on this GPU) and a CPS-shaped plan: the plan is one fused step
// whose ops (one per owner block) touch disjoint regions, and every input was written before
// the launch — so no flag is needed at all.  The ops' 16-byte vectors are concatenated and
// split evenly over every SM (148 CTAs instead of floor(148/R)·R), each CTA running the same
// bulk-copy pipeline and summation order as ar_exec_kernel; CTA 0 also does the unaligned
// heads/tails.  Bits are the plan's.
struct FlatArgs {
  char *base;
  long long stride, count;
  int world, esize, avg_n;
  int order[AR_MAX_RANKS];
  int stages, stage_bytes;
  // dynamic tile scheduling (world <= 8): [0, world) per-owner-block tile counters, [world] the
  // launch's finished-CTA count; nullptr = static equal slices of the concatenated blocks
  unsigned int *ctr;
};

__global__ void __launch_bounds__(kThreads, 1) ar_flat_kernel(const __grid_constant__ FlatArgs a) {
  __shared__ OpShared sh;
  __shared__ Pipe pp;
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  const bool bf16 = a.esize == 2;
  const long long E = 16 / a.esize;
  if (threadIdx.x == 0) {
    pp.stages = a.stages;
    pp.stage_bytes = a.stage_bytes;
    for (int st = 0; st < a.stages; st++) {
      mbar_init(&pp.full[st], 1);
      mbar_init(&pp.empty[st], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // total whole vectors over all owner blocks
  long long total = 0;
  for (int r = 0; r < a.world; r++) {
    const long long off = a.count / a.world * r + min((long long)r, a.count % a.world);
    const long long len = a.count / a.world + (r < a.count % a.world ? 1 : 0);
    const long long vb = (off * a.esize + 15) / 16, ve = (off + len) * a.esize / 16;
    if (ve > vb) total += ve - vb;
  }
  const long long my0 = total * blockIdx.x / gridDim.x, my1 = total * (blockIdx.x + 1) / gridDim.x;
  uint32_t g = 0;
  if (a.ctr) {
    // every CTA works on every owner block, taking tiles from the block's counter (same
    // pipeline and per-element order as the static split; body_bulk_st_dyn)
    for (int r = 0; r < a.world; r++) {
      const long long off = a.count / a.world * r + min((long long)r, a.count % a.world);
      const long long len = a.count / a.world + (r < a.count % a.world ? 1 : 0);
      const long long vb = (off * a.esize + 15) / 16, ve = (off + len) * a.esize / 16;
      const bool mine_scalar = blockIdx.x == 0 && len > 0 && (ve <= vb || vb * 16 > off * a.esize ||
                                                              ve * 16 < (off + len) * a.esize);
      if (ve <= vb && !mine_scalar) continue;
      __syncthreads();
      if (threadIdx.x < a.world) {
        sh.src[threadIdx.x] = (const uint4 *)(a.base + a.stride * a.order[threadIdx.x]);
        sh.dst[threadIdx.x] = (uint4 *)(a.base + a.stride * threadIdx.x);
      }
      if (threadIdx.x == 0) {
        sh.nsrc = a.world;
        sh.ndst = a.world;
        sh.div = a.avg_n;
      }
      __syncthreads();
      if (ve > vb) {
        if (bf16) body_dispatch_bulk_st_dyn<true>(sh, (size_t)vb, (size_t)ve, g, dyn_smem, pp, a.ctr + r);
        else body_dispatch_bulk_st_dyn<false>(sh, (size_t)vb, (size_t)ve, g, dyn_smem, pp, a.ctr + r);
      }
      if (mine_scalar) {
        if (ve <= vb) {
          scalar_elems(sh, off, off + len, bf16);
        } else {
          if (vb * 16 > off * a.esize) scalar_elems(sh, off, vb * E, bf16);
          if (ve * 16 < (off + len) * a.esize) scalar_elems(sh, ve * E, off + len, bf16);
        }
      }
    }
    bulk_store_drain();
    __syncthreads();
    if (threadIdx.x == 0 && atomicAdd(a.ctr + a.world, 1u) == gridDim.x - 1)
      for (int i = 0; i <= a.world; i++) a.ctr[i] = 0u;   // every CTA is past every block
    return;
  }
  long long acc = 0;
  for (int r = 0; r < a.world; r++) {
    const long long off = a.count / a.world * r + min((long long)r, a.count % a.world);
    const long long len = a.count / a.world + (r < a.count % a.world ? 1 : 0);
    const long long vb = (off * a.esize + 15) / 16, ve = (off + len) * a.esize / 16;
    const long long nv = ve > vb ? ve - vb : 0;
    const long long lo = max(my0, acc), hi = min(my1, acc + nv);
    const bool mine_vec = lo < hi;
    const bool mine_scalar = blockIdx.x == 0 && len > 0 && (nv == 0 || vb * 16 > off * a.esize ||
                                                            ve * 16 < (off + len) * a.esize);
    if (mine_vec || mine_scalar) {
      __syncthreads();
      if (threadIdx.x < a.world) {
        sh.src[threadIdx.x] = (const uint4 *)(a.base + a.stride * a.order[threadIdx.x]);
        sh.dst[threadIdx.x] = (uint4 *)(a.base + a.stride * threadIdx.x);
      }
      if (threadIdx.x == 0) {
        sh.nsrc = a.world;
        sh.ndst = a.world;
        sh.div = a.avg_n;
      }
      __syncthreads();
      if (mine_vec) {
        const size_t v0 = (size_t)(vb + lo - acc), v1 = (size_t)(vb + hi - acc);
        if (bf16) body_dispatch_bulk_st<true>(sh, v0, v1, g, dyn_smem, pp);
        else body_dispatch_bulk_st<false>(sh, v0, v1, g, dyn_smem, pp);
      }
      if (mine_scalar) {
        if (nv == 0) {
          scalar_elems(sh, off, off + len, bf16);
        } else {
          if (vb * 16 > off * a.esize) scalar_elems(sh, off, vb * E, bf16);
          if (ve * 16 < (off + len) * a.esize) scalar_elems(sh, ve * E, off + len, bf16);
        }
      }
    }
    acc += nv;
  }
  bulk_store_drain();
}

// ------------------------------------------------------------------ multi-step plans on emulated ranks
// All ranks in one HBM (emulated comm), a multi-step plan (Ring, RHD, HCPS, rearrangement):
// every executed step's ops are independent of each other (O3; the fusion rule keeps it so), so
// the ops of ALL ranks in a step are concatenated and split evenly over every SM, as in
// ar_flat_kernel, and a grid-wide barrier separates consecutive steps in place of the
// step-table kernel's per-rank flags.  Same bodies, summation order and rounding: the plan's
// bits.  One cooperative launch (every CTA resident for the barrier).  An A/B option
// (AR_FLATSTEPS=1): the barrier serialises the steps, and the step-table kernel's range waits
// (dependent steps overlapping CTA by CTA) measured as fast in bf16 and faster in fp32.
struct FlatStepsArgs {
  char *base;
  long long stride;
  const DevOp *ops;                  // the ops of global step s: [gbegin[s], gbegin[s + 1])
  const int *ranks;                  // src / dst rank lists of the ops
  const int *gbegin;
  int nsteps, esize, avg_n, stages, stage_bytes;
  unsigned int *bar;                 // [0] barrier arrivals, [1] finished CTAs (reset by the last)
  unsigned long long *err;
  unsigned long long timeout_ns;
};

__global__ void __launch_bounds__(kThreads, 1) ar_flatsteps_kernel(const __grid_constant__ FlatStepsArgs a) {
  __shared__ OpShared sh;
  __shared__ Pipe pp;
  extern __shared__ __align__(128) uint8_t dyn_smem[];
  const bool bf16 = a.esize == 2;
  const long long E = 16 / a.esize;
  const unsigned long long t0 = globaltimer();
  if (threadIdx.x == 0) {
    pp.stages = a.stages;
    pp.stage_bytes = a.stage_bytes;
    for (int st = 0; st < a.stages; st++) {
      mbar_init(&pp.full[st], 1);
      mbar_init(&pp.empty[st], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t g = 0;
  for (int s = 0; s < a.nsteps; s++) {
    if (s > 0) {
      // grid barrier: the previous step's bulk stores are complete (bulk_store_drain) and
      // released at gpu scope before this CTA's arrival; the acquire below orders this
      // step's reads (the bulk producer also fences the async proxy)
      __syncthreads();
      if (threadIdx.x == 0) {
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(a.bar) : "memory");
        const unsigned int target = (unsigned int)s * gridDim.x;
        unsigned int spins = 0;
        for (;;) {
          unsigned int v;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(a.bar) : "memory");
          if (v >= target) break;
          if ((++spins & 1023u) == 0 && globaltimer() - t0 > a.timeout_ns) {
            atomicExch(a.err, 1ull);
            break;
          }
        }
        asm volatile("fence.proxy.async.global;" ::: "memory");
      }
      __syncthreads();
    }
    const int o0 = a.gbegin[s], o1 = a.gbegin[s + 1];
    long long total = 0;
    for (int oi = o0; oi < o1; oi++) {
      const DevOp &op = a.ops[oi];
      const long long vb = (op.off * a.esize + 15) / 16, ve = (op.off + op.len) * a.esize / 16;
      if (ve > vb) total += ve - vb;
    }
    const long long my0 = total * blockIdx.x / gridDim.x, my1 = total * (blockIdx.x + 1) / gridDim.x;
    long long acc = 0;
    for (int oi = o0; oi < o1; oi++) {
      const DevOp op = a.ops[oi];
      const long long vb = (op.off * a.esize + 15) / 16, ve = (op.off + op.len) * a.esize / 16;
      const long long nv = ve > vb ? ve - vb : 0;
      const long long lo = max(my0, acc), hi = min(my1, acc + nv);
      const bool mine_vec = lo < hi;
      const bool mine_scalar = blockIdx.x == 0 && op.len > 0 &&
                               (nv == 0 || vb * 16 > op.off * a.esize || ve * 16 < (op.off + op.len) * a.esize);
      if (mine_vec || mine_scalar) {
        __syncthreads();
        if (threadIdx.x < op.nsrc) sh.src[threadIdx.x] = (const uint4 *)(a.base + a.stride * a.ranks[op.src_begin + threadIdx.x]);
        if (threadIdx.x < op.ndst) sh.dst[threadIdx.x] = (uint4 *)(a.base + a.stride * a.ranks[op.dst_begin + threadIdx.x]);
        if (threadIdx.x == 0) {
          sh.nsrc = op.nsrc;
          sh.ndst = op.ndst;
          sh.div = op.fin ? a.avg_n : 0;
        }
        __syncthreads();
        if (mine_vec) {
          const size_t v0 = (size_t)(vb + lo - acc), v1 = (size_t)(vb + hi - acc);
          if (bf16) body_dispatch_bulk_st<true>(sh, v0, v1, g, dyn_smem, pp);
          else body_dispatch_bulk_st<false>(sh, v0, v1, g, dyn_smem, pp);
        }
        if (mine_scalar) {
          if (nv == 0) {
            scalar_elems(sh, op.off, op.off + op.len, bf16);
          } else {
            if (vb * 16 > op.off * a.esize) scalar_elems(sh, op.off, vb * E, bf16);
            if (ve * 16 < (op.off + op.len) * a.esize) scalar_elems(sh, ve * E, op.off + op.len, bf16);
          }
        }
      }
      acc += nv;
    }
    bulk_store_drain();
  }
  __syncthreads();
  if (threadIdx.x == 0 && atomicAdd(a.bar + 1, 1u) == gridDim.x - 1) {
    a.bar[0] = 0u;   // every CTA is past its last barrier
    a.bar[1] = 0u;
    __threadfence();
  }
}

// ------------------------------------------------------------------ low-latency one-shot path
// Small messages on one rank per GPU, CPS-shaped plans (one fan-in-N reduce per block, every
// block with the same input order): every rank pushes its whole input to every peer's
// scratch as 16-byte lines {d0, e, d1, e} (8 payload bytes + the call's epoch twice; each
// 8-byte half is written atomically over NVLink, so a line is valid once both flags read e),
// then computes *every* block itself in the plan's order — bit-identical to the plan (same
// inputs, same association) — and writes only its own buffer.  No entry or exit flag round
// trips: inputs are read only by their owner, outputs written only by their owner.  Scratch
// is double-buffered by epoch parity: a peer that writes call e's lines has finished call
// e-1, which consumed this rank's call e-1 lines, pushed after this rank finished call e-2.
struct LLArgs {
  char *buf;                              // this rank's data (in place)
  char *peer_scratch[AR_MAX_RANKS];       // rank -> its scratch base as seen here
  char *my_scratch;
  int order[AR_MAX_RANKS];                // summation order (the plan's reduce inputs)
  long long bytes, cap_lines;
  int me, world, esize, avg_n;
  unsigned long long *epoch_dev;          // last completed LL call (device-resident)
  unsigned int *done_ctr;
  unsigned long long *err;
  unsigned long long timeout_ns;
};

__device__ __forceinline__ void st_vol_v4(void *p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d) : "memory");
}
__device__ __forceinline__ uint4 ld_vol_v4(const void *p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// 8 payload bytes of line i (zero-padded past the end of the buffer)
__device__ __forceinline__ uint2 ll_load(const char *buf, long long bytes, long long i) {
  if ((i + 1) * 8 <= bytes) return *(const uint2 *)(buf + i * 8);
  uint32_t w[2] = {0u, 0u};
  for (long long b = i * 8; b < bytes; b++) ((unsigned char *)w)[b - i * 8] = (unsigned char)buf[b];
  return make_uint2(w[0], w[1]);
}

__global__ void __launch_bounds__(kThreads) ar_ll_kernel(const __grid_constant__ LLArgs a) {
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = *(volatile unsigned long long *)a.epoch_dev + 1;
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const uint32_t e = (uint32_t)epoch;
  const int par = (int)(epoch & 1ull);
  const long long L = (a.bytes + 7) / 8;
  const long long nthr = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t plane = (size_t)a.cap_lines * 16;
  // phase 1: push my lines to every peer
  for (long long i = t0; i < L; i += nthr) {
    const uint2 v = ll_load(a.buf, a.bytes, i);
    for (int t = 0; t < a.world; t++) {
      if (t == a.me) continue;
      char *dst = a.peer_scratch[t] + ((size_t)par * a.world + a.me) * plane + (size_t)i * 16;
      st_vol_v4(dst, v.x, e, v.y, e);
    }
  }
  // phase 2: reduce every line in plan order (same thread <-> line mapping as phase 1)
  const unsigned long long start = globaltimer();
  const bool bf16 = a.esize == 2;
  for (long long i = t0; i < L; i += nthr) {
    float acc[4];
    const int per = bf16 ? 4 : 2;
    for (int k = 0; k < a.world; k++) {
      const int src = a.order[k];
      uint2 v;
      if (src == a.me) {
        v = ll_load(a.buf, a.bytes, i);
      } else {
        const char *p = a.my_scratch + ((size_t)par * a.world + src) * plane + (size_t)i * 16;
        uint4 x = ld_vol_v4(p);
        unsigned int spins = 0;
        while (x.y != e || x.w != e) {
          if ((++spins & 1023u) == 0 && globaltimer() - start > a.timeout_ns) {
            atomicExch(a.err, 1ull);
            break;
          }
          x = ld_vol_v4(p);
        }
        v = make_uint2(x.x, x.z);
      }
      float f[4];
      if (bf16) {
        f[0] = bf_lo(v.x); f[1] = bf_hi(v.x); f[2] = bf_lo(v.y); f[3] = bf_hi(v.y);
      } else {
        f[0] = __uint_as_float(v.x); f[1] = __uint_as_float(v.y);
      }
      for (int j = 0; j < per; j++) acc[j] = k == 0 ? f[j] : __fadd_rn(acc[j], f[j]);
    }
    if (a.avg_n)
      for (int j = 0; j < per; j++) acc[j] = __fdiv_rn(acc[j], (float)a.avg_n);
    uint2 o;
    if (bf16) {
      o.x = f2bf2(acc[0], acc[1]);
      o.y = f2bf2(acc[2], acc[3]);
    } else {
      o.x = __float_as_uint(acc[0]);
      o.y = __float_as_uint(acc[1]);
    }
    if ((i + 1) * 8 <= a.bytes) {
      *(uint2 *)(a.buf + i * 8) = o;
    } else {
      const uint32_t w[2] = {o.x, o.y};
      for (long long b = i * 8; b < a.bytes; b++) a.buf[b] = (char)((const unsigned char *)w)[b - i * 8];
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *(volatile unsigned int *)a.done_ctr = 0;
      *(volatile unsigned long long *)a.epoch_dev = epoch;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ LL128 two-shot path
// Mid-size messages on one rank per GPU, CPS-shaped plans whose blocks start on 16-byte
// boundaries: the CPS plan's RS and AG steps with the flags carried IN the data, so no flag
// round trip and no system-scope release is needed (each costs microseconds on B200, §6).
// Data moves in 128-byte lines: 120 payload bytes + an 8-byte flag = the call's epoch in the
// last 8 bytes.  Eight lanes write one line with one warp-wide 16-byte-per-lane store, which
// NVLink delivers as one 128-byte write; a reader loads the line the same way (one 128-byte
// read) and accepts it only when the flag equals its epoch — the property NCCL's LL128
// protocol relies on.  Per call and rank r:
//   1. for every block b != r: write my slice of block b as lines into owner b's RS area;
//   2. reduce my block r in the plan's order (my own slice from my buffer, the others'
//      from my RS area once their flags arrive), store the result into my buffer and as
//      lines into every peer's AG area;
//   3. copy every other owner's result lines from my AG area into my buffer.
// Same inputs, same association and the same rounding as the CPS plan: the plan's bits.
// Scratch is double-buffered by epoch parity, with the argument of ar_ll_kernel.
struct LL128Args {
  char *buf;                              // this rank's data (in place)
  char *peer_scr[AR_MAX_RANKS];           // rank -> its LL128 region as seen here
  char *my_scr;
  int order[AR_MAX_RANKS];                // the plan's summation order
  // the LL128 partition (not the plan's: a CPS-shaped plan's bits do not depend on which rank
  // sums an element): blocks 0..N-2 of blk_bytes (a multiple of 8), block N-1 the rest
  long long blk_bytes;                    // bytes of blocks 0..N-2
  long long lines;                        // 128-byte lines of blocks 0..N-2
  long long last_bytes, last_lines;       // block N-1 (blk_bytes <= last_bytes < blk_bytes + 8N)
  long long lines_cap;                    // lines per (parity, area, source) slot
  int me, world, esize, avg_n;
  unsigned long long *epoch_dev;          // last completed LL128 call (device-resident)
  unsigned int *done_ctr;
  unsigned long long *err;
  unsigned long long timeout_ns;
};
constexpr int kLineBytes = 128, kLinePayload = 120;

__device__ __forceinline__ void st_vol_v2u64(void *p, unsigned long long a, unsigned long long b) {
  asm volatile("st.volatile.global.v2.u64 [%0], {%1,%2};" ::"l"(p), "l"(a), "l"(b) : "memory");
}
__device__ __forceinline__ void ld_vol_v2u64(const void *p, unsigned long long &a, unsigned long long &b) {
  asm volatile("ld.volatile.global.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p) : "memory");
}
// scratch line: [parity][area (0 = RS, 1 = AG)][source rank][line]
__device__ __forceinline__ char *ll128_line(char *base, const LL128Args &a, int par, int area, int src, long long i) {
  return base + ((((long long)par * 2 + area) * a.world + src) * a.lines_cap + i) * kLineBytes;
}
// An 8-byte payload word at p with `rem` bytes of the block left from p: whole words directly,
// the block's last partial word (2, 4 or 6 bytes: elements are 2 or 4 bytes) element-pairwise
// out of line (at most one word per block), bytes past the block's end as 0 (never stored back)
__device__ __forceinline__ unsigned long long ll128_ld_partial(const char *p, int rem) {
  unsigned long long w = 0ull;
  for (int k = 0; k < rem; k += 2) w |= (unsigned long long)*(const unsigned short *)(p + k) << (8 * k);
  return w;
}
__device__ __forceinline__ void ll128_st_partial(char *p, int rem, unsigned long long w) {
  for (int k = 0; k < rem; k += 2) *(unsigned short *)(p + k) = (unsigned short)(w >> (8 * k));
}
__device__ __forceinline__ unsigned long long ll128_ld_word(const char *p, long long rem) {
  if (rem >= 8) return *(const unsigned long long *)p;
  return rem > 0 ? ll128_ld_partial(p, (int)rem) : 0ull;
}
__device__ __forceinline__ void ll128_st_word(char *p, long long rem, unsigned long long w) {
  if (rem >= 8) *(unsigned long long *)p = w;
  else if (rem > 0) ll128_st_partial(p, (int)rem, w);
}
// this lane's payload words of line i of a block that starts at `blk` (part j < 7: bytes
// 16j..16j+15, part 7: bytes 112..119).  RAGGED = false: blk_bytes is a multiple of 8 (equal
// 16-byte-aligned blocks), whole words only
template <bool RAGGED>
__device__ __forceinline__ void ll128_payload(const char *blk, long long blk_bytes, long long i, int j,
                                              unsigned long long &w0, unsigned long long &w1) {
  const long long o = i * kLinePayload + 16LL * j;
  if (RAGGED) {
    w0 = ll128_ld_word(blk + o, blk_bytes - o);
    w1 = j < 7 ? ll128_ld_word(blk + o + 8, blk_bytes - o - 8) : 0ull;
  } else {
    w0 = o + 8 <= blk_bytes ? *(const unsigned long long *)(blk + o) : 0ull;
    w1 = (j < 7 && o + 16 <= blk_bytes) ? *(const unsigned long long *)(blk + o + 8) : 0ull;
  }
}
template <bool RAGGED>
__device__ __forceinline__ void ll128_store_payload(char *blk, long long blk_bytes, long long i, int j,
                                                    unsigned long long w0, unsigned long long w1) {
  const long long o = i * kLinePayload + 16LL * j;
  if (RAGGED) {
    ll128_st_word(blk + o, blk_bytes - o, w0);
    if (j < 7) ll128_st_word(blk + o + 8, blk_bytes - o - 8, w1);
  } else {
    if (o + 8 <= blk_bytes) *(unsigned long long *)(blk + o) = w0;
    if (j < 7 && o + 16 <= blk_bytes) *(unsigned long long *)(blk + o + 8) = w1;
  }
}
// Load line i from a scratch slot until its flag (lane 7 of the 8-lane group, second word)
// equals `flag`.  Every lane of the warp runs the loop (__any_sync); lanes without a line
// (live == false) count as valid.
__device__ __forceinline__ bool ll128_load(const char *line, int j, bool live, unsigned long long flag,
                                           unsigned long long &w0, unsigned long long &w1,
                                           const LL128Args &a, unsigned long long start) {
  const int lane = threadIdx.x & 31;
  unsigned int spins = 0;
  for (;;) {
    if (live) ld_vol_v2u64(line + 16 * j, w0, w1);
    const unsigned long long f = __shfl_sync(0xffffffffu, w1, (lane & ~7) | 7);
    const bool bad = live && f != flag;
    if (!__any_sync(0xffffffffu, bad)) return true;
    if ((++spins & 1023u) == 0 && globaltimer() - start > a.timeout_ns) {
      atomicExch(a.err, 1ull);
      return false;
    }
  }
}

template <bool BF16>
__device__ __forceinline__ void ll128_acc(float (&acc)[8], unsigned long long w0, unsigned long long w1, bool first) {
  const uint32_t u[4] = {(uint32_t)w0, (uint32_t)(w0 >> 32), (uint32_t)w1, (uint32_t)(w1 >> 32)};
#pragma unroll
  for (int k = 0; k < (BF16 ? 8 : 4); k++) {
    const float v = BF16 ? ((k & 1) ? bf_hi(u[k >> 1]) : bf_lo(u[k >> 1])) : __uint_as_float(u[k]);
    acc[k] = first ? v : __fadd_rn(acc[k], v);
  }
}
template <bool BF16>
__device__ __forceinline__ void ll128_pack(const float (&acc)[8], unsigned long long &w0, unsigned long long &w1) {
  uint32_t u[4];
  if (BF16) {
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = f2bf2(acc[2 * k], acc[2 * k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < 4; k++) u[k] = __float_as_uint(acc[k]);
  }
  w0 = (unsigned long long)u[0] | ((unsigned long long)u[1] << 32);
  w1 = (unsigned long long)u[2] | ((unsigned long long)u[3] << 32);
}

// RAGGED = false: all N blocks equal (last_bytes == blk_bytes), the measured fast path;
// RAGGED = true: any count (the last block longer, possibly ending in a partial word)
template <bool BF16, bool RAGGED>
__global__ void __launch_bounds__(kThreads, 3) ar_ll128_kernel(const __grid_constant__ LL128Args a) {
  __shared__ unsigned long long s_epoch;
  if (threadIdx.x == 0) s_epoch = *(volatile unsigned long long *)a.epoch_dev + 1;
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  const int par = (int)(epoch & 1ull);
  const int lane = threadIdx.x & 31, j = lane & 7, sub = lane >> 3;
  const long long gwarp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  const unsigned long long start = globaltimer();
  // block b's bytes and lines in the LL128 partition; loop trip counts depend only on b, so
  // every lane of a warp runs the same number of iterations (the loads' warp votes)
  auto bbytes = [&](int b) { return RAGGED && b == a.world - 1 ? a.last_bytes : a.blk_bytes; };
  auto blines = [&](int b) { return RAGGED && b == a.world - 1 ? a.last_lines : a.lines; };
  auto trips = [&](long long L) { return (L + nwarps * 4 - 1) / (nwarps * 4); };
  // 1. scatter my slices of the other blocks to their owners
  for (int b = 0; b < a.world; b++) {
    if (b == a.me) continue;
    const char *blk = a.buf + (long long)b * a.blk_bytes;
    const long long L = blines(b), nb = bbytes(b), iters = trips(L);
    char *dst = ll128_line(a.peer_scr[b], a, par, 0, a.me, 0);
    for (long long it = 0; it < iters; it++) {
      const long long i = (it * nwarps + gwarp) * 4 + sub;
      if (i >= L) continue;
      unsigned long long w0, w1;
      ll128_payload<RAGGED>(blk, nb, i, j, w0, w1);
      st_vol_v2u64(dst + i * kLineBytes + 16 * j, w0, j == 7 ? epoch : w1);
    }
  }
  // 2. reduce my block in the plan's order; result to my buffer and every peer's AG area
  {
    char *blk = a.buf + (long long)a.me * a.blk_bytes;
    const long long L = blines(a.me), nb = bbytes(a.me), iters = trips(L);
    for (long long it = 0; it < iters; it++) {
      const long long i = (it * nwarps + gwarp) * 4 + sub;
      const bool live = i < L;
      float acc[8];
      for (int k = 0; k < a.world; k++) {
        const int q = a.order[k];
        unsigned long long w0 = 0, w1 = 0;
        if (q == a.me) {
          if (live) ll128_payload<RAGGED>(blk, nb, i, j, w0, w1);
        } else {
          ll128_load(ll128_line(a.my_scr, a, par, 0, q, live ? i : 0), j, live, epoch, w0, w1, a, start);
          if (j == 7) w1 = 0ull;   // the flag word carries no payload
        }
        ll128_acc<BF16>(acc, w0, w1, k == 0);
      }
      if (!live) continue;
      if (a.avg_n)
        for (int k = 0; k < 8; k++) acc[k] = __fdiv_rn(acc[k], (float)a.avg_n);
      unsigned long long r0, r1;
      ll128_pack<BF16>(acc, r0, r1);
      ll128_store_payload<RAGGED>(blk, nb, i, j, r0, r1);
      for (int d = 0; d < a.world; d++) {
        if (d == a.me) continue;
        st_vol_v2u64(ll128_line(a.peer_scr[d], a, par, 1, a.me, i) + 16 * j, r0, j == 7 ? epoch : r1);
      }
    }
  }
  // 3. gather the other owners' results
  for (int o = 0; o < a.world; o++) {
    if (o == a.me) continue;
    char *blk = a.buf + (long long)o * a.blk_bytes;
    const long long L = blines(o), nb = bbytes(o), iters = trips(L);
    for (long long it = 0; it < iters; it++) {
      const long long i = (it * nwarps + gwarp) * 4 + sub;
      const bool live = i < L;
      unsigned long long w0 = 0, w1 = 0;
      ll128_load(ll128_line(a.my_scr, a, par, 1, o, live ? i : 0), j, live, epoch, w0, w1, a, start);
      if (live) ll128_store_payload<RAGGED>(blk, nb, i, j, w0, w1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (atomicAdd(a.done_ctr, 1u) == gridDim.x - 1) {
      *(volatile unsigned int *)a.done_ctr = 0;
      *(volatile unsigned long long *)a.epoch_dev = epoch;
      __threadfence();
    }
  }
}

// ------------------------------------------------------------------ synthetic inputs
__device__ __forceinline__ unsigned long long splitmix64(unsigned long long x) {
  x += 0x9E3779B97F4A7C15ull;
  unsigned long long z = x;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

__constant__ uint32_t kSpecF32[12] = {0x00000000u, 0x80000000u, 0x00000001u, 0x807FFFFFu, 0x7F7FFFFFu, 0xFF7FFFFFu,
                                       0x7F800000u, 0xFF800000u, 0x7FC00000u, 0x00800000u, 0x80000010u, 0x3F800000u};
__constant__ uint16_t kSpecBF16[12] = {0x0000, 0x8000, 0x0001, 0x807F, 0x7F7F, 0xFF7F,
                                        0x7F80, 0xFF80, 0x7FC0, 0x0080, 0x8010, 0x3F80};

__global__ void fill_kernel(void *dptr, unsigned long long count, int bf16, unsigned long long seed, int rank,
                            int mode, unsigned long long start) {
  const unsigned long long key = (seed * 0x9E3779B97F4A7C15ull) ^ ((unsigned long long)rank << 48);
  for (unsigned long long j = blockIdx.x * (unsigned long long)blockDim.x + threadIdx.x; j < count;
       j += (unsigned long long)gridDim.x * blockDim.x) {
    const unsigned long long i = start + j;
    const unsigned long long z = splitmix64(key ^ i);
    uint32_t bits;
    if (mode == 1) {
      long long m = bf16 ? (long long)(z % 65ull) - 32 : (long long)(z % 2049ull) - 1024;
      bits = __float_as_uint((float)m);
      if (bf16) bits >>= 16;
    } else {
      const int e = 7 + (int)(splitmix64((seed ^ 0xA5A5ull) ^ (i >> 16)) % 12ull);
      if (!bf16) {
        long long m = (long long)((z >> 40) & 0xFFFFFFull) - 0x800000ll;
        bits = __float_as_uint(ldexpf((float)m, -(23 + e)));
        if (mode == 2 && (i % 8ull) == 0) bits = kSpecF32[(i / 8ull) % 12ull];
      } else {
        long long m = (long long)((z >> 56) & 0xFFull) - 0x80ll;
        bits = __float_as_uint(ldexpf((float)m, -(7 + e))) >> 16;
        if (mode == 2 && (i % 8ull) == 0) bits = kSpecBF16[(i / 8ull) % 12ull];
      }
    }
    if (bf16) ((uint16_t *)dptr)[j] = (uint16_t)bits;
    else ((uint32_t *)dptr)[j] = bits;
  }
}

// Eq. 6 local fan-in reduce: out = ((in0 + in1) + ...) + in_{k-1}.
struct LocalReduceArgs {
  const uint4 *in[AR_MAX_RANKS];
  uint4 *out;
  unsigned long long nvec;
  int k;
};
template <bool BF16>
__global__ void __launch_bounds__(kThreads, 2) local_reduce_kernel(const __grid_constant__ LocalReduceArgs a) {
  __shared__ OpShared sh;
  if (threadIdx.x < a.k) sh.src[threadIdx.x] = a.in[threadIdx.x];
  if (threadIdx.x == 0) {
    sh.nsrc = a.k;
    sh.ndst = 1;
    sh.dst[0] = a.out;
    sh.div = 0;
  }
  __syncthreads();
  const size_t v0 = a.nvec * blockIdx.x / gridDim.x, v1 = a.nvec * (blockIdx.x + 1) / gridDim.x;
  body_dispatch<BF16>(sh, v0, v1);
}

// ------------------------------------------------------------------ host side
#define CUDA_OK(x)                                                                           \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) throw SysError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

struct SysError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

struct Registration {
  char *local = nullptr;
  size_t bytes = 0;
  std::vector<char *> peer;   // process -> mapped pointer (own = local)
  bool opened = false;
  cudaIpcMemHandle_t handle;  // of the allocation (ar_comm_open_peers matches its own blob by it)
  uint64_t offset = 0;
};

struct Lowered {
  DevStep *steps = nullptr;
  DevOp *ops = nullptr;
  DevWait *waits = nullptr;
  int *ranks = nullptr;
  int *prog_begin = nullptr;
  int *prog_len = nullptr;
  int nctas = 0;
  bool ll_shape = false;     // CPS-shaped: one all-rank reduce per block, identical input order
  std::vector<int> ll_order;
  unsigned int *dyn_ctr = nullptr;   // per-op tile counters (dynamic scheduling), nullptr = static
  int nops = 0;
};
// an emulated comm's multi-step plan for ar_flatsteps_kernel: every rank's ops grouped by step
struct FlatSteps {
  DevOp *ops = nullptr;
  int *ranks = nullptr;
  int *gbegin = nullptr;
  int nsteps = 0;
};

}  // namespace

struct ar_comm {
  int rank = 0, world = 0, device = 0;         // rank = first rank hosted by this process
  bool local = false;
  int rpp = 1;                                 // ranks hosted by this process (grid.y)
  int proc = 0, nproc = 1;                     // process index / count (multi-process comms)
  int nctas = 0, cta_cap = 0, max_ctas = 0;
  unsigned long long epoch = 0;
  size_t page_elems = 0;                       // uint64 per flag page
  unsigned long long *sig_local = nullptr;     // own page (multi) or all pages (local)
  std::vector<unsigned long long *> sig;       // rank -> page as seen here
  bool sig_opened = false;
  std::map<std::string, char *> ipc_opened;    // handle bytes -> base (opened once)
  std::vector<Registration> regs;
  std::map<uint64_t, Lowered> lowered;
  std::map<uint64_t, FlatSteps> flatsteps_cache;   // plan uid -> ar_flatsteps_kernel tables
  unsigned long long *err = nullptr;
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;
  int last_launches = 0;
  const char *last_kernel = "";                // kernel of the last allreduce_exec (ar_comm_last_kernel)
  bool bulk = true;                            // cp.async.bulk-staged body (AR_EXEC_BODY=regs: register body)
  // launch-argument cache for back-to-back calls with the same plan and buffer
  bool fast_valid = false;
  uint64_t fast_uid = 0;
  void *fast_dptr = nullptr;
  int fast_nctas = -1;
  ExecArgs fast_args{};
  int fence_mode = -1;                         // -1 = default (see ExecArgs::fence_mode); AR_FENCE_MODE
  bool store_tma = true;                       // bulk-copy stores of results (AR_EXEC_STORE=regs: st.global)
  int stages = kDefStages, stage_bytes = kDefStageBytes;   // AR_STAGES, AR_STAGE_KB
  unsigned int jitter_ns = 0;                  // AR_JITTER_NS (stress testing)
  bool plain_launch = false;                   // AR_LAUNCH=plain (see launch_exec)
  bool flat = true;                            // emulated single-step plans via ar_flat_kernel (AR_FLAT=0: off)
  bool dyn = true;                             // dynamic tile scheduling of CPS-shaped plans (AR_DYN=0: off)
  unsigned int *flat_ctr = nullptr;            // ar_flat_kernel tile counters (local comms)
  unsigned int *fs_bar = nullptr;              // ar_flatsteps_kernel grid-barrier words (local comms)
  // emulated multi-step plans via ar_flatsteps_kernel (AR_FLATSTEPS=1; off by default: measured
  // equal in bf16 and 10-14 % slower in fp32 than the step-table kernel, whose range waits let
  // dependent steps overlap CTA by CTA — profiles/round2/README.md §17)
  bool flatsteps = false;
  // low-latency one-shot path (ar_ll_kernel): scratch [parity][src][cap_lines] 16-byte lines
  long long ll_max_bytes = 0;                  // largest message sent this way (AR_LL_MAX_KB; 0 = off)
  long long ll_cap_lines = 0;
  // push protocol (lower_push) for CPS-shaped plans up to push_max_bytes (AR_PUSH_MAX_MB; 0 = off):
  // its scratch follows the LL region in the same allocation, [parity][src][push_slot]
  long long ll_region = 0, push_max_bytes = 0, push_slot = 0, push_plane = 0;
  std::map<uint64_t, Lowered> lowered_push;
  char *ll_scratch = nullptr;
  std::vector<char *> ll_peer;                 // rank -> scratch as seen here
  bool ll_opened = false;
  int ll_ctas = 32;
  // LL128 two-shot path (ar_ll128_kernel) for CPS-shaped plans (any count; its own block
  // partition), min(ll128_min_bytes, ll_max_bytes) < message <= ll128_max_bytes (AR_LL128_MIN_KB,
  // AR_LL128_MAX_KB; max 0 = off) — it takes such messages before the one-shot path; its
  // scratch follows the push planes: [parity][area][source][ll128_cap_lines] 128-byte lines
  long long ll128_min_bytes = 0, ll128_max_bytes = 0, ll128_cap_lines = 0, ll128_off = 0;
  int ll128_per_sm = 1;        // resident ar_ll128_kernel CTAs per SM
  int ll128_ctas = 296;
  std::map<uint64_t, std::vector<int>> ll_shape;   // plan uid -> summation order (empty: not CPS-shaped)
  // chunked end-to-end path (exec_host_chunked)
  cudaStream_t h2d = nullptr, d2h = nullptr;
  std::vector<cudaEvent_t> evs;
  std::map<std::pair<uint64_t, uint64_t>, gt_plan *> sub_plans;
  unsigned long long *trace = nullptr;         // in-kernel globaltimer stamps (ar_comm_set_trace)
  size_t trace_elems = 0;
  bool settings_fixed = false;                 // peers opened: the CTA count is agreed (Blob)
  char *checked_base = nullptr;                // local comms: last buffer extent validated
  size_t checked_need = 0;
  bool entry_fence = false;                    // AR_ENTRY_FENCE=1: fence.acq_rel.sys before relaxed entry flags
  ar_nvls *nvls = nullptr;                     // NVLS buffer for switch_reduce plans (ar_comm_attach_nvls)
};

namespace {

struct Blob {
  uint32_t magic, version;
  int32_t rank, world;
  uint64_t bytes, offset;
  cudaIpcMemHandle_t data, sig;
  cudaIpcMemHandle_t ll;      // low-latency scratch (valid iff has_ll)
  int32_t has_ll, pad;
  // settings every rank must share (checked by ar_comm_open_peers): the flag-page geometry,
  // the CTA count the range/paired waits are computed for, the one-shot scratch plane size and
  // the path cut-offs
  int32_t nctas, cta_cap, rpp, pad2;
  int64_t ll_cap_lines, ll_max_bytes, push_max_bytes, ll128_max_bytes;
  // same-process peers (several communicators in one process, e.g. one per rank on one GPU):
  // CUDA IPC handles cannot be opened by the exporting process, so the raw pointers are used
  int64_t pid;
  int32_t device, pad3;
  uint64_t raw_base, raw_sig, raw_ll;
  int64_t ll128_min_bytes;
};
static_assert(sizeof(Blob) <= AR_BLOB_BYTES, "blob too large");

typedef CUresult (*PFN_getAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);

static void base_of(void *p, char **base, size_t *size) {
  static PFN_getAddressRange fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void *f = nullptr;
    CUDA_OK(cudaGetDriverEntryPoint("cuMemGetAddressRange", &f, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !f) throw SysError("cuMemGetAddressRange unavailable");
    fn = (PFN_getAddressRange)f;
  }
  CUdeviceptr b;
  size_t s;
  if (fn(&b, &s, (CUdeviceptr)p) != CUDA_SUCCESS) throw InvalidArg("pointer is not device memory from cudaMalloc");
  *base = (char *)b;
  *size = s;
}

// ------------------------------------------------------------------ lowering
struct HostOp {
  long long off, len;
  std::vector<int> src, dst;
  bool fin = false;          // last RS op writing this region (reading AV1)
};
struct Access {
  int step, rank;              // executing rank
  long long off, len;
  bool write;
};

static bool overlap(long long a0, long long al, long long b0, long long bl) {
  return a0 < b0 + bl && b0 < a0 + al;
}

// Plan -> per-rank programs.  Ops of one rank and step are contiguous ranges; the final RS
// op of an owner is fused with the AG pushes of the same region in the next step when that
// creates no conflict inside the step.  Dependencies come from a conflict analysis of the
// buffer regions every op reads or writes (entry = every rank writes its own buffer before
// slot 0; exit = every rank overwrites its own buffer after the kernel).
static void lower_plan(const Plan &p, int world, std::vector<DevStep> &steps, std::vector<DevOp> &ops,
                       std::vector<DevWait> &waits, std::vector<int> &ranks, std::vector<int> &prog_begin,
                       std::vector<int> &prog_len) {
  const int n = p.n;
  const int S = (int)p.steps.size();
  if (S + 1 > kMaxSlots) throw InvalidArg("plan has too many steps");
  // ops[step][rank]
  std::vector<std::vector<std::vector<HostOp>>> H(S, std::vector<std::vector<HostOp>>(n));
  std::vector<int> last_rs(n, -1);   // block -> last RS step with a Reduce writing it
  for (int s = 0; s < S; s++)
    if (!p.steps[s].ag)
      for (auto &rd : p.steps[s].reduces) last_rs[rd.block] = s;
  for (int s = 0; s < S; s++) {
    const Step &st = p.steps[s];
    if (!st.ag) {
      std::vector<std::vector<const Reduce *>> by(n);
      for (auto &rd : st.reduces) by[rd.server].push_back(&rd);
      for (int r = 0; r < n; r++) {
        std::sort(by[r].begin(), by[r].end(), [](const Reduce *a, const Reduce *b) { return a->block < b->block; });
        for (const Reduce *rd : by[r]) {
          long long off = block_offset(p.count, n, rd->block), len = block_size(p.count, n, rd->block);
          if (len == 0) continue;
          auto &v = H[s][r];
          const bool fin = last_rs[rd->block] == s;
          if (!v.empty() && v.back().off + v.back().len == off && v.back().src == rd->inputs && v.back().fin == fin)
            v.back().len += len;
          else v.push_back({off, len, rd->inputs, {r}, fin});
        }
      }
    } else {
      std::vector<std::map<int, std::vector<int>>> by(n);   // src -> block -> dsts
      for (auto &t : st.transfers) by[t.src][t.block].push_back(t.dst);
      for (int r = 0; r < n; r++)
        for (auto &kv : by[r]) {
          std::vector<int> d = kv.second;
          std::sort(d.begin(), d.end());
          long long off = block_offset(p.count, n, kv.first), len = block_size(p.count, n, kv.first);
          if (len == 0) continue;
          auto &v = H[s][r];
          if (!v.empty() && v.back().off + v.back().len == off && v.back().dst == d) v.back().len += len;
          else v.push_back({off, len, {r}, d, false});
        }
    }
  }
  // conflict check inside one step (reads vs writes of different ops)
  auto step_conflict_free = [&](int s) {
    std::vector<std::pair<const HostOp *, int>> all;
    for (int r = 0; r < n; r++)
      for (auto &o : H[s][r]) all.push_back({&o, r});
    for (size_t i = 0; i < all.size(); i++)
      for (size_t j = 0; j < all.size(); j++) {
        if (i == j) continue;
        const HostOp &A = *all[i].first, &B = *all[j].first;
        if (!overlap(A.off, A.len, B.off, B.len)) continue;
        for (int w : A.dst) {
          for (int x : B.src)
            if (x == w) return false;
          for (int x : B.dst)
            if (x == w) return false;
        }
      }
    return true;
  };
  // fusion: RS op (dst = {r}) at s-1 + AG copy of the same region by r at s
  for (int s = 1; s < S; s++) {
    if (!p.steps[s].ag || p.steps[s - 1].ag) continue;
    auto saveA = H[s - 1];
    auto saveB = H[s];
    bool any = false;
    for (int r = 0; r < n; r++) {
      auto &ag = H[s][r];
      for (size_t i = 0; i < ag.size();) {
        bool fused = false;
        for (auto &x : H[s - 1][r])
          if (x.off == ag[i].off && x.len == ag[i].len && x.dst.size() == 1 && x.dst[0] == r && x.src.size() >= 2) {
            for (int d : ag[i].dst) x.dst.push_back(d);
            fused = true;
            break;
          }
        if (fused) { ag.erase(ag.begin() + i); any = true; }
        else i++;
      }
    }
    if (any && !step_conflict_free(s - 1)) {
      H[s - 1] = saveA;
      H[s] = saveB;
    }
  }
  // the kernel stages an op's source and destination lists in fixed arrays (OpShared)
  for (int s = 0; s < S; s++)
    for (int r = 0; r < n; r++)
      for (auto &o : H[s][r])
        if (o.src.empty() || (int)o.src.size() > AR_MAX_RANKS || (int)o.dst.size() > AR_MAX_RANKS)
          throw InvalidArg("plan op has more than AR_MAX_RANKS sources or destinations");
  // accesses per buffer rank
  std::vector<std::vector<Access>> acc(n);
  for (int s = 0; s < S; s++)
    for (int r = 0; r < n; r++)
      for (auto &o : H[s][r]) {
        for (int q : o.src) acc[q].push_back({s, r, o.off, o.len, false});
        for (int q : o.dst) acc[q].push_back({s, r, o.off, o.len, true});
      }
  // Waits of consumer (r, s): one entry per conflicting earlier producer op (rank t, step s',
  // range) — a *range* wait: the consumer CTA polls only the producer CTAs whose slice of
  // the producer op intersects its own slice of the consumer op (both sliced by the kernel's
  // rule), so dependent steps pipeline CTA by CTA.  Entry waits (t's input ready) are paired.
  using WaitKey = std::tuple<int, int, int, long long, long long, long long, long long>;
  // AR_WAITS=full: every inter-step dependency waits for all producer CTAs (no CTA-level
  // pipelining of dependent steps) — the A/B baseline for the range waits
  const char *wenv = std::getenv("AR_WAITS");
  const bool full_waits = wenv && std::string(wenv) == "full";
  std::vector<std::vector<std::set<WaitKey>>> wl(n, std::vector<std::set<WaitKey>>(S));
  std::vector<std::map<int, int>> exitdeps(n);
  for (int s = 0; s < S; s++)
    for (int r = 0; r < n; r++)
      for (auto &o : H[s][r]) {
        auto visit = [&](int q, bool write) {
          auto &d = wl[r][s];
          if (q != r) d.insert(WaitKey{q, 0, kWaitPaired, 0, 0, 0, 0});   // entry of q
          for (const Access &x : acc[q]) {
            if (x.step >= s) continue;
            if (!write && !x.write) continue;
            if (!overlap(o.off, o.len, x.off, x.len)) continue;
            if (full_waits) d.insert(WaitKey{x.rank, x.step + 1, kWaitFull, 0, 0, 0, 0});
            else d.insert(WaitKey{x.rank, x.step + 1, kWaitRange, x.off, x.len, o.off, o.len});
          }
        };
        for (int q : o.src) visit(q, false);
        for (int q : o.dst) visit(q, true);
      }
  for (int r = 0; r < n; r++)
    for (const Access &x : acc[r]) {
      if (x.rank == r) continue;
      auto it = exitdeps[r].find(x.rank);
      if (it == exitdeps[r].end() || it->second < x.step) exitdeps[r][x.rank] = x.step;
    }
  // notify lists: notify[t][slot] = consumers of t's step slot
  std::vector<std::vector<std::set<int>>> notify(n, std::vector<std::set<int>>(S + 1));
  for (int r = 0; r < n; r++) {
    for (int s = 0; s < S; s++)
      for (auto &w : wl[r][s]) notify[std::get<0>(w)][std::get<1>(w)].insert(r);
    for (auto &kv : exitdeps[r]) notify[kv.first][kv.second + 1].insert(r);
  }
  // programs
  prog_begin.assign(world, 0);
  prog_len.assign(world, 0);
  for (int r = 0; r < n; r++) {
    prog_begin[r] = (int)steps.size();
    auto emit = [&](int slot, const std::vector<HostOp> *hops, const std::set<WaitKey> *wk, const std::map<int, int> *dp,
                    bool exit) {
      DevStep d{};
      d.slot = slot;
      d.op_begin = (int)ops.size();
      if (hops)
        for (auto &o : *hops) {
          DevOp x{};
          x.off = o.off;
          x.len = o.len;
          x.nsrc = (int)o.src.size();
          x.ndst = (int)o.dst.size();
          x.fin = o.fin ? 1 : 0;
          x.src_begin = (int)ranks.size();
          ranks.insert(ranks.end(), o.src.begin(), o.src.end());
          x.dst_begin = (int)ranks.size();
          ranks.insert(ranks.end(), o.dst.begin(), o.dst.end());
          ops.push_back(x);
        }
      d.op_count = (int)ops.size() - d.op_begin;
      d.wait_begin = (int)waits.size();
      if (wk)
        for (auto &k : *wk) {
          DevWait w{};
          w.rank = std::get<0>(k);
          w.slot = std::get<1>(k);
          w.kind = std::get<2>(k);
          w.p_off = std::get<3>(k);
          w.p_len = std::get<4>(k);
          w.c_off = std::get<5>(k);
          w.c_len = std::get<6>(k);
          waits.push_back(w);
        }
      if (dp)
        for (auto &kv : *dp) {   // exit: paired waits on every remote accessor's last step
          DevWait w{};
          w.rank = kv.first;
          w.slot = kv.second + 1;
          w.kind = kWaitPaired;
          waits.push_back(w);
        }
      d.wait_count = (int)waits.size() - d.wait_begin;
      d.notify_begin = (int)ranks.size();
      if (!exit)
        for (int c : notify[r][slot]) ranks.push_back(c);
      d.notify_count = (int)ranks.size() - d.notify_begin;
      if (d.op_count || d.wait_count || d.notify_count) steps.push_back(d);
    };
    emit(0, nullptr, nullptr, nullptr, false);
    for (int s = 0; s < S; s++) {
      if (H[s][r].empty() && notify[r][s + 1].empty() && wl[r][s].empty()) continue;
      emit(s + 1, &H[s][r], &wl[r][s], nullptr, false);
    }
    emit(0, nullptr, nullptr, &exitdeps[r], true);
    prog_len[r] = (int)steps.size() - prog_begin[r];
  }
}

// Push protocol for CPS-shaped plans (see exec_impl): per rank three steps —
//   slot 1: copy block o of my buffer into owner o's scratch slot [parity][me], for every
//           o != me; notify every owner;
//   slot 2: (paired waits on every source's slot 1) reduce my block in the plan's order from
//           my buffer and the scratch slots, write it to every rank's buffer; notify all;
//   exit:   paired waits on every owner's slot 2 (its block landed in my buffer).
// No entry barrier: only the owner reads its own input, and a peer's scratch slot of parity
// p is rewritten only two calls later (see ar_ll_kernel's argument).  Same-index CTAs slice
// the same block range in both steps, so paired waits are exact.
static void lower_push(const Plan &p, const std::vector<int> &order, std::vector<DevStep> &steps,
                       std::vector<DevOp> &ops, std::vector<DevWait> &waits, std::vector<int> &ranks,
                       std::vector<int> &prog_begin, std::vector<int> &prog_len) {
  const int n = p.n;
  prog_begin.assign(n, 0);
  prog_len.assign(n, 0);
  auto scr = [](int owner, int src) { return kScrRef + owner * AR_MAX_RANKS + src; };
  for (int r = 0; r < n; r++) {
    prog_begin[r] = (int)steps.size();
    auto add_op = [&](long long off, long long len, const std::vector<int> &src, const std::vector<int> &dst,
                      int fin) {
      DevOp x{};
      x.off = off;
      x.len = len;
      x.nsrc = (int)src.size();
      x.ndst = (int)dst.size();
      x.src_begin = (int)ranks.size();
      ranks.insert(ranks.end(), src.begin(), src.end());
      x.dst_begin = (int)ranks.size();
      ranks.insert(ranks.end(), dst.begin(), dst.end());
      x.fin = fin;
      ops.push_back(x);
    };
    // slot 1: scatter my input blocks to their owners' scratch
    DevStep a{};
    a.slot = 1;
    a.op_begin = (int)ops.size();
    for (int o = 0; o < n; o++) {
      if (o == r) continue;
      const long long len = block_size(p.count, n, o);
      if (len > 0) add_op(block_offset(p.count, n, o), len, {r}, {scr(o, r)}, 0);
    }
    a.op_count = (int)ops.size() - a.op_begin;
    a.wait_begin = (int)waits.size();
    a.wait_count = 0;
    a.notify_begin = (int)ranks.size();
    for (int o = 0; o < n; o++)
      if (o != r) ranks.push_back(o);
    a.notify_count = (int)ranks.size() - a.notify_begin;
    steps.push_back(a);
    // slot 2: reduce my block, broadcast it
    DevStep b{};
    b.slot = 2;
    b.wait_begin = (int)waits.size();
    for (int s2 = 0; s2 < n; s2++) {
      if (s2 == r) continue;
      DevWait w{};
      w.rank = s2;
      w.slot = 1;
      w.kind = kWaitPaired;
      waits.push_back(w);
    }
    b.wait_count = (int)waits.size() - b.wait_begin;
    b.op_begin = (int)ops.size();
    const long long len = block_size(p.count, n, r);
    if (len > 0) {
      std::vector<int> src, dst{r};
      for (int q : order) src.push_back(q == r ? r : scr(r, q));
      for (int d = 0; d < n; d++)
        if (d != r) dst.push_back(d);
      add_op(block_offset(p.count, n, r), len, src, dst, 1);
    }
    b.op_count = (int)ops.size() - b.op_begin;
    b.notify_begin = (int)ranks.size();
    for (int d = 0; d < n; d++)
      if (d != r) ranks.push_back(d);
    b.notify_count = (int)ranks.size() - b.notify_begin;
    steps.push_back(b);
    // exit: every other block has landed
    DevStep e{};
    e.slot = 0;
    e.op_begin = (int)ops.size();
    e.wait_begin = (int)waits.size();
    for (int o = 0; o < n; o++) {
      if (o == r) continue;
      DevWait w{};
      w.rank = o;
      w.slot = 2;
      w.kind = kWaitPaired;
      waits.push_back(w);
    }
    e.wait_count = (int)waits.size() - e.wait_begin;
    e.notify_begin = (int)ranks.size();
    steps.push_back(e);
    prog_len[r] = (int)steps.size() - prog_begin[r];
  }
}

template <typename T>
static T *upload(const std::vector<T> &v) {
  T *d = nullptr;
  size_t bytes = std::max<size_t>(1, v.size()) * sizeof(T);
  CUDA_OK(cudaMalloc(&d, bytes));
  if (!v.empty()) CUDA_OK(cudaMemcpy(d, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

static void free_lowered(Lowered &L) {
  cudaFree(L.steps);
  cudaFree(L.ops);
  cudaFree(L.waits);
  cudaFree(L.ranks);
  cudaFree(L.prog_begin);
  cudaFree(L.prog_len);
  if (L.dyn_ctr) cudaFree(L.dyn_ctr);
}

static int resident_ctas(int device) {
  int nsm = 0, per = 0;
  CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device));
  CUDA_OK(cudaFuncSetAttribute(ar_exec_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  CUDA_OK(cudaFuncSetAttribute(ar_flat_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  CUDA_OK(cudaFuncSetAttribute(ar_flatsteps_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxDynSmem));
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ar_exec_kernel, kThreads, kMaxDynSmem));
  return nsm * std::max(per, 1);
}

#define SYS_TRY(...)                                          \
  try {                                                        \
    __VA_ARGS__                                                \
  } catch (const InvalidArg &e) {                              \
    set_error(e.what());                                       \
    return AR_EINVAL;                                          \
  } catch (const SysError &e) {                                \
    set_error(e.what());                                       \
    return AR_ESYS;                                            \
  } catch (const std::exception &e) {                          \
    set_error(std::string("internal error: ") + e.what());     \
    return AR_ESYS;                                            \
  }

constexpr long long kLLDefaultMaxBytes = 1536 * 1024;

// Default path cut-offs of a one-rank-per-GPU communicator of `world` ranks (bytes per rank),
// measured on 2 and 4 B200s (fp32 and bf16, graph timing; profiles/round2/README.md §12):
//  * one-shot path (ar_ll_kernel) up to 1.5 MiB/(N−1): it beats the flag protocol there
//    (~(N−1)·2S of line traffic against two flag round trips);
//  * the LL128 two-shot path (ar_ll128_kernel) takes CPS-shaped messages from 768 KiB/(N−1)
//    (at most 384 KiB) up to 64 MiB/N: above the floor it beats the one-shot path (N = 4, 512 KiB: 9.3 vs 13.6 us; N = 2, 1.5 MiB: 8.4 vs 17.5 us), and up to
//    the ceiling the step-table kernel (N = 2, 24-32 MiB: 564 vs 492-516 GB/s; N = 4, 32 MiB:
//    508 vs 554 — the ceiling falls with N).
static void default_paths(int world, long long *oneshot_max, long long *ll128_min, long long *ll128_max) {
  const long long w1 = std::max(1, world - 1);
  *oneshot_max = std::min<long long>(kLLDefaultMaxBytes, (3LL << 19) / w1) / 256 * 256;
  *ll128_min = std::min<long long>(*oneshot_max, std::min<long long>(384 << 10, (768LL << 10) / w1)) / 256 * 256;
  *ll128_max = std::max<long long>(1LL << 20, ((64LL << 20) / std::max(1, world)) >> 20 << 20);
}
// Off by default: measured slower than the pull protocol on 2 and 4 B200s (4 GPUs, 1 MiB:
// 27.7 vs 22.0 us; 16 MiB: 66.9 vs 55.4 us — the scatter step's per-block copies serialise
// load -> store -> completion per tile, and the owner cannot start before every source's
// scatter has landed).  Kept for A/B measurement behind AR_PUSH_MAX_MB.
constexpr long long kPushDefaultMaxBytes = 0;

static void init_comm(ar_comm *c) {
  CUDA_OK(cudaSetDevice(c->device));
  int nsm = 0;
  CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
  c->max_ctas = resident_ctas(c->device);
  if (c->rpp > 1) {   // emulated, or several ranks per process: the SMs are shared
    c->cta_cap = std::max(1, c->max_ctas / c->rpp);
    c->nctas = c->cta_cap;
  } else {
    c->cta_cap = kCtaCapMulti;
    c->nctas = std::min(nsm, kCtaCapMulti);
  }
  c->page_elems = (size_t)kMaxSlots * c->world * c->cta_cap;
  const size_t pages = c->rpp;
  CUDA_OK(cudaMalloc(&c->sig_local, pages * c->page_elems * sizeof(unsigned long long)));
  CUDA_OK(cudaMemset(c->sig_local, 0, pages * c->page_elems * sizeof(unsigned long long)));
  // device words: [0] error, [1] last completed epoch, [2] finished-CTA counter,
  // [3] last completed LL epoch, [4] LL finished-CTA counter, [5] LL128 epoch, [6] LL128 counter
  CUDA_OK(cudaMalloc(&c->err, 8 * sizeof(unsigned long long)));
  CUDA_OK(cudaMemset(c->err, 0, 8 * sizeof(unsigned long long)));
  if (c->local) {   // ar_flat_kernel's tile counters (dynamic scheduling)
    CUDA_OK(cudaMalloc(&c->flat_ctr, (AR_MAX_RANKS + 1) * sizeof(unsigned int)));
    CUDA_OK(cudaMemset(c->flat_ctr, 0, (AR_MAX_RANKS + 1) * sizeof(unsigned int)));
    CUDA_OK(cudaMalloc(&c->fs_bar, 2 * sizeof(unsigned int)));
    CUDA_OK(cudaMemset(c->fs_bar, 0, 2 * sizeof(unsigned int)));
  }
  c->sig.assign(c->world, nullptr);
  for (int i = 0; i < c->rpp; i++) c->sig[c->rank + i] = c->sig_local + (size_t)i * c->page_elems;
  if (c->local) c->sig_opened = true;
  if (const char *t = std::getenv("AR_FLAG_TIMEOUT_MS")) c->timeout_ns = std::strtoull(t, nullptr, 10) * 1000000ull;
  if (const char *b = std::getenv("AR_EXEC_BODY")) c->bulk = std::string(b) != "regs";
  if (const char *f = std::getenv("AR_FENCE_MODE")) c->fence_mode = std::atoi(f);
  if (const char *st = std::getenv("AR_EXEC_STORE")) c->store_tma = std::string(st) != "regs";
  // measured defaults (profiles/round1/stages): HBM-bound emulated ranks, dynamic tiles: 3 x 48
  // KB (713-718 GB/s busbw at 8 ranks x 256 MiB bf16; 2 x 40 KB 695, 2 x 64 / 3 x 56 KB 716,
  // 5-6 stages 700-703); with static slices a short 2 x 40 KB ring had been best; NVLink 3 x 40 KB
  if (c->local) {
    c->stages = 3;
    c->stage_bytes = 48 * 1024;
  } else {
    c->stages = 3;
    c->stage_bytes = 40 * 1024;
  }
  if (const char *v = std::getenv("AR_STAGES")) c->stages = std::max(2, std::min(kMaxStages, std::atoi(v)));
  if (const char *v = std::getenv("AR_STAGE_KB")) c->stage_bytes = std::max(4, std::atoi(v)) * 1024;
  while (dyn_smem_bytes(c->stages, c->stage_bytes) > kMaxDynSmem) c->stage_bytes -= 1024;
  if (const char *v = std::getenv("AR_JITTER_NS")) c->jitter_ns = (unsigned int)std::strtoul(v, nullptr, 10);
  if (const char *v = std::getenv("AR_LAUNCH")) c->plain_launch = std::string(v) == "plain";
  if (const char *v = std::getenv("AR_FLAT")) c->flat = std::string(v) != "0";
  if (const char *v = std::getenv("AR_FLATSTEPS")) c->flatsteps = std::string(v) == "1";
  if (const char *v = std::getenv("AR_DYN")) c->dyn = std::string(v) != "0";
  if (const char *v = std::getenv("AR_ENTRY_FENCE")) c->entry_fence = std::string(v) == "1";
  if (!c->local && c->rpp == 1) {
    c->push_max_bytes = kPushDefaultMaxBytes;
    if (const char *v = std::getenv("AR_PUSH_MAX_MB")) c->push_max_bytes = std::strtoll(v, nullptr, 10) << 20;
    // measured on 4 x B200 (profiles/README.md): the one-shot path costs ~(N-1)·2S of line
    // traffic per GPU; it beats the flag protocol up to ~768 KiB at N = 4 (13.6 vs 21.4 us at
    // 512 KiB, 25.2 vs 21.9 at 1 MiB), so the cut-off scales as 1.5 MiB / (N - 1)
    default_paths(c->world, &c->ll_max_bytes, &c->ll128_min_bytes, &c->ll128_max_bytes);
    if (const char *v = std::getenv("AR_LL_MAX_KB")) c->ll_max_bytes = std::strtoll(v, nullptr, 10) * 1024;
    c->ll_max_bytes = std::max(0LL, c->ll_max_bytes);
    c->push_max_bytes = std::max(0LL, c->push_max_bytes);
    if (const char *v = std::getenv("AR_LL128_MIN_KB")) c->ll128_min_bytes = std::strtoll(v, nullptr, 10) * 1024;
    c->ll128_min_bytes = std::max(0LL, c->ll128_min_bytes);
    if (const char *v = std::getenv("AR_LL128_MAX_KB")) c->ll128_max_bytes = std::strtoll(v, nullptr, 10) * 1024;
    c->ll128_max_bytes = std::max(0LL, c->ll128_max_bytes);
    if (c->ll_max_bytes > 0 || c->push_max_bytes > 0 || c->ll128_max_bytes > 0) {
      c->ll_cap_lines = (2 * c->ll_max_bytes + 7) / 8;   // room to raise the cut-off 2x (ar_comm_set_oneshot_max)
      c->ll_region = ((long long)2 * c->world * c->ll_cap_lines * 16 + 255) / 256 * 256;
      // one block of the largest pushed message + 16 bytes of alignment phase
      c->push_slot = ((c->push_max_bytes + c->world - 1) / c->world + 16 + 255) / 256 * 256;
      c->push_plane = c->push_slot * c->world;
      c->ll128_off = c->ll_region + (c->push_max_bytes > 0 ? 2 * c->push_plane : 0);
      // + 1: the last block of the LL128 partition carries up to 8N bytes more than max/N
      c->ll128_cap_lines = (c->ll128_max_bytes / c->world + kLinePayload - 1) / kLinePayload + 1;
      const size_t sz = (size_t)c->ll128_off + (size_t)4 * c->world * c->ll128_cap_lines * kLineBytes;
      CUDA_OK(cudaMalloc(&c->ll_scratch, sz));
      CUDA_OK(cudaMemset(c->ll_scratch, 0, sz));
      c->ll_peer.assign(c->world, nullptr);
      c->ll_peer[c->rank] = c->ll_scratch;
    }
  }
  if (const char *v = std::getenv("AR_LL_CTAS")) c->ll_ctas = std::max(1, std::atoi(v));
  // as many CTAs as are resident (3 per SM): measured best of 32 / 64 / 148 / 296 / 444 on 2 and
  // 4 B200s (profiles/round2/ll128; a variant batching the loads of the N-1 incoming lines
  // measured 0-6 % slower: not kept)
  {
    int per = 0, per2 = 0;
    int per3 = 0, per4 = 0;
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, ar_ll128_kernel<false, false>, kThreads, 0));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per2, ar_ll128_kernel<true, false>, kThreads, 0));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per3, ar_ll128_kernel<false, true>, kThreads, 0));
    CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per4, ar_ll128_kernel<true, true>, kThreads, 0));
    c->ll128_per_sm = std::max(1, std::min(std::min(per, per2), std::min(per3, per4)));
  }
  c->ll128_ctas = c->ll128_per_sm * nsm;   // 3 per SM: equal to 2 up to 8 MiB, +1-11 % at 16-32 MiB
  if (const char *v = std::getenv("AR_LL128_CTAS")) c->ll128_ctas = std::max(1, std::atoi(v));
}

}  // namespace

extern "C" {

uint64_t ar_rank_stride_bytes(uint64_t count, int32_t dtype) {
  uint64_t b = count * (uint64_t)(dtype == AR_BF16 ? 2 : 4);
  static const uint64_t pad = [] {   // experiment knob: extra bytes between emulated ranks
    const char *e = std::getenv("AR_EMU_STRIDE_PAD");
    return e ? (std::strtoull(e, nullptr, 10) + 255) / 256 * 256 : 0ull;
  }();
  return (b + 255) / 256 * 256 + pad;
}

int ar_comm_create(int32_t rank, int32_t world, int32_t cuda_device, ar_comm **out) {
  return ar_comm_create_multi(rank, world, 1, cuda_device, out);
}

int ar_comm_create_multi(int32_t proc, int32_t nproc, int32_t ranks_per_proc, int32_t cuda_device, ar_comm **out) {
  SYS_TRY({
    if (!out) throw InvalidArg("null out");
    const long long world = (long long)nproc * ranks_per_proc;
    if (nproc < 1 || ranks_per_proc < 1 || world < 2 || world > AR_MAX_RANKS || proc < 0 || proc >= nproc)
      throw InvalidArg("bad proc/nproc/ranks_per_proc");
    if (nproc == 1) throw InvalidArg("one process: use ar_comm_create_local");
    ar_comm *c = new ar_comm();
    c->rank = proc * ranks_per_proc;
    c->world = (int)world;
    c->rpp = ranks_per_proc;
    c->proc = proc;
    c->nproc = nproc;
    c->device = cuda_device;
    try {
      init_comm(c);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
    return AR_OK;
  })
}

int ar_comm_create_local(int32_t world, int32_t cuda_device, ar_comm **out) {
  SYS_TRY({
    if (!out) throw InvalidArg("null out");
    if (world < 2 || world > AR_MAX_RANKS) throw InvalidArg("bad world");
    ar_comm *c = new ar_comm();
    c->rank = 0;
    c->world = world;
    c->rpp = world;
    c->device = cuda_device;
    c->local = true;
    try {
      init_comm(c);
    } catch (...) {
      delete c;
      throw;
    }
    if (c->cta_cap < 1 || c->max_ctas < world) {
      delete c;
      throw InvalidArg("too many emulated ranks for one device");
    }
    *out = c;
    return AR_OK;
  })
}

int ar_comm_set_ctas(ar_comm *c, int32_t ctas) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    int want = ctas > 0 ? ctas : (c->rpp > 1 ? c->cta_cap : std::min(c->max_ctas, kCtaCapMulti));
    if (want > c->cta_cap) throw InvalidArg("ctas exceeds the flag page capacity");
    if ((long long)want * c->rpp > c->max_ctas) throw InvalidArg("ctas exceeds resident capacity");
    if (ctas <= 0 && c->rpp == 1) {
      int nsm = 0;
      CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, c->device));
      want = std::min(nsm, kCtaCapMulti);
    }
    if (c->settings_fixed && want != c->nctas)
      throw InvalidArg("ar_comm_set_ctas after ar_comm_open_peers: the peers' waits are computed for the agreed "
                       "CTA count; set it before ar_comm_register on every rank");
    c->nctas = want;
    return AR_OK;
  })
}

int ar_comm_register(ar_comm *c, void *dptr, size_t bytes, void *blob_out) {
  SYS_TRY({
    if (!c || !dptr || !blob_out) throw InvalidArg("null argument");
    if (c->local) throw InvalidArg("emulated communicators need no registration");
    if ((uintptr_t)dptr % 16) throw InvalidArg("buffer must be 16-byte aligned");
    CUDA_OK(cudaSetDevice(c->device));
    char *base;
    size_t size;
    base_of(dptr, &base, &size);
    if ((char *)dptr + bytes > base + size) throw InvalidArg("buffer extends past its allocation");
    Blob b;
    std::memset(&b, 0, sizeof b);
    b.magic = kBlobMagic;
    b.version = 2;
    b.rank = c->proc;
    b.world = c->world;
    b.bytes = bytes;
    b.offset = (uint64_t)((char *)dptr - base);
    CUDA_OK(cudaIpcGetMemHandle(&b.data, base));
    CUDA_OK(cudaIpcGetMemHandle(&b.sig, c->sig_local));
    if (c->ll_scratch) {
      CUDA_OK(cudaIpcGetMemHandle(&b.ll, c->ll_scratch));
      b.has_ll = 1;
    }
    b.nctas = c->nctas;
    b.cta_cap = c->cta_cap;
    b.rpp = c->rpp;
    b.ll_cap_lines = c->ll_cap_lines;
    b.ll_max_bytes = c->ll_max_bytes;
    b.push_max_bytes = c->push_max_bytes;
    b.ll128_max_bytes = c->ll128_max_bytes;
    b.ll128_min_bytes = c->ll128_min_bytes;
    b.pid = (int64_t)getpid();
    b.device = c->device;
    b.raw_base = (uint64_t)(uintptr_t)base;
    b.raw_sig = (uint64_t)(uintptr_t)c->sig_local;
    b.raw_ll = (uint64_t)(uintptr_t)c->ll_scratch;
    std::memset(blob_out, 0, AR_BLOB_BYTES);
    std::memcpy(blob_out, &b, sizeof b);
    Registration reg;
    reg.local = (char *)dptr;
    reg.bytes = bytes;
    reg.peer.assign(c->nproc, nullptr);
    reg.peer[c->proc] = (char *)dptr;
    reg.handle = b.data;
    reg.offset = b.offset;
    for (auto it = c->regs.begin(); it != c->regs.end(); ++it)
      if (it->local == reg.local) { c->regs.erase(it); break; }
    c->regs.push_back(reg);
    c->fast_valid = false;
    return AR_OK;
  })
}

int ar_comm_open_peers(ar_comm *c, const void *blobs) {
  SYS_TRY({
    if (!c || !blobs) throw InvalidArg("null argument");
    if (c->local) throw InvalidArg("emulated communicators need no peers");
    CUDA_OK(cudaSetDevice(c->device));
    const char *bb = (const char *)blobs;
    const Blob *mine = (const Blob *)(bb + (size_t)c->proc * AR_BLOB_BYTES);
    if (mine->magic != kBlobMagic || mine->version != 2 || mine->rank != c->proc) throw InvalidArg("corrupt or misordered blob");
    // this process's registration of the buffer the blobs describe: same allocation, offset, size
    Registration *reg = nullptr;
    for (auto it = c->regs.rbegin(); it != c->regs.rend(); ++it)
      if ((uint64_t)it->bytes == mine->bytes && it->offset == mine->offset &&
          std::memcmp(&it->handle, &mine->data, sizeof(cudaIpcMemHandle_t)) == 0) {
        reg = &*it;
        break;
      }
    if (!reg) throw InvalidArg("no local registration matches this process's blob");
    const int64_t me_pid = (int64_t)getpid();
    for (int t = 0; t < c->nproc; t++) {   // one blob per process
      const Blob *b = (const Blob *)(bb + (size_t)t * AR_BLOB_BYTES);
      if (b->magic != kBlobMagic || b->version != 2 || b->world != c->world || b->rank != t)
        throw InvalidArg("corrupt or misordered blob");
      if (b->bytes != mine->bytes) throw InvalidArg("ranks registered buffers of different sizes");
      if (b->nctas != c->nctas || b->cta_cap != c->cta_cap || b->rpp != c->rpp || b->ll_cap_lines != c->ll_cap_lines ||
          b->ll_max_bytes != mine->ll_max_bytes || b->push_max_bytes != c->push_max_bytes ||
          b->ll128_max_bytes != c->ll128_max_bytes || b->ll128_min_bytes != c->ll128_min_bytes)
        throw InvalidArg("ranks disagree on communicator settings (ar_comm_set_ctas, AR_LL_MAX_KB, "
                         "AR_LL128_MIN_KB, AR_LL128_MAX_KB, AR_PUSH_MAX_MB or the one-shot cut-off must be identical on every rank)");
      if (t == c->proc) continue;
      const bool same_proc = b->pid == me_pid;
      if (same_proc && b->device != c->device) {
        // a communicator of this process on another GPU: direct peer access instead of IPC
        cudaError_t e = cudaDeviceEnablePeerAccess(b->device, 0);
        if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
        else CUDA_OK(e);
      }
      auto open = [&](const cudaIpcMemHandle_t &h, uint64_t raw) -> char * {
        if (same_proc) return (char *)(uintptr_t)raw;   // IPC handles cannot be opened by their exporter
        std::string key((const char *)&h, sizeof h);
        key += std::to_string(t);
        auto it = c->ipc_opened.find(key);
        if (it != c->ipc_opened.end()) return it->second;
        void *p = nullptr;
        CUDA_OK(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
        c->ipc_opened[key] = (char *)p;
        return (char *)p;
      };
      reg->peer[t] = open(b->data, b->raw_base) + b->offset;
      if (c->ll_scratch && b->has_ll && !c->ll_peer[t]) c->ll_peer[t] = open(b->ll, b->raw_ll);
      unsigned long long *pages = nullptr;
      for (int i = 0; i < c->rpp; i++)
        if (!c->sig[t * c->rpp + i]) {
          if (!pages) pages = (unsigned long long *)open(b->sig, b->raw_sig);
          c->sig[t * c->rpp + i] = pages + (size_t)i * c->page_elems;
        }
    }
    c->settings_fixed = true;
    reg->opened = true;
    c->fast_valid = false;
    c->sig_opened = true;
    if (c->ll_scratch) {
      bool all = true;
      for (int t = 0; t < c->world; t++) all = all && c->ll_peer[t] != nullptr;
      c->ll_opened = all;
    }
    return AR_OK;
  })
}

int ar_comm_get_async_error(ar_comm *c) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaDeviceSynchronize());
    unsigned long long e = 0;
    CUDA_OK(cudaMemcpy(&e, c->err, sizeof e, cudaMemcpyDeviceToHost));
    if (e) {
      CUDA_OK(cudaMemset(c->err, 0, sizeof e));
      throw SysError("flag wait timed out on the device (peer not progressing)");
    }
    unsigned long long pe = 0;
    CUDA_OK(cudaMemcpyFromSymbol(&pe, g_pipe_err, sizeof pe));
    if (pe) {
      const unsigned long long z = 0;
      CUDA_OK(cudaMemcpyToSymbol(g_pipe_err, &z, sizeof z));
      throw SysError("bulk-copy pipeline wait timed out on the device (internal error)");
    }
    return AR_OK;
  })
}

int ar_comm_destroy(ar_comm *c) {
  if (!c) return AR_OK;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto &kv : c->lowered) free_lowered(kv.second);
  for (auto &kv : c->lowered_push) free_lowered(kv.second);
  for (auto &kv : c->sub_plans) delete kv.second;
  for (cudaEvent_t e : c->evs) cudaEventDestroy(e);
  if (c->h2d) cudaStreamDestroy(c->h2d);
  if (c->d2h) cudaStreamDestroy(c->d2h);
  for (auto &kv : c->ipc_opened) cudaIpcCloseMemHandle(kv.second);
  cudaFree(c->sig_local);
  cudaFree(c->ll_scratch);
  cudaFree(c->err);
  if (c->flat_ctr) cudaFree(c->flat_ctr);
  if (c->fs_bar) cudaFree(c->fs_bar);
  for (auto &kv : c->flatsteps_cache) {
    cudaFree(kv.second.ops);
    cudaFree(kv.second.ranks);
    cudaFree(kv.second.gbegin);
  }
  cudaFree(c->trace);
  delete c;
  return AR_OK;
}

const char *ar_comm_last_kernel(ar_comm *c) { return c ? c->last_kernel : ""; }

int ar_comm_attach_nvls(ar_comm *c, ar_nvls *nvls) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    if (c->local || c->rpp != 1) throw InvalidArg("NVLS needs one rank per GPU");
    c->nvls = nvls;
    return AR_OK;
  })
}

int ar_default_paths(int32_t world, uint64_t *oneshot_max_bytes, uint64_t *ll128_min_bytes, uint64_t *ll128_max_bytes) {
  if (world < 2 || world > AR_MAX_RANKS) {
    set_error("world must be in [2, AR_MAX_RANKS]");
    return AR_EINVAL;
  }
  long long a, b, c;
  default_paths(world, &a, &b, &c);
  if (oneshot_max_bytes) *oneshot_max_bytes = (uint64_t)a;
  if (ll128_min_bytes) *ll128_min_bytes = (uint64_t)b;
  if (ll128_max_bytes) *ll128_max_bytes = (uint64_t)c;
  return AR_OK;
}

int ar_comm_get_paths(ar_comm *c, uint64_t *oneshot_max_bytes, uint64_t *ll128_min_bytes, uint64_t *ll128_max_bytes) {
  if (!c) {
    set_error("null comm");
    return AR_EINVAL;
  }
  const bool on = c->ll_scratch != nullptr;   // emulated / several ranks per GPU: neither path
  if (oneshot_max_bytes) *oneshot_max_bytes = on ? (uint64_t)c->ll_max_bytes : 0;
  if (ll128_min_bytes) *ll128_min_bytes = on ? (uint64_t)std::min(c->ll128_min_bytes, c->ll_max_bytes) : 0;
  if (ll128_max_bytes) *ll128_max_bytes = on && c->world <= 8 ? (uint64_t)c->ll128_max_bytes : 0;
  return AR_OK;
}

int ar_comm_set_oneshot_max(ar_comm *c, uint64_t bytes) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    if (!c->ll_scratch && bytes > 0) throw InvalidArg("this communicator has no one-shot scratch");
    if ((long long)bytes > c->ll_cap_lines * 8) throw InvalidArg("above the scratch capacity (AR_LL_MAX_KB at creation)");
    c->ll_max_bytes = (long long)bytes;
    return AR_OK;
  })
}

int ar_comm_last_launch_count(ar_comm *c, int32_t *kernels) {
  if (!c || !kernels) { set_error("null argument"); return AR_EINVAL; }
  *kernels = c->last_launches;
  return AR_OK;
}

// GenModel of the executed plan (reading A6x): the per-step formula
// applied to the lowered programs — the entry flag round, then every slot in which some rank
// runs ops.  shared = all ranks on one GPU (reading A6e): a slot costs the memory traffic of
// all ranks together (D = Σ (sources + destinations)·len, C = Σ (k − 1)·len), no link term.
static Breakdown predict_executed_impl(const gt_plan *plan, const gm_params *params, bool shared) {
  if (plan->plan.switch_reduce) {   // NVLS: its closed-form row (reading NV1)
    if (shared) throw InvalidArg("an NVLS plan cannot run on ranks sharing one GPU");
    Params q;
    q.alpha = params->alpha; q.beta = params->beta; q.gamma = params->gamma; q.delta = params->delta;
    q.epsilon = params->epsilon; q.w_t = params->w_t; q.has_combined = params->has_combined != 0;
    q.combined = params->combined;
    return closed_form_f64("nvls", plan->plan.n, plan->plan.count * (int64_t)plan->esize, q, {});
  }
  std::vector<DevStep> st;
  std::vector<DevOp> ops;
  std::vector<DevWait> w;
  std::vector<int> rk, pb, pl;
  const int n = plan->plan.n;
  lower_plan(plan->plan, n, st, ops, w, rk, pb, pl);
  const int64_t es = plan->esize;
  // per executed slot: in/out bytes per rank (full duplex), reduce work, distinct peers
  std::map<int, std::vector<int64_t>> in, outb, cc, dd;
  std::map<int, std::vector<std::set<int>>> peers;
  for (int r = 0; r < n; r++)
    for (int i = 0; i < pl[r]; i++) {
      const DevStep &d = st[pb[r] + i];
      if (d.op_count == 0) continue;
      const int s = d.slot;
      if (!in.count(s)) {
        in[s].assign(n, 0); outb[s].assign(n, 0); cc[s].assign(n, 0); dd[s].assign(n, 0);
        peers[s].assign(n, std::set<int>());
      }
      for (int k = 0; k < d.op_count; k++) {
        const DevOp &x = ops[d.op_begin + k];
        const int64_t L = x.len * es;
        for (int j = 0; j < x.nsrc; j++) {
          const int q = rk[x.src_begin + j];
          if (q == r) continue;
          in[s][r] += L;
          outb[s][q] += L;
          peers[s][r].insert(q);
        }
        for (int j = 0; j < x.ndst; j++) {
          const int q = rk[x.dst_begin + j];
          if (q == r) continue;
          outb[s][r] += L;
          in[s][q] += L;
          peers[s][q].insert(r);
        }
        if (x.nsrc >= 2) cc[s][r] += (x.nsrc - 1) * L;
        if (shared) dd[s][r] += (x.nsrc + x.ndst) * L;
        else if (x.nsrc >= 2) dd[s][r] += (x.nsrc + 1) * L;
      }
    }
  std::vector<StepCoeffs> co;
  co.push_back(StepCoeffs{1, 0, 0, 0, 1});   // the entry flag round (one alpha)
  for (auto &kv : in) {
    const int s = kv.first;
    StepCoeffs c{1, 0, 0, 0, 1};
    for (int r = 0; r < n; r++) {
      if (shared) {
        c.C += cc[s][r];
        c.D += dd[s][r];
        continue;
      }
      c.B = std::max(c.B, std::max(in[s][r], outb[s][r]));
      c.C = std::max(c.C, cc[s][r]);
      c.D = std::max(c.D, dd[s][r]);
      c.w = std::max(c.w, 1 + (int)peers[s][r].size());
    }
    co.push_back(c);
  }
  Params p;
  p.alpha = params->alpha; p.beta = params->beta; p.gamma = params->gamma; p.delta = params->delta;
  p.epsilon = params->epsilon; p.w_t = params->w_t; p.has_combined = params->has_combined != 0;
  p.combined = params->combined;
  return predict_f64(co, uniform_step_params(p, co.size()));
}

static void fill_breakdown(gm_breakdown *out, const Breakdown &b) {
  out->latency = b.latency; out->bandwidth = b.bandwidth; out->compute = b.compute;
  out->memory = b.memory; out->incast = b.incast; out->total = b.total;
}

int genmodel_predict_executed(const gt_plan *plan, const gm_params *params, gm_breakdown *out) {
  SYS_TRY({
    if (!plan || !params || !out) throw InvalidArg("null argument");
    fill_breakdown(out, predict_executed_impl(plan, params, false));
    return AR_OK;
  })
}

int genmodel_predict_executed_shared(const gt_plan *plan, const gm_params *params, gm_breakdown *out) {
  SYS_TRY({
    if (!plan || !params || !out) throw InvalidArg("null argument");
    fill_breakdown(out, predict_executed_impl(plan, params, true));
    return AR_OK;
  })
}

int ar_comm_set_trace(ar_comm *c, int32_t enable) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    CUDA_OK(cudaSetDevice(c->device));
    if (c->trace) {
      CUDA_OK(cudaDeviceSynchronize());
      cudaFree(c->trace);
      c->trace = nullptr;
      c->trace_elems = 0;
    }
    if (enable) {
      c->trace_elems = (size_t)c->rpp * c->cta_cap * kTraceSlots;
      CUDA_OK(cudaMalloc(&c->trace, c->trace_elems * sizeof(unsigned long long)));
      CUDA_OK(cudaMemset(c->trace, 0, c->trace_elems * sizeof(unsigned long long)));
    }
    c->fast_valid = false;
    return AR_OK;
  })
}

int ar_comm_read_trace(ar_comm *c, uint64_t *out, size_t cap, size_t *n, int32_t *slots_per_cta,
                       int32_t *ctas_per_rank) {
  SYS_TRY({
    if (!c) throw InvalidArg("null comm");
    if (!c->trace) throw InvalidArg("tracing is off (ar_comm_set_trace)");
    const size_t used = (size_t)c->rpp * c->cta_cap * kTraceSlots;
    if (n) *n = used;
    if (slots_per_cta) *slots_per_cta = kTraceSlots;
    if (ctas_per_rank) *ctas_per_rank = c->cta_cap;
    if (!out || cap < used) throw InvalidArg("buffer too small");
    CUDA_OK(cudaSetDevice(c->device));
    CUDA_OK(cudaDeviceSynchronize());
    CUDA_OK(cudaMemcpy(out, c->trace, used * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    return AR_OK;
  })
}

int ar_plan_lowering_json(const gt_plan *plan, char *buf, size_t cap, size_t *needed) {
  SYS_TRY({
    if (!plan) throw InvalidArg("null plan");
    if (plan->plan.switch_reduce) throw InvalidArg("an NVLS plan has no step tables (the switch reduces)");
    std::vector<DevStep> st;
    std::vector<DevOp> ops;
    std::vector<DevWait> w;
    std::vector<int> rk, pb, pl;
    lower_plan(plan->plan, plan->plan.n, st, ops, w, rk, pb, pl);
    std::string o = "{\"ranks\":[";
    for (int r = 0; r < plan->plan.n; r++) {
      o += r ? ",{\"steps\":[" : "{\"steps\":[";
      for (int i = 0; i < pl[r]; i++) {
        const DevStep &d = st[pb[r] + i];
        o += i ? "," : "";
        o += "{\"slot\":" + std::to_string(d.slot) + ",\"ops\":[";
        for (int k = 0; k < d.op_count; k++) {
          const DevOp &x = ops[d.op_begin + k];
          o += k ? "," : "";
          o += "{\"off\":" + std::to_string(x.off) + ",\"len\":" + std::to_string(x.len) + ",\"src\":[";
          for (int j = 0; j < x.nsrc; j++) o += (j ? "," : "") + std::to_string(rk[x.src_begin + j]);
          o += "],\"dst\":[";
          for (int j = 0; j < x.ndst; j++) o += (j ? "," : "") + std::to_string(rk[x.dst_begin + j]);
          o += "],\"fin\":" + std::to_string(x.fin) + "}";
        }
        o += "],\"waits\":[";
        for (int k = 0; k < d.wait_count; k++) {
          const DevWait &x = w[d.wait_begin + k];
          o += (k ? ",[" : "[") + std::to_string(x.rank) + "," + std::to_string(x.slot) + "," +
               std::to_string(x.kind) + "," + std::to_string(x.p_off) + "," + std::to_string(x.p_len) + "," +
               std::to_string(x.c_off) + "," + std::to_string(x.c_len) + "]";
        }
        o += "],\"notify\":[";
        for (int k = 0; k < d.notify_count; k++) o += (k ? "," : "") + std::to_string(rk[d.notify_begin + k]);
        o += "]}";
      }
      o += "]}";
    }
    o += "]}";
    if (needed) *needed = o.size() + 1;
    if (!buf || cap < o.size() + 1) throw InvalidArg("buffer too small");
    std::memcpy(buf, o.c_str(), o.size() + 1);
    return AR_OK;
  })
}

// Cooperative launch guarantees the co-residency the intra-GPU CTA waits need; a plain launch
// of the same grid (1 CTA per SM, grid <= resident capacity) is co-resident whenever the GPU
// is otherwise idle — AR_LAUNCH=plain selects it for latency measurements.
static void launch_exec(ar_comm *c, dim3 grid, void **args, cudaStream_t stream) {
  const size_t smem = c->bulk ? dyn_smem_bytes(c->stages, c->stage_bytes) : 0;
  if (c->plain_launch) {
    CUDA_OK(cudaLaunchKernel((const void *)ar_exec_kernel, grid, dim3(kThreads), args, smem, stream));
  } else {
    CUDA_OK(cudaLaunchCooperativeKernel((const void *)ar_exec_kernel, grid, dim3(kThreads), args, smem, stream));
  }
}

// stride_override: bytes between consecutive hosted ranks' buffers when dptr points into the
// middle of larger rank buffers (the chunked end-to-end path); 0 = derived from count.
static void check_local_extent(ar_comm *c, void *dptr, size_t need) {
  // emulated comm: dptr is the base of world rank buffers; the whole extent must be one
  // allocation.  One rank per GPU: the flag-free paths (one-shot, LL128) write only this
  // rank's buffer and the communicator's scratch, so they need no registration, but the
  // buffer must hold count elements (cached: the last checked pointer and extent)
  if ((char *)dptr == c->checked_base && need <= c->checked_need) return;
  char *base;
  size_t size;
  if (c->local) {
    base_of(dptr, &base, &size);
  } else {
    try {
      base_of(dptr, &base, &size);
    } catch (const std::exception &) {
      return;   // not a driver allocation it can size (e.g. a virtual-memory mapping): unchecked
    }
  }
  if ((char *)dptr + need > base + size)
    throw InvalidArg(c->local ? "buffer too small: an emulated communicator needs world rank buffers at "
                                "ar_rank_stride_bytes"
                              : "buffer too small: it must hold count elements of dtype");
  c->checked_base = (char *)dptr;
  c->checked_need = need;
}

static int exec_impl(const gt_plan *plan, ar_comm *c, void *dptr, uint64_t count, int32_t dtype, void *stream,
                     int op = AR_OP_SUM, uint64_t stride_override = 0, bool movement = false) {
  if (!plan || !c || !dptr) throw InvalidArg("null argument");
  if (!plan->is_allreduce && !movement)
    throw InvalidArg("plan is not an AllReduce (failed symbolic verification); data-movement plans run through "
                     "ar_exec_movement_plan");
  if (plan->plan.switch_reduce) {
    // NVLS plan kind: the fan-in-N reduce and the broadcast happen in the NVSwitch
    if (op != AR_OP_SUM && op != AR_OP_AVG) throw InvalidArg("unknown reduction op");
    if (!c->nvls) throw InvalidArg("NVLS plan: attach the NVLS buffer first (ar_comm_attach_nvls)");
    if (plan->plan.n != c->world) throw InvalidArg("plan and communicator have different world sizes");
    if ((uint64_t)plan->plan.count != count || plan->dtype != dtype) throw InvalidArg("count/dtype differ from the plan's");
    nvls_launch(c->nvls, dptr, count, dtype, stream, op == AR_OP_AVG ? plan->plan.n : 0);
    c->last_launches = 1;
    c->last_kernel = "nvls_kernel";
    return AR_OK;
  }
  if (op != AR_OP_SUM && op != AR_OP_AVG) throw InvalidArg("unknown reduction op");
  const int avg_n = op == AR_OP_AVG ? plan->plan.n : 0;
  if (plan->plan.n != c->world) throw InvalidArg("plan and communicator have different world sizes");
  if ((uint64_t)plan->plan.count != count || plan->dtype != dtype) throw InvalidArg("count/dtype differ from the plan's");
  if ((uintptr_t)dptr % 16) throw InvalidArg("buffer must be 16-byte aligned");
  int cur = -1;
  CUDA_OK(cudaGetDevice(&cur));
  if (cur != c->device) CUDA_OK(cudaSetDevice(c->device));
  dim3 grid(c->nctas, c->rpp);
  const size_t nbytes_call = count * (size_t)plan->esize;
  if (c->local)
    check_local_extent(c, dptr,
                       (stride_override ? stride_override : ar_rank_stride_bytes(count, dtype)) * (c->world - 1) +
                           nbytes_call);
  if (!c->local && c->ll_opened) check_local_extent(c, dptr, nbytes_call);   // flag-free paths below
  if (c->ll_opened && c->ll128_max_bytes > 0 && c->world <= 8 &&
      (long long)nbytes_call > std::min(c->ll128_min_bytes, c->ll_max_bytes) &&
      (long long)nbytes_call <= c->ll128_max_bytes && nbytes_call >= 8ull * c->world && (uintptr_t)dptr % 8 == 0) {
    // LL128 two-shot path for CPS-shaped plans (ar_ll128_kernel), any count: blocks of its own
    // partition (8-byte multiples, the remainder on the last block; the plan's bits do not depend
    // on the partition because every block sums its elements in the same order)
    auto lit = c->ll_shape.find(plan->uid);
    if (lit == c->ll_shape.end()) lit = c->ll_shape.emplace(plan->uid, oneshot_order(plan->plan)).first;
    if (!lit->second.empty()) {
      LL128Args la{};
      la.buf = (char *)dptr;
      for (int t = 0; t < c->world; t++) la.peer_scr[t] = c->ll_peer[t] + c->ll128_off;
      la.my_scr = c->ll_scratch + c->ll128_off;
      for (int k = 0; k < c->world; k++) la.order[k] = lit->second[k];
      const long long unit = 8 / plan->esize;   // elements per 8-byte word
      const long long blk = (long long)(count / c->world) / unit * unit;
      la.blk_bytes = blk * plan->esize;
      la.lines = (la.blk_bytes + kLinePayload - 1) / kLinePayload;
      la.last_bytes = ((long long)count - (long long)(c->world - 1) * blk) * plan->esize;
      la.last_lines = (la.last_bytes + kLinePayload - 1) / kLinePayload;
      la.lines_cap = c->ll128_cap_lines;
      if (la.last_lines > la.lines_cap) throw SysError("LL128 scratch too small (internal error)");
      la.me = c->rank;
      la.world = c->world;
      la.esize = plan->esize;
      la.avg_n = avg_n;
      la.epoch_dev = c->err + 5;
      la.done_ctr = (unsigned int *)(c->err + 6);
      la.err = c->err;
      la.timeout_ns = c->timeout_ns;
      const long long warps_needed = (la.last_lines + 3) / 4;
      // every CTA of every rank must be resident at once (a resident CTA may wait for lines a
      // not-yet-scheduled CTA of a peer would write): at most the kernel's occupancy per SM times
      // the caller's share of the GPU (ar_comm_set_ctas; several ranks' comms on one GPU)
      const long long cap = std::min<long long>(c->ll128_ctas, (long long)c->ll128_per_sm * c->nctas);
      const int ctas = (int)std::max(1LL, std::min<long long>(cap, (warps_needed + 15) / 16));
      const bool ragged = la.last_bytes != la.blk_bytes;
      if (plan->esize == 2) {
        if (ragged) ar_ll128_kernel<true, true><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(la);
        else ar_ll128_kernel<true, false><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(la);
      } else {
        if (ragged) ar_ll128_kernel<false, true><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(la);
        else ar_ll128_kernel<false, false><<<ctas, kThreads, 0, (cudaStream_t)stream>>>(la);
      }
      CUDA_OK(cudaGetLastError());
      c->last_launches = 1;
      c->last_kernel = "ar_ll128_kernel";
      return AR_OK;
    }
  }
  if (c->ll_opened && (long long)nbytes_call <= c->ll_max_bytes) {
    // low-latency one-shot path for CPS-shaped plans (see ar_ll_kernel)
    auto lit = c->ll_shape.find(plan->uid);
    if (lit == c->ll_shape.end()) lit = c->ll_shape.emplace(plan->uid, oneshot_order(plan->plan)).first;
    if (!lit->second.empty()) {
      LLArgs la{};
      la.buf = (char *)dptr;
      for (int t = 0; t < c->world; t++) la.peer_scratch[t] = c->ll_peer[t];
      la.my_scratch = c->ll_scratch;
      for (int k = 0; k < c->world; k++) la.order[k] = lit->second[k];
      la.bytes = (long long)nbytes_call;
      la.cap_lines = c->ll_cap_lines;
      la.me = c->rank;
      la.world = c->world;
      la.esize = plan->esize;
      la.avg_n = avg_n;
      la.epoch_dev = c->err + 3;
      la.done_ctr = (unsigned int *)(c->err + 4);
      la.err = c->err;
      la.timeout_ns = c->timeout_ns;
      const long long lines = (la.bytes + 7) / 8;
      const int ctas = (int)std::max(1LL, std::min<long long>(c->ll_ctas, (lines + kThreads - 1) / kThreads));
      ar_ll_kernel<<<ctas, kThreads, 0, (cudaStream_t)stream>>>(la);
      CUDA_OK(cudaGetLastError());
      c->last_launches = 1;
      c->last_kernel = "ar_ll_kernel";
      return AR_OK;
    }
  }
  if (c->local && c->flat && c->bulk && c->store_tma && c->trace == nullptr) {
    // emulated ranks, CPS-shaped plan: one flag-free launch over every SM (ar_flat_kernel)
    auto lit = c->ll_shape.find(plan->uid);
    if (lit == c->ll_shape.end()) lit = c->ll_shape.emplace(plan->uid, oneshot_order(plan->plan)).first;
    if (!lit->second.empty()) {
      FlatArgs fa{};
      fa.base = (char *)dptr;
      fa.stride = (long long)(stride_override ? stride_override : ar_rank_stride_bytes(count, dtype));
      fa.count = (long long)count;
      fa.world = c->world;
      fa.esize = plan->esize;
      fa.avg_n = avg_n;
      for (int k = 0; k < c->world; k++) fa.order[k] = lit->second[k];
      fa.stages = c->stages;
      fa.stage_bytes = c->stage_bytes;
      fa.ctr = (c->dyn && c->world <= 8) ? c->flat_ctr : nullptr;
      ar_flat_kernel<<<c->max_ctas, kThreads, dyn_smem_bytes(c->stages, c->stage_bytes), (cudaStream_t)stream>>>(fa);
      CUDA_OK(cudaGetLastError());
      c->last_launches = 1;
      c->last_kernel = "ar_flat_kernel";
      return AR_OK;
    }
    if (c->flatsteps) {
      // emulated ranks, multi-step plan: every step's ops over every SM, grid barriers between
      // steps (ar_flatsteps_kernel)
      auto fit = c->flatsteps_cache.find(plan->uid);
      if (fit == c->flatsteps_cache.end()) {
        std::vector<DevStep> st;
        std::vector<DevOp> ops;
        std::vector<DevWait> w;
        std::vector<int> rk, pb, pl;
        lower_plan(plan->plan, c->world, st, ops, w, rk, pb, pl);
        int maxslot = 0;
        for (const DevStep &x : st) maxslot = std::max(maxslot, x.slot);
        std::vector<std::vector<int>> by(maxslot + 1);   // slot s + 1 = after plan step s
        for (const DevStep &x : st)
          for (int i = 0; i < x.op_count; i++) by[x.slot].push_back(x.op_begin + i);
        std::vector<DevOp> gops;
        std::vector<int> gb{0};
        for (const auto &v : by) {
          if (v.empty()) continue;
          for (int i : v) gops.push_back(ops[i]);
          gb.push_back((int)gops.size());
        }
        FlatSteps F;
        F.nsteps = (int)gb.size() - 1;
        F.ops = upload(gops);
        F.ranks = upload(rk);
        F.gbegin = upload(gb);
        fit = c->flatsteps_cache.emplace(plan->uid, F).first;
      }
      FlatStepsArgs fs{};
      fs.base = (char *)dptr;
      fs.stride = (long long)(stride_override ? stride_override : ar_rank_stride_bytes(count, dtype));
      fs.ops = fit->second.ops;
      fs.ranks = fit->second.ranks;
      fs.gbegin = fit->second.gbegin;
      fs.nsteps = fit->second.nsteps;
      fs.esize = plan->esize;
      fs.avg_n = avg_n;
      fs.stages = c->stages;
      fs.stage_bytes = c->stage_bytes;
      fs.bar = c->fs_bar;
      fs.err = c->err;
      fs.timeout_ns = c->timeout_ns;
      void *args[] = {&fs};
      CUDA_OK(cudaLaunchCooperativeKernel((const void *)ar_flatsteps_kernel, dim3(c->max_ctas), dim3(kThreads), args,
                                          dyn_smem_bytes(c->stages, c->stage_bytes), (cudaStream_t)stream));
      c->last_launches = 1;
      c->last_kernel = "ar_flatsteps_kernel";
      return AR_OK;
    }
  }
  if (c->fast_valid && c->fast_uid == plan->uid && c->fast_dptr == dptr && c->fast_nctas == c->nctas) {
    // steady state: same plan and buffer as the previous call — launch the cached arguments
    ++c->epoch;
    c->fast_args.avg_n = avg_n;
    void *args[] = {&c->fast_args};
    launch_exec(c, grid, args, (cudaStream_t)stream);
    c->last_launches = 1;
    c->last_kernel = "ar_exec_kernel";
    return AR_OK;
  }
  const size_t bytes = count * (size_t)plan->esize;
  ExecArgs a{};
  if (c->local) {
    const uint64_t stride = stride_override ? stride_override : ar_rank_stride_bytes(count, dtype);
    for (int r = 0; r < c->world; r++) {
      a.bufs[r] = (char *)dptr + stride * r;
      a.sigs[r] = c->sig[r];
    }
  } else {
    // several ranks per process: consecutive rank buffers at the emulated stride
    const uint64_t stride =
        c->rpp > 1 ? (stride_override ? stride_override : ar_rank_stride_bytes(count, dtype)) : 0;
    const size_t need = c->rpp > 1 ? stride * (c->rpp - 1) + bytes : bytes;
    // dptr may point inside a registered buffer (same offset on every rank)
    Registration *reg = nullptr;
    size_t inner = 0;
    for (auto &r : c->regs)
      if (r.opened && (char *)dptr >= r.local && (char *)dptr + need <= r.local + r.bytes) {
        reg = &r;
        inner = (size_t)((char *)dptr - r.local);
      }
    if (!reg) throw InvalidArg("buffer is not registered and opened on this communicator (or too small)");
    for (int r = 0; r < c->world; r++) {
      char *base = reg->peer[r / c->rpp];
      a.bufs[r] = base ? base + inner + stride * (r % c->rpp) : nullptr;
      a.sigs[r] = c->sig[r];
      if (!a.bufs[r] || !a.sigs[r]) throw InvalidArg("peer buffer not opened");
    }
  }
  // push protocol for CPS-shaped plans of moderate size (one rank per GPU)
  bool use_push = false;
  if (c->ll_opened && c->push_max_bytes > 0 && (long long)bytes <= c->push_max_bytes) {
    auto lit = c->ll_shape.find(plan->uid);
    if (lit == c->ll_shape.end()) lit = c->ll_shape.emplace(plan->uid, oneshot_order(plan->plan)).first;
    use_push = !lit->second.empty();
  }
  std::map<uint64_t, Lowered> &cache = use_push ? c->lowered_push : c->lowered;
  auto it = cache.find(plan->uid);
  if (it == cache.end()) {
    std::vector<DevStep> st;
    std::vector<DevOp> ops;
    std::vector<DevWait> w;
    std::vector<int> rk, pb, pl;
    if (use_push) lower_push(plan->plan, c->ll_shape[plan->uid], st, ops, w, rk, pb, pl);
    else lower_plan(plan->plan, c->world, st, ops, w, rk, pb, pl);
    Lowered L;
    if (!c->local) {  // this process runs only the programs of the ranks it hosts
      std::vector<int> pb1(pb.begin() + c->rank, pb.begin() + c->rank + c->rpp);
      std::vector<int> pl1(pl.begin() + c->rank, pl.begin() + c->rank + c->rpp);
      pb = pb1;
      pl = pl1;
    }
    L.steps = upload(st);
    L.ops = upload(ops);
    if (c->dyn && !c->local && c->rpp == 1 && !use_push) {
      // CPS-shaped plans only: their one data step sits between paired entry and exit waits,
      // and any CTA of a peer having posted implies the whole peer buffer is ready / done, so
      // tiles need not belong to fixed CTAs (range waits of multi-step plans do need that)
      auto lit = c->ll_shape.find(plan->uid);
      if (lit == c->ll_shape.end()) lit = c->ll_shape.emplace(plan->uid, oneshot_order(plan->plan)).first;
      if (!lit->second.empty() && !ops.empty()) {
        L.nops = (int)ops.size();
        CUDA_OK(cudaMalloc(&L.dyn_ctr, ops.size() * sizeof(unsigned int)));
        CUDA_OK(cudaMemset(L.dyn_ctr, 0, ops.size() * sizeof(unsigned int)));
      }
    }
    L.waits = upload(w);
    L.ranks = upload(rk);
    L.prog_begin = upload(pb);
    L.prog_len = upload(pl);
    it = cache.emplace(plan->uid, L).first;
  }
  if (use_push)
    for (int t = 0; t < c->world; t++) a.scr[t] = c->ll_peer[t] + c->ll_region;
  a.scr_plane = c->push_plane;
  a.scr_slot = c->push_slot;
  const Lowered &L = it->second;
  a.steps = L.steps;
  a.ops = L.ops;
  a.waits = L.waits;
  a.ranks = L.ranks;
  a.prog_begin = L.prog_begin;
  a.prog_len = L.prog_len;
  a.err = c->err;
  ++c->epoch;
  a.epoch_dev = c->err + 1;
  a.done_ctr = (unsigned int *)(c->err + 2);
  a.timeout_ns = c->timeout_ns;
  a.rank0 = c->local ? 0 : c->rank;
  a.world = c->world;
  a.cta_cap = c->cta_cap;
  a.esize = plan->esize;
  a.bulk = c->bulk ? 1 : 0;
  a.trace = c->trace;
  a.fence_mode = c->fence_mode >= 0 ? c->fence_mode : (c->local ? 3 : 1);
  a.store_tma = c->store_tma ? 1 : 0;
  a.stages = c->stages;
  a.stage_bytes = c->stage_bytes;
  a.jitter_ns = c->jitter_ns;
  a.avg_n = avg_n;
  a.dyn_ctr = (a.bulk && a.store_tma) ? L.dyn_ctr : nullptr;
  a.dyn_nops = a.dyn_ctr ? L.nops : 0;
  a.entry_fence = c->entry_fence ? 1 : 0;
  c->fast_args = a;
  c->fast_uid = plan->uid;
  c->fast_dptr = dptr;
  c->fast_nctas = c->nctas;
  c->fast_valid = true;
  void *args[] = {&a};
  launch_exec(c, grid, args, (cudaStream_t)stream);
  c->last_launches = 1;
  c->last_kernel = "ar_exec_kernel";
  return AR_OK;
}

int allreduce_exec(const gt_plan *plan, ar_comm *c, void *dptr, uint64_t count, int32_t dtype, void *stream) {
  SYS_TRY({ return exec_impl(plan, c, dptr, count, dtype, stream); })
}

int allreduce_exec_op(const gt_plan *plan, ar_comm *c, void *dptr, uint64_t count, int32_t dtype, int32_t op,
                      void *stream) {
  SYS_TRY({ return exec_impl(plan, c, dptr, count, dtype, stream, op); })
}

int ar_exec_movement_plan(const gt_plan *plan, ar_comm *c, void *dptr, uint64_t count, int32_t dtype, void *stream) {
  SYS_TRY({ return exec_impl(plan, c, dptr, count, dtype, stream, AR_OP_SUM, 0, true); })
}

// A plan whose every element is summed in ascending rank order by one reduce (natural CPS):
// any element range can then run as its own CPS plan with the same bits.
static bool ascending_cps(const Plan &p) {
  std::vector<int> ord = oneshot_order(p);
  if (ord.empty()) return false;
  for (int i = 0; i < (int)ord.size(); i++)
    if (ord[i] != i) return false;
  return true;
}

// End to end with host buffers, pipelined: the element range is split into chunks run as
// natural-CPS sub-plans (same bits, see ascending_cps); chunk k's H2D, AllReduce and D2H run
// on three streams so the copies of neighbouring chunks overlap each other (PCIe is full
// duplex) and the kernels.  Plans of other shapes copy, execute and copy back in sequence.
static void exec_host_chunked(const gt_plan *plan, ar_comm *c, char *dptr, char *host, uint64_t count,
                              int32_t dtype, cudaStream_t s, int chunks) {
  const int es = plan->esize;
  const size_t stride = c->rpp > 1 ? ar_rank_stride_bytes(count, dtype) : count * (size_t)es;
  const uint64_t per = ((count + chunks - 1) / chunks + 127) / 128 * 128;
  if (!c->h2d) {
    CUDA_OK(cudaStreamCreateWithFlags(&c->h2d, cudaStreamNonBlocking));
    CUDA_OK(cudaStreamCreateWithFlags(&c->d2h, cudaStreamNonBlocking));
  }
  while ((int)c->evs.size() < 2 * chunks + 2) {
    cudaEvent_t e;
    CUDA_OK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    c->evs.push_back(e);
  }
  cudaEvent_t start = c->evs[0], done = c->evs[1];
  CUDA_OK(cudaEventRecord(start, s));
  CUDA_OK(cudaStreamWaitEvent(c->h2d, start, 0));
  CUDA_OK(cudaStreamWaitEvent(c->d2h, start, 0));
  for (int k = 0; k < chunks; k++) {
    const uint64_t off = per * k;
    if (off >= count) break;
    const uint64_t n = std::min<uint64_t>(per, count - off);
    auto key = std::make_pair(plan->uid, n);
    auto it = c->sub_plans.find(key);
    if (it == c->sub_plans.end()) {
      gt_plan *g = new gt_plan();
      g->plan = build_plan_natural("cps", plan->plan.n, (int64_t)n);
      g->dtype = plan->dtype;
      g->esize = plan->esize;
      g->uid = next_plan_uid();
      it = c->sub_plans.emplace(key, g).first;
    }
    cudaEvent_t eh = c->evs[2 + 2 * k], ec = c->evs[3 + 2 * k];
    CUDA_OK(cudaMemcpy2DAsync(dptr + off * es, stride, host + off * es, stride, n * es, c->rpp,
                              cudaMemcpyHostToDevice, c->h2d));
    CUDA_OK(cudaEventRecord(eh, c->h2d));
    CUDA_OK(cudaStreamWaitEvent(s, eh, 0));
    int rc = exec_impl(it->second, c, dptr + off * es, n, dtype, s, AR_OP_SUM, c->rpp > 1 ? stride : 0);
    if (rc != AR_OK) throw SysError("chunk execution failed");
    CUDA_OK(cudaEventRecord(ec, s));
    CUDA_OK(cudaStreamWaitEvent(c->d2h, ec, 0));
    CUDA_OK(cudaMemcpy2DAsync(host + off * es, stride, dptr + off * es, stride, n * es, c->rpp,
                              cudaMemcpyDeviceToHost, c->d2h));
  }
  CUDA_OK(cudaEventRecord(done, c->d2h));
  CUDA_OK(cudaStreamWaitEvent(s, done, 0));
}

int allreduce_exec_host(const gt_plan *plan, ar_comm *c, void *dptr, void *host, uint64_t count, int32_t dtype,
                        void *stream) {
  SYS_TRY({
    if (!host) throw InvalidArg("null host buffer");
    if (!c) throw InvalidArg("null comm");
    if (!plan) throw InvalidArg("null plan");
    if (!plan->is_allreduce) throw InvalidArg("plan is not an AllReduce (failed symbolic verification)");
    CUDA_OK(cudaSetDevice(c->device));
    const size_t bytes = c->rpp > 1 ? ar_rank_stride_bytes(count, dtype) * c->rpp
                                    : count * (size_t)(dtype == AR_BF16 ? 2 : 4);
    cudaStream_t s = (cudaStream_t)stream;
    // chunks of >= 4 MiB per rank, at most 32: the copies of the first and last chunk cannot
    // overlap anything, so more chunks shorten that fill/drain (bench N = 1, 8 x 256 MiB:
    // 8 / 16 / 32 / 64 chunks -> 9.89 / 10.29 / 10.42 / 10.32 GB/s busbw end to end)
    const uint64_t per_rank = count * (uint64_t)plan->esize;
    int chunks = (int)std::min<uint64_t>(32, std::max<uint64_t>(2, per_rank / (4u << 20)));
    if (const char *v = std::getenv("AR_E2E_CHUNKS")) chunks = std::max(1, std::atoi(v));
    if (chunks > 1 && count * (uint64_t)plan->esize >= (8u << 20) && (uint64_t)plan->plan.count == count &&
        plan->dtype == dtype && ascending_cps(plan->plan)) {
      exec_host_chunked(plan, c, (char *)dptr, (char *)host, count, dtype, s, chunks);
      return AR_OK;
    }
    CUDA_OK(cudaMemcpyAsync(dptr, host, bytes, cudaMemcpyHostToDevice, s));
    int rc = exec_impl(plan, c, dptr, count, dtype, stream);
    if (rc != AR_OK) return rc;
    CUDA_OK(cudaMemcpyAsync(host, dptr, bytes, cudaMemcpyDeviceToHost, s));
    return AR_OK;
  })
}

int ar_fill_synthetic(void *dptr, uint64_t count, int32_t dtype, uint64_t seed, int32_t rank, int32_t mode,
                      uint64_t start, void *stream) {
  SYS_TRY({
    if (!dptr) throw InvalidArg("null pointer");
    if (dtype != AR_F32 && dtype != AR_BF16) throw InvalidArg("unknown dtype");
    if (mode < 0 || mode > 2) throw InvalidArg("unknown mode");
    if (count == 0) return AR_OK;
    unsigned long long blocks = std::min<unsigned long long>((count + 255) / 256, 148ull * 16);
    fill_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(dptr, count, dtype == AR_BF16, seed, rank, mode,
                                                                    start);
    CUDA_OK(cudaGetLastError());
    return AR_OK;
  })
}

int ar_local_reduce(void *const *inputs, int32_t k, void *out, uint64_t count, int32_t dtype, void *stream) {
  SYS_TRY({
    if (!inputs || !out) throw InvalidArg("null argument");
    if (k < 1 || k > AR_MAX_RANKS) throw InvalidArg("k must be in 1..64");
    const int es = dtype == AR_BF16 ? 2 : 4;
    if ((count * es) % 16) throw InvalidArg("count * element size must be a multiple of 16 bytes");
    LocalReduceArgs a{};
    for (int i = 0; i < k; i++) {
      if ((uintptr_t)inputs[i] % 16) throw InvalidArg("inputs must be 16-byte aligned");
      a.in[i] = (const uint4 *)inputs[i];
    }
    if ((uintptr_t)out % 16) throw InvalidArg("output must be 16-byte aligned");
    a.out = (uint4 *)out;
    a.nvec = count * es / 16;
    a.k = k;
    int dev = 0, nsm = 148;
    CUDA_OK(cudaGetDevice(&dev));
    CUDA_OK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
    if (dtype == AR_BF16) local_reduce_kernel<true><<<nsm * 2, kThreads, 0, (cudaStream_t)stream>>>(a);
    else local_reduce_kernel<false><<<nsm * 2, kThreads, 0, (cudaStream_t)stream>>>(a);
    CUDA_OK(cudaGetLastError());
    return AR_OK;
  })
}

}  // extern "C"
