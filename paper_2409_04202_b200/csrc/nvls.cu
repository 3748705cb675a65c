// NVLS plan kind: the fan-in-N reduction of a Co-located-PS step done
// inside the NVSwitch.  Rank r owns block r; for every 16-byte vector of its block it
// issues one multimem.ld_reduce on the multicast address — the switch reads the vector from
// all N GPUs and returns their sum — and one multimem.st that the switch replicates into all N
// GPUs' buffers.  Per GPU and direction ~S bytes cross NVLink instead of 2(N−1)/N·S, and the
// GPU-side memory term δ of the reduce vanishes (the switch reduces).  The summation order is
// the switch's, not fixed by a plan: results are checked against the float64 sum (and exactly
// on integer-valued inputs), not bit-for-bit against the oracle's plan order.
//
// Memory: each rank backs its buffer with cuMemCreate'd memory bound to one multicast object
// (cuMulticastCreate by rank 0, POSIX-FD handle passed to the other processes with
// pidfd_getfd); the buffer is mapped twice: unicast (this GPU's copy, the tensor the caller
// uses) and multicast.  A small flag area after the data holds per-(slot, CTA) counters that
// every rank increments on all GPUs at once with multimem.red — the entry and exit barriers.
#include <cuda.h>
#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cstdint>
#include <cstring>
#include <string>

#include "../../include/gentree_ar.h"
#include "internal.hpp"

using namespace gtar;

namespace {

constexpr int kNvThreads = 512;
constexpr int kNvCtaCap = 256;
constexpr uint32_t kNvMagic = 0x4E564C53u;   // "NVLS"

struct SysErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

#define CU_CALL(fn, ...)                                                              \
  do {                                                                                \
    CUresult r_ = drv().fn(__VA_ARGS__);                                              \
    if (r_ != CUDA_SUCCESS) throw SysErr(std::string(#fn) + " failed: " + std::to_string((int)r_)); \
  } while (0)
#define RT_CALL(x)                                                                         \
  do {                                                                                     \
    cudaError_t e_ = (x);                                                                  \
    if (e_ != cudaSuccess) throw SysErr(std::string(#x) + ": " + cudaGetErrorString(e_));  \
  } while (0)

// Driver entry points resolved through the runtime (no -lcuda link dependency).
struct Drv {
  decltype(&::cuMemCreate) cuMemCreate = nullptr;
  decltype(&::cuMemRelease) cuMemRelease = nullptr;
  decltype(&::cuMemAddressReserve) cuMemAddressReserve = nullptr;
  decltype(&::cuMemAddressFree) cuMemAddressFree = nullptr;
  decltype(&::cuMemMap) cuMemMap = nullptr;
  decltype(&::cuMemUnmap) cuMemUnmap = nullptr;
  decltype(&::cuMemSetAccess) cuMemSetAccess = nullptr;
  decltype(&::cuMemExportToShareableHandle) cuMemExportToShareableHandle = nullptr;
  decltype(&::cuMemImportFromShareableHandle) cuMemImportFromShareableHandle = nullptr;
  decltype(&::cuMulticastCreate) cuMulticastCreate = nullptr;
  decltype(&::cuMulticastAddDevice) cuMulticastAddDevice = nullptr;
  decltype(&::cuMulticastBindMem) cuMulticastBindMem = nullptr;
  decltype(&::cuMulticastUnbind) cuMulticastUnbind = nullptr;
  decltype(&::cuMulticastGetGranularity) cuMulticastGetGranularity = nullptr;
  decltype(&::cuDeviceGet) cuDeviceGet = nullptr;
};

template <typename F>
static void load(F &f, const char *name) {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess || !p)
    throw SysErr(std::string("driver entry point unavailable: ") + name);
  f = reinterpret_cast<F>(p);
}

static Drv &drv() {
  static Drv d;
  static bool init = false;
  if (!init) {
    load(d.cuMemCreate, "cuMemCreate");
    load(d.cuMemRelease, "cuMemRelease");
    load(d.cuMemAddressReserve, "cuMemAddressReserve");
    load(d.cuMemAddressFree, "cuMemAddressFree");
    load(d.cuMemMap, "cuMemMap");
    load(d.cuMemUnmap, "cuMemUnmap");
    load(d.cuMemSetAccess, "cuMemSetAccess");
    load(d.cuMemExportToShareableHandle, "cuMemExportToShareableHandle");
    load(d.cuMemImportFromShareableHandle, "cuMemImportFromShareableHandle");
    load(d.cuMulticastCreate, "cuMulticastCreate");
    load(d.cuMulticastAddDevice, "cuMulticastAddDevice");
    load(d.cuMulticastBindMem, "cuMulticastBindMem");
    load(d.cuMulticastUnbind, "cuMulticastUnbind");
    load(d.cuMulticastGetGranularity, "cuMulticastGetGranularity");
    load(d.cuDeviceGet, "cuDeviceGet");
    init = true;
  }
  return d;
}

struct Blob {
  uint32_t magic;
  int32_t rank, world, pid, fd;
  uint64_t size;
};
static_assert(sizeof(Blob) <= AR_BLOB_BYTES, "blob");

struct NvArgs {
  char *uc;                       // this rank's buffer (unicast)
  char *mc;                       // the same buffer through the multicast object
  unsigned long long *flags_uc;   // [2][cta_cap] counters (local copy)
  unsigned long long *flags_mc;
  unsigned long long *epoch_dev;  // [0] epoch, [1] finished-CTA counter, [2] error
  long long off, len;             // this rank's whole 16-byte vectors (elements)
  long long tail_off, tail_len;   // trailing elements past the last whole vector (rank world-1)
  int world, esize;
  unsigned long long timeout_ns;
  int dyn;                        // 1 = chunks handed out by atomicAdd on epoch_dev[3] (AR_NVLS_DYN)
  int avg_n;                      // AVG (fp32): divide the switch's sum by N (0 = SUM)
};

__device__ __forceinline__ unsigned long long nv_ld_acquire(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void nv_red_release(unsigned long long *mc, unsigned long long v) {
  asm volatile("multimem.red.release.sys.global.add.u64 [%0], %1;" ::"l"(mc), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long nv_timer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

// All N ranks add 1 to counter (slot, cta) on every GPU; wait until the local copy reaches
// world * epoch (counters only grow; epochs are consecutive per call).
__device__ void nv_barrier(const NvArgs &a, int slot, unsigned long long epoch, unsigned long long t0) {
  __syncthreads();
  const int cap = kNvCtaCap;
  if (threadIdx.x == 0) {
    nv_red_release(a.flags_mc + slot * cap + blockIdx.x, 1ull);
    const unsigned long long want = (unsigned long long)a.world * epoch;
    unsigned int spins = 0;
    while (nv_ld_acquire(a.flags_uc + slot * cap + blockIdx.x) < want) {
      if ((++spins & 1023u) == 0 && nv_timer() - t0 > a.timeout_ns) {
        atomicExch(a.epoch_dev + 2, 1ull);
        break;
      }
    }
  }
  __syncthreads();
}

// MODE: 0 = fp32; 1 = bf16 with fp32 accumulation in the switch (acc::f32, the default);
// 2 = bf16 accumulated in bf16 by the switch (measurement only: AR_NVLS_BF16_ACC=bf16)
template <int MODE>
__device__ __forceinline__ uint4 ld_reduce(const void *mc) {
  uint4 v;
  if (MODE == 1)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(mc)
                 : "memory");
  else if (MODE == 2)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.bf16x2 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(mc)
                 : "memory");
  else
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(mc)
                 : "memory");
  return v;
}
template <int MODE>
__device__ __forceinline__ void mc_store(void *mc, const uint4 &v) {
  if (MODE != 0)
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
  else
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(mc), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w)
                 : "memory");
}

// AVG (fp32 only, reading NV3): the switch's correctly rounded sum divided by N with one
// correctly rounded IEEE division per element, before the multicast store
__device__ __forceinline__ uint4 avg4(uint4 v, int n) {
  const float d = (float)n;
  v.x = __float_as_uint(__fdiv_rn(__uint_as_float(v.x), d));
  v.y = __float_as_uint(__fdiv_rn(__uint_as_float(v.y), d));
  v.z = __float_as_uint(__fdiv_rn(__uint_as_float(v.z), d));
  v.w = __float_as_uint(__fdiv_rn(__uint_as_float(v.w), d));
  return v;
}

// Scalar tail (count not a multiple of 16 bytes): fp32 one element, bf16 an element pair.
template <int MODE>
__device__ __forceinline__ void tail_reduce_store(char *mc, int avg_n) {
  uint32_t v;
  if (MODE == 1)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.bf16x2 %0, [%1];" : "=r"(v) : "l"(mc) : "memory");
  else if (MODE == 2)
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.bf16x2 %0, [%1];" : "=r"(v) : "l"(mc) : "memory");
  if (MODE != 0) {
    asm volatile("multimem.st.relaxed.sys.global.bf16x2 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
  } else {
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.f32 %0, [%1];" : "=r"(v) : "l"(mc) : "memory");
    if (avg_n) v = __float_as_uint(__fdiv_rn(__uint_as_float(v), (float)avg_n));
    asm volatile("multimem.st.relaxed.sys.global.f32 [%0], %1;" ::"l"(mc), "r"(v) : "memory");
  }
}

template <int MODE, int U>
__global__ void __launch_bounds__(kNvThreads) nvls_kernel(const __grid_constant__ NvArgs a) {
  __shared__ unsigned long long s_epoch;
  const unsigned long long t0 = nv_timer();
  if (threadIdx.x == 0) s_epoch = *(volatile unsigned long long *)a.epoch_dev + 1;
  __syncthreads();
  const unsigned long long epoch = s_epoch;
  nv_barrier(a, 0, epoch, t0);   // every rank's input is in place
  const long long vb = a.off * a.esize / 16, nv = a.len * a.esize / 16;
  const long long v0 = vb + nv * blockIdx.x / gridDim.x, v1 = vb + nv * (blockIdx.x + 1) / gridDim.x;
  if (a.dyn) {
    // dynamic chunks of 8 x (blockDim x U) vectors: CTAs that get more switch bandwidth take
    // more chunks (the same scheme as the P2P executor's tiles).  A/B option, off by default:
    // measured equal at 256 MiB - 1 GiB and 1-3 % slower at 16 MiB on 2 and 4 B200s
    // (profiles/round1/dyn/nvls_dyn_ab.txt) — the 16 NVLS CTAs are not imbalanced
    __shared__ long long s_chunk;
    unsigned int *ctr = (unsigned int *)(a.epoch_dev + 3);
    const long long CH = (long long)blockDim.x * U * 8;
    const long long nch = (nv + CH - 1) / CH;
    for (;;) {
      if (threadIdx.x == 0) s_chunk = (long long)atomicAdd(ctr, 1u);
      __syncthreads();
      const long long c = s_chunk;
      __syncthreads();
      if (c >= nch) break;
      const long long c0 = vb + c * CH, c1 = min(vb + nv, c0 + CH);
      for (long long base = c0 + threadIdx.x; base < c1; base += (long long)blockDim.x * U) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; u++) {
          const long long v = base + (long long)u * blockDim.x;
          if (v < c1) x[u] = ld_reduce<MODE>(a.mc + v * 16);
        }
#pragma unroll
        for (int u = 0; u < U; u++) {
          const long long v = base + (long long)u * blockDim.x;
          if (v < c1) mc_store<MODE>(a.mc + v * 16, (MODE == 0 && a.avg_n) ? avg4(x[u], a.avg_n) : x[u]);
        }
      }
    }
  } else
  for (long long base = v0 + threadIdx.x; base < v1; base += (long long)blockDim.x * U) {
    uint4 x[U];
#pragma unroll
    for (int u = 0; u < U; u++) {
      const long long v = base + (long long)u * blockDim.x;
      if (v < v1) x[u] = ld_reduce<MODE>(a.mc + v * 16);
    }
#pragma unroll
    for (int u = 0; u < U; u++) {
      const long long v = base + (long long)u * blockDim.x;
      if (v < v1) mc_store<MODE>(a.mc + v * 16, (MODE == 0 && a.avg_n) ? avg4(x[u], a.avg_n) : x[u]);
    }
  }
  if (a.tail_len > 0 && blockIdx.x == 0) {
    const int step = MODE != 0 ? 2 : 1;
    for (long long e = a.tail_off + (long long)threadIdx.x * step; e < a.tail_off + a.tail_len;
         e += (long long)blockDim.x * step)
      tail_reduce_store<MODE>(a.mc + e * a.esize, a.avg_n);
  }
  nv_barrier(a, 1, epoch, t0);   // every rank's results have landed in every GPU's buffer
  if (threadIdx.x == 0) {
    if (atomicAdd((unsigned int *)(a.epoch_dev + 1), 1u) == gridDim.x - 1) {
      *(volatile unsigned int *)(a.epoch_dev + 1) = 0;
      *(volatile unsigned int *)(a.epoch_dev + 3) = 0;   // dynamic chunk counter
      *(volatile unsigned long long *)a.epoch_dev = epoch;
      __threadfence();
    }
  }
}

}  // namespace

struct ar_nvls {
  int rank = 0, world = 0, device = 0;
  size_t data_bytes = 0, size = 0;   // size = data + flags, rounded to the multicast granularity
  CUmemGenericAllocationHandle mc = 0, mem = 0;
  bool have_mc = false, have_mem = false, bound = false;
  CUdeviceptr uc = 0, mcva = 0;
  int mc_fd = -1;
  unsigned long long *dev_words = nullptr;
  int nctas = 0;
  unsigned long long timeout_ns = 10ull * 1000 * 1000 * 1000;
  bool dyn = false;
  int unroll = 4;              // 16-byte vectors in flight per thread (AR_NVLS_U: 2, 4, 8, 16)
  bool bf16_acc_bf16 = false;  // AR_NVLS_BF16_ACC=bf16: switch accumulates bf16 (measurement only)
};

namespace {
template <int MODE>
void launch_unroll(int unroll, int nctas, cudaStream_t st, const NvArgs &a) {
  switch (unroll) {
    case 2: nvls_kernel<MODE, 2><<<nctas, kNvThreads, 0, st>>>(a); break;
    case 8: nvls_kernel<MODE, 8><<<nctas, kNvThreads, 0, st>>>(a); break;
    case 16: nvls_kernel<MODE, 16><<<nctas, kNvThreads, 0, st>>>(a); break;
    default: nvls_kernel<MODE, 4><<<nctas, kNvThreads, 0, st>>>(a); break;
  }
}
void launch_mode(int mode, int unroll, int nctas, cudaStream_t st, const NvArgs &a) {
  if (mode == 1) launch_unroll<1>(unroll, nctas, st, a);
  else if (mode == 2) launch_unroll<2>(unroll, nctas, st, a);
  else launch_unroll<0>(unroll, nctas, st, a);
}
}  // namespace

namespace gtar {
// Launch the in-switch AllReduce of `count` elements of this rank's NVLS buffer (dptr must be
// its unicast base).  Whole 16-byte vectors are split evenly over the ranks (the result does
// not depend on the split: the switch reduces every element once); the trailing elements past
// the last whole vector go to the last rank (fp32: any count; bf16: even counts).
void nvls_launch(ar_nvls *n, const void *dptr, uint64_t count, int32_t dtype, void *stream, int avg_n) {
  if (!n || !n->bound) throw InvalidArg("nvls buffer not bound");
  if (dtype != AR_F32 && dtype != AR_BF16) throw InvalidArg("unknown dtype");
  if ((CUdeviceptr)dptr != n->uc) throw InvalidArg("the buffer is not this communicator's NVLS buffer");
  const int es = dtype == AR_BF16 ? 2 : 4;
  if (count < 1 || count * es > n->data_bytes) throw InvalidArg("count exceeds the nvls buffer");
  if (dtype == AR_BF16 && count % 2) throw InvalidArg("nvls bf16 needs an even count");
  if (avg_n && dtype != AR_F32) throw InvalidArg("NVLS AVG is fp32 only");
  int cur = -1;
  RT_CALL(cudaGetDevice(&cur));
  if (cur != n->device) RT_CALL(cudaSetDevice(n->device));
  NvArgs a{};
  a.uc = (char *)n->uc;
  a.mc = (char *)n->mcva;
  a.flags_uc = (unsigned long long *)((char *)n->uc + n->data_bytes);
  a.flags_mc = (unsigned long long *)((char *)n->mcva + n->data_bytes);
  a.epoch_dev = n->dev_words;
  const long long E = 16 / es;
  const long long nvec = (long long)count / E;
  const long long v0 = nvec * n->rank / n->world, v1 = nvec * (n->rank + 1) / n->world;
  a.off = v0 * E;
  a.len = (v1 - v0) * E;
  a.tail_off = nvec * E;
  a.tail_len = n->rank == n->world - 1 ? (long long)count - nvec * E : 0;
  a.world = n->world;
  a.esize = es;
  a.timeout_ns = n->timeout_ns;
  a.dyn = n->dyn ? 1 : 0;
  a.avg_n = avg_n;
  const int mode = dtype == AR_BF16 ? (n->bf16_acc_bf16 ? 2 : 1) : 0;
  launch_mode(mode, n->unroll, n->nctas, (cudaStream_t)stream, a);
  RT_CALL(cudaGetLastError());
}
}  // namespace gtar

#define NV_TRY(...)                                         \
  try {                                                     \
    __VA_ARGS__                                             \
  } catch (const InvalidArg &e) {                           \
    set_error(e.what());                                    \
    return AR_EINVAL;                                       \
  } catch (const std::exception &e) {                       \
    set_error(e.what());                                    \
    return AR_ESYS;                                         \
  }

extern "C" {

int ar_nvls_create(int32_t rank, int32_t world, int32_t cuda_device, uint64_t bytes, ar_nvls **out,
                   void *blob_out) {
  NV_TRY({
    if (!out || !blob_out) throw InvalidArg("null argument");
    if (world < 2 || world > AR_MAX_RANKS || rank < 0 || rank >= world) throw InvalidArg("bad rank/world");
    if (bytes < 16 || bytes % 16) throw InvalidArg("bytes must be a positive multiple of 16");
    RT_CALL(cudaSetDevice(cuda_device));
    RT_CALL(cudaFree(0));   // make sure the primary context exists
    ar_nvls *n = new ar_nvls();
    n->rank = rank;
    n->world = world;
    n->device = cuda_device;
    n->data_bytes = bytes;
    CUmulticastObjectProp prop{};
    prop.numDevices = world;
    prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    prop.size = bytes + 2 * kNvCtaCap * 8;
    size_t gran = 0;
    CU_CALL(cuMulticastGetGranularity, &gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED);
    n->size = (prop.size + gran - 1) / gran * gran;
    prop.size = n->size;
    Blob b{};
    b.magic = kNvMagic;
    b.rank = rank;
    b.world = world;
    b.pid = (int)getpid();
    b.fd = -1;
    b.size = n->size;
    if (rank == 0) {
      CU_CALL(cuMulticastCreate, &n->mc, &prop);
      n->have_mc = true;
      int fd = -1;
      CU_CALL(cuMemExportToShareableHandle, (void *)&fd, n->mc, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0);
      n->mc_fd = fd;
      b.fd = fd;
    }
    std::memset(blob_out, 0, AR_BLOB_BYTES);
    std::memcpy(blob_out, &b, sizeof b);
    int nsm = 148;
    RT_CALL(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, cuda_device));
    // few CTAs: the switch serves multimem requests best with little contention (measured:
    // 4 x B200 bf16 256 MiB, 16 CTAs 674 GB/s busbw vs 148 CTAs 591; 2 x B200 fp32 256 MiB,
    // 32 CTAs 402 vs 16 CTAs 361 and 148 CTAs 352 — profiles/round1/nvls_ctas)
    n->nctas = std::min(world == 2 ? 32 : 16, std::min(nsm, kNvCtaCap));
    if (const char *v = std::getenv("AR_NVLS_CTAS")) n->nctas = std::max(1, std::min(kNvCtaCap, std::atoi(v)));
    if (const char *t = std::getenv("AR_FLAG_TIMEOUT_MS")) n->timeout_ns = std::strtoull(t, nullptr, 10) * 1000000ull;
    if (const char *v = std::getenv("AR_NVLS_DYN")) n->dyn = std::string(v) != "0";
    if (const char *v = std::getenv("AR_NVLS_U")) {
      const int u = std::atoi(v);
      if (u != 2 && u != 4 && u != 8 && u != 16) throw InvalidArg("AR_NVLS_U must be 2, 4, 8 or 16");
      n->unroll = u;
    }
    if (const char *v = std::getenv("AR_NVLS_BF16_ACC")) n->bf16_acc_bf16 = std::string(v) == "bf16";
    *out = n;
    return AR_OK;
  })
}

int ar_nvls_attach(ar_nvls *n, const void *blobs) {
  NV_TRY({
    if (!n || !blobs) throw InvalidArg("null argument");
    RT_CALL(cudaSetDevice(n->device));
    const Blob *b0 = (const Blob *)blobs;
    if (b0->magic != kNvMagic || b0->world != n->world || b0->rank != 0) throw InvalidArg("bad nvls blob");
    if (b0->size != n->size) throw InvalidArg("ranks disagree on the nvls buffer size");
    if (n->rank != 0) {
      // duplicate rank 0's exported file descriptor into this process (pidfd_getfd, Linux 5.6+)
      int pidfd = (int)syscall(SYS_pidfd_open, b0->pid, 0);
      if (pidfd < 0) throw SysErr("pidfd_open failed: " + std::to_string(errno));
      int fd = (int)syscall(SYS_pidfd_getfd, pidfd, b0->fd, 0);
      close(pidfd);
      if (fd < 0) throw SysErr("pidfd_getfd failed: " + std::to_string(errno));
      CU_CALL(cuMemImportFromShareableHandle, &n->mc, (void *)(intptr_t)fd, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
      close(fd);
      n->have_mc = true;
    }
    CUdevice dev;
    CU_CALL(cuDeviceGet, &dev, n->device);
    CU_CALL(cuMulticastAddDevice, n->mc, dev);
    return AR_OK;
  })
}

int ar_nvls_bind(ar_nvls *n, void **uc_ptr_out) {
  NV_TRY({
    if (!n || !uc_ptr_out) throw InvalidArg("null argument");
    RT_CALL(cudaSetDevice(n->device));
    CUmemAllocationProp ap{};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = n->device;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    CU_CALL(cuMemCreate, &n->mem, n->size, &ap, 0);
    n->have_mem = true;
    CU_CALL(cuMulticastBindMem, n->mc, 0, n->mem, 0, n->size, 0);
    n->bound = true;
    CUmemAccessDesc acc{};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = n->device;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU_CALL(cuMemAddressReserve, &n->uc, n->size, 0, 0, 0);
    CU_CALL(cuMemMap, n->uc, n->size, 0, n->mem, 0);
    CU_CALL(cuMemSetAccess, n->uc, n->size, &acc, 1);
    CU_CALL(cuMemAddressReserve, &n->mcva, n->size, 0, 0, 0);
    CU_CALL(cuMemMap, n->mcva, n->size, 0, n->mc, 0);
    CU_CALL(cuMemSetAccess, n->mcva, n->size, &acc, 1);
    RT_CALL(cudaMemset((void *)n->uc, 0, n->size));
    RT_CALL(cudaMalloc(&n->dev_words, 4 * sizeof(unsigned long long)));
    RT_CALL(cudaMemset(n->dev_words, 0, 4 * sizeof(unsigned long long)));
    RT_CALL(cudaDeviceSynchronize());
    *uc_ptr_out = (void *)n->uc;
    return AR_OK;
  })
}

int allreduce_exec_nvls(ar_nvls *n, uint64_t count, int32_t dtype, void *stream) {
  NV_TRY({
    if (!n || !n->bound) throw InvalidArg("nvls buffer not bound");
    gtar::nvls_launch(n, (const void *)n->uc, count, dtype, stream, 0);
    return AR_OK;
  })
}

int ar_nvls_get_async_error(ar_nvls *n) {
  NV_TRY({
    if (!n) throw InvalidArg("null argument");
    RT_CALL(cudaSetDevice(n->device));
    RT_CALL(cudaDeviceSynchronize());
    if (!n->dev_words) return AR_OK;
    unsigned long long w[4];
    RT_CALL(cudaMemcpy(w, n->dev_words, sizeof w, cudaMemcpyDeviceToHost));
    if (w[2]) {
      RT_CALL(cudaMemset(n->dev_words + 2, 0, 8));
      throw SysErr("nvls barrier timed out on the device");
    }
    return AR_OK;
  })
}

int ar_nvls_destroy(ar_nvls *n) {
  if (!n) return AR_OK;
  cudaSetDevice(n->device);
  cudaDeviceSynchronize();
  try {
    Drv &d = drv();
    if (n->mcva) { d.cuMemUnmap(n->mcva, n->size); d.cuMemAddressFree(n->mcva, n->size); }
    if (n->uc) { d.cuMemUnmap(n->uc, n->size); d.cuMemAddressFree(n->uc, n->size); }
    if (n->bound) { CUdevice dev; d.cuDeviceGet(&dev, n->device); d.cuMulticastUnbind(n->mc, dev, 0, n->size); }
    if (n->have_mem) d.cuMemRelease(n->mem);
    if (n->have_mc) d.cuMemRelease(n->mc);
  } catch (...) {
  }
  if (n->mc_fd >= 0) close(n->mc_fd);
  cudaFree(n->dev_words);
  delete n;
  return AR_OK;
}

}  // extern "C"
