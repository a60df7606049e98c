// sm_100a kernels of the H-SADMM synchronization step (see hsx_kernels.cuh).
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <utility>

#include "hsx_kernels.cuh"

namespace hsx {

constexpr unsigned kFull = 0xffffffffu;
constexpr int kThreads = 256;

// opt a kernel into large dynamic shared memory (dynamic + static must fit the
// per-block limit, so anything above 32 KB opts in); the attribute is per device
// and kernel, so one driver call per (device, kernel, size), remembered in a
// small table (a process may drive several GPUs)
constexpr int kMaxDevices = 16;
static int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev < 0 ? 0 : dev % kMaxDevices;
}
template <typename K>
static void allow_smem(K kernel, size_t bytes) {
  constexpr int kSlots = 64;
  static const void* keys[kSlots];
  static int devs[kSlots];
  static size_t granted[kSlots];
  if (bytes <= 32 * 1024) return;
  const void* key = reinterpret_cast<const void*>(kernel);
  const int dev = current_device();
  int slot = 0;
  while (slot < kSlots && keys[slot] && !(keys[slot] == key && devs[slot] == dev)) ++slot;
  if (slot < kSlots && keys[slot] == key && devs[slot] == dev && granted[slot] >= bytes) return;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (slot < kSlots) {
    keys[slot] = key;
    devs[slot] = dev;
    granted[slot] = bytes;
  }
}

// Programmatic dependent launch: the chain kernels are launched with
// programmatic stream serialization, so a kernel's launch and CTA rasterization
// overlap the tail of its predecessor. Every such kernel calls pdl_wait() first,
// unconditionally (completion of a grid then implies completion of everything
// before it in the stream), then pdl_trigger() so its successor may be scheduled
// once all of its CTAs are running.
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }
#define PDL_ENTRY() \
  do {              \
    pdl_wait();     \
    pdl_trigger();  \
  } while (0)

template <typename... P, typename... A>
static void launch_pdl(void (*kernel)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t st, A&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  static const bool pdl = [] {
    const char* v = std::getenv("HSX_PDL");
    return !(v && v[0] == '0');
  }();
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl ? 1 : 0;
  cudaLaunchKernelEx(&cfg, kernel, std::forward<A>(args)...);
}

// streaming 128-bit load of data read exactly once (evict-first)
__device__ __forceinline__ float4 ldcs4(const float* p) {
  return __ldcs(reinterpret_cast<const float4*>(p));
}
__device__ __forceinline__ void st4(float* p, float4 v) { *reinterpret_cast<float4*>(p) = v; }

// L2 eviction-priority hints (createpolicy, on the cp.async loads): within a step
// z_node is read by K3, K6 and K7 and the compact buffer by K7, so those are
// re-read evict_last and stay resident in the 126 MB L2, while single-use
// streams are read evict_first and written with st.global.cs (evict-first
// stores). The policy must be warp-uniform (it becomes the load's memory
// descriptor), so it is a compile-time choice; -DHSX_NO_L2_HINTS builds the
// evict_normal (= no hint) variant for A/B runs.
enum { kL2First = 0, kL2Last = 1 };
__device__ __forceinline__ unsigned long long l2pol(int kind) {
  unsigned long long p;
#ifdef HSX_NO_L2_HINTS
  (void)kind;
  asm("createpolicy.fractional.L2::evict_normal.b64 %0, 1.0;" : "=l"(p));
#else
  if (kind == kL2Last)
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  else
    asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ void stcs4(float* p, float4 v) { __stcs(reinterpret_cast<float4*>(p), v); }
__device__ __forceinline__ float f4get(const float4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}
__device__ __forceinline__ void f4set(float4& v, int i, float x) {
  if (i == 0) v.x = x; else if (i == 1) v.y = x; else if (i == 2) v.z = x; else v.w = x;
}
__device__ __forceinline__ int i4get(const int4& v, int i) {
  return i == 0 ? v.x : (i == 1 ? v.y : (i == 2 ? v.z : v.w));
}

// u + (a - b) in fp64, rounded once (dual updates, consensus.py:186 / :505)
__device__ __forceinline__ float dual1(float u, float a, float b) {
  return (float)__dadd_rn((double)u, __dsub_rn((double)a, (double)b));
}

// ---------------------------------------------------------------------------
// Per-thread cp.async (LDGSTS) rings. A streaming kernel gives every thread a
// sequence of element quads; the thread keeps kDepth-1 quads' loads in flight
// in its private shared-memory slots (no registers held, no block barriers:
// a thread only reads slots it filled itself, visible after cp.async.wait_group).
// Dropped coordinates of a gather are zero-filled by the copy engine
// (src-size 0) instead of being read.
// ---------------------------------------------------------------------------

constexpr int kDepth = 4;

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void cp16(float4* dst, const float* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp16h(float4* dst, const float* src, unsigned long long pol) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "l"(pol)
               : "memory");
}
// 4-byte copy, zero-fill when !valid (the global address is not dereferenced)
__device__ __forceinline__ void cp4z(float* dst, const float* src, bool valid) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(valid ? 4 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// TMA 1-D bulk copies (global -> shared, completion counted in bytes on an mbarrier)
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// slot (stage d, buffer b) of this thread in a [kDepth][NB][kThreads] float4 ring
template <int NB>
__device__ __forceinline__ float4* ring_slot(float4* ring, int d, int b) {
  return ring + ((d * NB + b) * kThreads + threadIdx.x);
}

// quad (4 consecutive elements at e) of `src` into a slot; partial quads past n
// are zero-filled element-wise
__device__ __forceinline__ void cp_quad_h(float4* dst, const float* src, long long e, long long n,
                                          unsigned long long pol) {
  if (e + 3 < n) {
    cp16h(dst, src + e, pol);
  } else {
    float* d = reinterpret_cast<float*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) cp4z(d + i, src + (e + i < n ? e + i : 0), e + i < n);
  }
}
__device__ __forceinline__ void cp_quad(float4* dst, const float* src, long long e, long long n) {
  if (e + 3 < n) {
    cp16(dst, src + e);
  } else {
    float* d = reinterpret_cast<float*>(dst);
#pragma unroll
    for (int i = 0; i < 4; ++i) cp4z(d + i, src + (e + i < n ? e + i : 0), e + i < n);
  }
}

// Drive `count` iterations of (issue(slot, i), consume(slot, i)) through the ring:
// ring_prologue puts the first kDepth-1 quads in flight (a kernel can do other
// setup before ring_loop), ring_run does both.
template <int D = kDepth, class Issue>
__device__ __forceinline__ void ring_prologue(int count, Issue issue) {
#pragma unroll
  for (int d = 0; d < D - 1; ++d) {
    if (d < count) issue(d, d);
    cp_commit();
  }
}
template <int D = kDepth, class Issue, class Consume>
__device__ __forceinline__ void ring_loop(int count, Issue issue, Consume consume) {
  for (int i = 0; i < count; ++i) {
    const int ahead = i + D - 1;
    if (ahead < count) issue(ahead % D, ahead);
    cp_commit();
    cp_wait<D - 1>();
    consume(i % D, i);
  }
}
template <int D = kDepth, class Issue, class Consume>
__device__ __forceinline__ void ring_run(int count, Issue issue, Consume consume) {
  ring_prologue<D>(count, issue);
  ring_loop<D>(count, issue, consume);
}

// ---------------------------------------------------------------------------
// Keep sets (shrinkage.py:45-58 derive_keep_sets; sparsity.py:118-122 drift
// numerator; transport.py:239-280 concatenation order). Two derivations:
//  * from mask bits (K5, any M): every CTA marks the K_out / K_in "any" flags
//    of its word range and accumulates popcount(mask) and popcount(mask ^ prev)
//    per layer; the layer's last CTA scans the flags (keep_sets_tail);
//  * structured (one node, M == 1: the union is the local mask kept && z != 0):
//    the mask is the rectangle R x C of kept rows x kept columns unless a kept
//    element is exactly zero, so the selection's last pass derives K_out = R,
//    K_in = channels meeting C, the popcount |R||C| and the drift against the
//    previous rectangle straight from the group flags (structured_keep_sets, in
//    the K1 / K2 tail). K3 flags layers with a kept zero ("irregular");
//    k_keep_fixup re-derives those exactly from their mask bits.
// Both write positions, payload maps and the summary row of the layer; the last
// layer to finish lays out the flat buffer (exclusive scan of payload sizes in
// layer order). Flags and accumulators are left zeroed (no memsets).
// ---------------------------------------------------------------------------

// block-wide exclusive prefix sum of one int per thread (blockDim <= 1024)
__device__ int block_exclusive_scan(int x, int* warp_tot, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = x;
#pragma unroll
  for (int off = 1; off < 32; off <<= 1) {
    int y = __shfl_up_sync(kFull, incl, off);
    if (lane >= off) incl += y;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int nw = blockDim.x >> 5;
    int t = lane < nw ? warp_tot[lane] : 0;
    int ti = t;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      int y = __shfl_up_sync(kFull, ti, off);
      if (lane >= off) ti += y;
    }
    if (lane < nw) warp_tot[lane] = ti - t;
    if (lane == 31) *total = ti;
  }
  __syncthreads();
  int r = incl - x + warp_tot[warp];
  __syncthreads();
  return r;
}

// block-wide sums of two values per thread (one pass), results in every thread
__device__ ulonglong2 block_sum2(unsigned long long x, unsigned long long y) {
  __shared__ ulonglong2 wsum2[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    x += __shfl_xor_sync(kFull, x, off);
    y += __shfl_xor_sync(kFull, y, off);
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum2[warp] = make_ulonglong2(x, y);
  __syncthreads();
  if (warp == 0) {  // warp 0 folds the warp sums, then broadcasts through slot 0
    const bool in = lane < (int)(blockDim.x >> 5);
    unsigned long long a = in ? wsum2[lane].x : 0ull, b = in ? wsum2[lane].y : 0ull;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      a += __shfl_xor_sync(kFull, a, off);
      b += __shfl_xor_sync(kFull, b, off);
    }
    __syncwarp();
    if (lane == 0) wsum2[0] = make_ulonglong2(a, b);
  }
  __syncthreads();
  const ulonglong2 s = wsum2[0];
  __syncthreads();
  return s;
}

// block-wide sum of one value per thread, result in every thread
template <typename T>
__device__ T block_sum(T x) {
  __shared__ T wsum[32];
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0) wsum[warp] = x;
  __syncthreads();
  T s = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) s += wsum[w];
  __syncthreads();
  return s;
}

// flag byte i: through L2 when written by other CTAs of the launch, plain when
// in shared memory
template <bool SMEM>
__device__ __forceinline__ bool flag_at(const uint8_t* f, int i) {
  if constexpr (SMEM)
    return f[i] != 0;
  else
    return __ldcg(f + i) != 0;
}

// Positions of the set K_in / K_out flags of one layer (-1 for clear ones) in
// one block scan when every thread owns <= 8 consecutive flags of each array
// (the two counts packed in one int, 16 bits each), else in rounds; returns
// (|K_in|, |K_out|).
template <bool SMEM>
__device__ int2 scan_keep(const uint8_t* fin, int cin, const uint8_t* fout, int rows, int* pos_in, int* pos_out) {
  __shared__ int warp_tot[32];
  __shared__ int total;
  constexpr int kPer = 8;
  const int nt = blockDim.x, t = threadIdx.x;
  const int per = (max(cin, rows) + nt - 1) / nt;
  if (per <= 1) {  // one flag of each array per thread
    const bool fi = t < cin && flag_at<SMEM>(fin, t);
    const bool fo = t < rows && flag_at<SMEM>(fout, t);
    const int ex = block_exclusive_scan((int)fi | ((int)fo << 16), warp_tot, &total);
    const int tot = total;
    if (t < cin) pos_in[t] = fi ? (ex & 0xffff) : -1;
    if (t < rows) pos_out[t] = fo ? (ex >> 16) : -1;
    __syncthreads();
    return make_int2(tot & 0xffff, tot >> 16);
  }
  if (per <= kPer) {
    bool fi[kPer], fo[kPer];
    int ci = 0, co = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int x = t * per + i;
      fi[i] = i < per && x < cin && flag_at<SMEM>(fin, x);
      fo[i] = i < per && x < rows && flag_at<SMEM>(fout, x);
      ci += fi[i];
      co += fo[i];
    }
    const int ex = block_exclusive_scan(ci | (co << 16), warp_tot, &total);
    const int tot = total;
    int pi = ex & 0xffff, po = ex >> 16;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
      const int x = t * per + i;
      if (i < per && x < cin) pos_in[x] = fi[i] ? pi++ : -1;
      if (i < per && x < rows) pos_out[x] = fo[i] ? po++ : -1;
    }
    __syncthreads();
    return make_int2(tot & 0xffff, tot >> 16);
  }
  int n[2];
  for (int a = 0; a < 2; ++a) {
    const uint8_t* f = a ? fout : fin;
    const int m = a ? rows : cin;
    int* pos = a ? pos_out : pos_in;
    int carry = 0;
    for (int base = 0; base < m; base += nt) {
      const int i = base + t;
      const int fr = (i < m && flag_at<SMEM>(f, i)) ? 1 : 0;
      const int ex = block_exclusive_scan(fr, warp_tot, &total);
      if (i < m) pos[i] = fr ? carry + ex : -1;
      carry += total;
    }
    n[a] = carry;
  }
  __syncthreads();
  return make_int2(n[0], n[1]);
}

// flat-buffer layout: exclusive scan of the payload sizes of all layers (block-wide)
__device__ void layout_flat(const KeepArgs& a) {
  __shared__ long long wsum[32];
  __shared__ long long carry;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nt = blockDim.x;
  for (int base = 0; base < a.n_layers; base += nt) {
    int i = base + threadIdx.x;
    volatile long long* ri = a.summary + (long long)i * kSumCols;
    long long e = i < a.n_layers ? ri[2] : 0;
    long long incl = e;
#pragma unroll
    for (int off = 1; off < 32; off <<= 1) {
      long long y = __shfl_up_sync(kFull, incl, off);
      if (lane >= off) incl += y;
    }
    if (lane == 31) wsum[warp] = incl;
    __syncthreads();
    if (warp == 0) {
      long long t = lane < nt / 32 ? wsum[lane] : 0, ti = t;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        long long y = __shfl_up_sync(kFull, ti, off);
        if (lane >= off) ti += y;
      }
      wsum[lane] = ti - t;
    }
    __syncthreads();
    long long ex = carry + wsum[warp] + incl - e;
    if (i < a.n_layers) ri[3] = ex;
    __syncthreads();
    if (threadIdx.x == nt - 1) carry = ex + e;
    __syncthreads();
  }
  if (threadIdx.x == 0) a.summary[(long long)a.n_layers * kSumCols] = carry;
}

// summary row of layer l, then count the layer done; the last one lays out the
// flat buffer. One gpu-scope fence by thread 0 releases the block's writes.
__device__ void finish_layer(const KeepArgs& a, int l, int n_out, int n_in, int k, long long drift,
                             long long pop) {
  __shared__ bool last_layer;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long* row = a.summary + (long long)l * kSumCols;
    row[0] = n_out;
    row[1] = n_in;
    row[2] = (long long)n_out * n_in * k;
    row[4] = drift;
    row[5] = pop;
    __threadfence();
    last_layer = atomicAdd(a.done, 1u) == (unsigned)a.n_prunable - 1;
  }
  __syncthreads();
  if (!last_layer) return;
  __threadfence();
  layout_flat(a);
  if (threadIdx.x == 0) *a.done = 0;
}

// K5 tail, run by the last CTA of layer l: keep sets from the global any-flags
__device__ void keep_sets_tail(const KeepArgs& a, int l, const DevLayer& gly) {
  // layer fields in registers: the flag stores below may alias the table
  const int cin = gly.cin, rows = gly.rows, k = gly.k, pidx = gly.pidx;
  const long long ikeep = gly.ikeep, okeep = gly.okeep;
  const int2 nio = scan_keep<false>(a.iflag + ikeep, cin, a.oflag + okeep, rows, a.pos_in + ikeep, a.pos_out + okeep);
  // leave the any-flags zeroed for the next derivation
  for (int i = threadIdx.x; i < cin; i += blockDim.x) a.iflag[ikeep + i] = 0;
  for (int i = threadIdx.x; i < rows; i += blockDim.x) a.oflag[okeep + i] = 0;
  long long drift = 0, pop = 0;
  if (threadIdx.x == 0) {
    drift = (long long)atomicExch(a.acc + 2 * pidx, 0ULL);
    pop = (long long)atomicExch(a.acc + 2 * pidx + 1, 0ULL);
    a.layer_done[pidx] = 0;
  }
  finish_layer(a, l, nio.y, nio.x, k, drift, pop);
}

// end of a K5 marking CTA: fold its popcounts into the layer's accumulators, then
// count it done; the layer's last CTA runs the tail
__device__ void keep_mark_done(const KeepArgs& a, int l, const DevLayer& ly, int nitems,
                               unsigned long long pop, unsigned long long drift) {
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
    pop += __shfl_xor_sync(kFull, pop, off);
    drift += __shfl_xor_sync(kFull, drift, off);
  }
  if ((threadIdx.x & 31) == 0) {
    if (drift) atomicAdd(a.acc + 2 * ly.pidx, drift);
    if (pop) atomicAdd(a.acc + 2 * ly.pidx + 1, pop);
  }
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.layer_done + ly.pidx, 1u) == (unsigned)nitems - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  keep_sets_tail(a, l, ly);
}

// Structured keep sets of layer l at its last selection pass (one node): the
// rectangle R x C from the group flags (this pass in sflag, earlier passes in
// global memory). C is a set of whole channels unless the layer has SHAPE
// groups, so the work is O(rows + c_in) (O(rows + L) with SHAPE groups).
// Updates the previous-rectangle state (rk_prev, ch_prev / ck_prev).
// smem: structured_smem(rows, L, c_in) bytes.
__host__ __device__ inline size_t structured_smem(int rows, int L, int cin) {
  return ((size_t)rows + cin + L + 15) / 16 * 16;
}

// previous-rectangle flags of the layer (rows, then channels or columns) staged
// into shared memory by cp.async at the start of the selection, so their loads
// overlap the norms and the top-k (16-B chunks: okeep / ikeep / cpoff are
// 16-B aligned per layer); waited for in structured_keep_sets
__host__ __device__ inline size_t prev_stage_bytes(int rows, int cin, int L, bool shape) {
  return ((size_t)rows + 15) / 16 * 16 + ((size_t)(shape ? L : cin) + 15) / 16 * 16;
}

__host__ __device__ inline size_t structured_bytes(int rows, int L, int cin) {
  return structured_smem(rows, L, cin) + prev_stage_bytes(rows, cin, L, true) + 16;
}

__device__ void stage_prev(const KeepArgs& a, const DevLayer& gly, uint8_t* stage) {
  bool shape = false;
  for (int q = 0; q < gly.ncons; ++q) shape |= gly.group[q] == kShape;
  const int rows = gly.rows, ncol = shape ? gly.L : gly.cin;
  const int nr = (rows + 15) / 16, nc = (ncol + 15) / 16;
  const uint8_t* src_r = a.rk_prev + gly.okeep;
  const uint8_t* src_c = shape ? a.ck_prev + gly.cpoff : a.ch_prev + gly.ikeep;
  for (int i = threadIdx.x; i < nr + nc; i += blockDim.x) {
    const uint8_t* src = i < nr ? src_r + 16 * i : src_c + 16 * (i - nr);
    uint8_t* dst = stage + 16 * i;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
  }
  cp_commit();
}

__device__ void structured_keep_sets(const KeepArgs& a, int l, const DevLayer& gly, int pass,
                                     const uint8_t* sflag, uint8_t* smem, const uint8_t* stage) {
  const int cin = gly.cin, rows = gly.rows, k = gly.k, L = gly.L, npass = gly.ncons;
  const long long ikeep = gly.ikeep, okeep = gly.okeep, cpoff = gly.cpoff;
  const FastDiv divk = gly.divk;
  int gq[kMaxPasses];
  const uint8_t* fq[kMaxPasses];
  bool shape = false;
#pragma unroll
  for (int q = 0; q < kMaxPasses; ++q) {
    gq[q] = q < npass ? gly.group[q] : -1;
    fq[q] = q < npass ? a.flags.f[q] + gly.goff[q] : nullptr;
    shape |= gq[q] == kShape;
  }
#ifdef HSX_PROBE_SELECT
  long long tq[8];
  tq[0] = clock64();
#define ST_MARK(i) do { __syncthreads(); tq[i] = clock64(); } while (0)
#else
#define ST_MARK(i) do { } while (0)
#endif
  uint8_t* srk = smem;        // R
  uint8_t* sch = srk + rows;  // channels meeting C
  uint8_t* sck = sch + cin;   // C by column (SHAPE groups)
  const uint8_t* prev_r = stage;                          // staged rk_prev
  const uint8_t* prev_c = stage + (rows + 15) / 16 * 16;  // staged ch_prev / ck_prev
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  // three counts packed per word (21 bits each; rows, columns < 2^20)
  unsigned long long rsum = 0, csum = 0;
  for (int o = threadIdx.x; o < rows; o += blockDim.x) {
    uint8_t kp = 1;
#pragma unroll
    for (int q = 0; q < kMaxPasses; ++q)
      if (gq[q] == kFilter) kp &= q == pass ? sflag[o] : fq[q][o];
    const uint8_t pv = prev_r[o];
    srk[o] = kp;
    a.rk_prev[okeep + o] = kp;
    rsum += (unsigned long long)kp | ((unsigned long long)pv << 21) | ((unsigned long long)(kp & pv) << 42);
  }
  if (!shape) {  // C = the channels kept by every CHANNEL pass, all kh*kw columns each
    for (int c = threadIdx.x; c < cin; c += blockDim.x) {
      uint8_t kp = 1;
#pragma unroll
      for (int q = 0; q < kMaxPasses; ++q)
        if (gq[q] == kChannel) kp &= q == pass ? sflag[c] : fq[q][c];
      const uint8_t pv = prev_c[c];
      sch[c] = kp;
      a.ch_prev[ikeep + c] = kp;
      csum += (unsigned long long)kp | ((unsigned long long)pv << 21) | ((unsigned long long)(kp & pv) << 42);
    }
  } else {
    for (int col = threadIdx.x; col < L; col += blockDim.x) {
      const int c = (int)fdiv((unsigned)col, divk);
      uint8_t kp = 1;
#pragma unroll
      for (int q = 0; q < kMaxPasses; ++q) {
        if (gq[q] != kChannel && gq[q] != kShape) continue;
        const int g = gq[q] == kChannel ? c : col;
        kp &= q == pass ? sflag[g] : fq[q][g];
      }
      const uint8_t pv = prev_c[col];
      sck[col] = kp;
      a.ck_prev[cpoff + col] = kp;
      csum += (unsigned long long)kp | ((unsigned long long)pv << 21) | ((unsigned long long)(kp & pv) << 42);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < cin; c += blockDim.x) {
      uint8_t any = 0;
      for (int jx = 0; jx < k; ++jx) any |= sck[c * k + jx];
      sch[c] = any;
    }
  }
  ST_MARK(1);
  {
    const ulonglong2 t = block_sum2(rsum, csum);
    rsum = t.x;
    csum = t.y;
  }
  ST_MARK(2);
  constexpr unsigned long long m21 = (1ULL << 21) - 1;
  const long long cm = shape ? 1 : k;  // columns per counted unit
  const long long nR = rsum & m21, nRp = (rsum >> 21) & m21, nRR = rsum >> 42;
  const long long nC = cm * (csum & m21), nCp = cm * ((csum >> 21) & m21), nCC = cm * (csum >> 42);
  // K_out = R when C is non-empty; K_in = channels meeting C when R is non-empty
  if (nC == 0)
    for (int o = threadIdx.x; o < rows; o += blockDim.x) srk[o] = 0;
  if (nR == 0)
    for (int c = threadIdx.x; c < cin; c += blockDim.x) sch[c] = 0;
  __syncthreads();
  ST_MARK(3);
  const int2 nio = scan_keep<true>(sch, cin, srk, rows, a.pos_in + ikeep, a.pos_out + okeep);
  ST_MARK(4);
  // |A ^ B| = |A| + |B| - 2 |A n B| for rectangles A = R x C, B = Rp x Cp
  const long long pop = nR * nC;
  const long long drift = pop + nRp * nCp - 2 * nRR * nCC;
  finish_layer(a, l, nio.y, nio.x, k, drift, pop);
#ifdef HSX_PROBE_SELECT
  ST_MARK(5);
  if (threadIdx.x == 0)
    printf("structured l=%d rows=%d cin=%d nt=%d: RC %lld sums %lld zero %lld scan %lld finish %lld\n", l, rows, cin,
           (int)blockDim.x, tq[1] - tq[0], tq[2] - tq[1], tq[3] - tq[2], tq[4] - tq[3], tq[5] - tq[4]);
#endif
}

// ---------------------------------------------------------------------------
// K2 select: norms = sqrt(sum of partials); keep the `keep` largest groups, lower
// index on ties (SparsityConstraint.resolve + _kept_group_indices,
// sparsity.py:53-68). One block per layer. Runs in the tail of the layer's last
// K1 tile when its keys fit the candidate kernel's shared memory
// (DevLayer::fsel), else as its own launch.
// ---------------------------------------------------------------------------

// Top-`keep` of G non-negative fp64 norms. Their bit patterns order like the
// values, so an 8-bit MSD radix select over the 64-bit keys narrows to the bin
// holding the keep-th largest key, one byte per round (O(G) per round, vs O(G^2)
// rank counting or O(G log^2 G) barriers of a bitonic sort). It stops as soon
// as every candidate of the chosen bin is kept (distinct norms: 2-3 rounds).
// Groups above the bin are kept; when the full 64-bit key T is reached with
// more equal keys than slots, the lowest-index ones fill the remainder (the
// stable argsort of -norms). Writes the 0/1 flags into sflag[G].
__device__ void radix_top_k(const unsigned long long* __restrict__ key, int G, int keep, uint8_t* sflag) {
  __shared__ __align__(16) int hist[2][256];  // bin 255 - digit: lanes scan descending digits
  __shared__ unsigned long long s_prefix;
  __shared__ int s_rem, s_eq;
  __shared__ int warp_tot[32];
  __shared__ int total;
  const int t = threadIdx.x, nt = blockDim.x;
  __shared__ unsigned long long s_diff[32];
  unsigned long long prefix = 0, himask = 0;
  int rem = keep, eq = G, buf = 0;
  for (int i = t; i < 256; i += nt) hist[0][i] = 0;
  // bytes above the highest one where any two keys differ are common to all keys:
  // start the radix rounds there (norms of a layer share sign and exponent bytes)
  {
    const unsigned long long k0 = key[0];
    unsigned long long d = 0;
    for (int g = t; g < G; g += nt) d |= key[g] ^ k0;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) d |= __shfl_xor_sync(kFull, d, off);
    if ((t & 31) == 0) s_diff[t >> 5] = d;
    __syncthreads();
    d = 0;
    for (int w = 0; w < (nt >> 5); ++w) d |= s_diff[w];
    const int top = d ? 63 - __clzll((long long)d) : 0;  // highest differing bit
    const int first = (top >> 3) << 3;                     // its byte's shift
    himask = first >= 56 ? 0ull : (~0ull << (first + 8));
    prefix = k0 & himask;
    s_prefix = prefix;  // (unused until written by a round)
    __syncthreads();
    buf = 0;
    // the first round below starts at `first`
    rem = keep;
    eq = G;
    for (int shift = first;; shift -= 8) {
    // norms of one layer share their top bytes: warp-aggregate equal bins so a
    // round costs G/32 shared atomics instead of G serialized on one address
    for (int g0 = t - (t & 31); g0 < G; g0 += nt) {
      const int g = g0 + (t & 31);
      int bin = -1 - (t & 31);  // unique non-bin for lanes past G / off the prefix
      if (g < G) {
        const unsigned long long x = key[g];
        if ((x & himask) == prefix) bin = 255 - ((int)(x >> shift) & 255);
      }
      const unsigned same = __match_any_sync(kFull, bin);
      if (bin >= 0 && (t & 31) == __ffs(same) - 1) atomicAdd(&hist[buf][bin], __popc(same));
    }
    for (int i = t; i < 256; i += nt) hist[buf ^ 1][i] = 0;  // next round's bins
    __syncthreads();
    if (t < 32) {
      const int4 h0 = *reinterpret_cast<const int4*>(&hist[buf][8 * t]);
      const int4 h1 = *reinterpret_cast<const int4*>(&hist[buf][8 * t + 4]);
      const int c[8] = {h0.x, h0.y, h0.z, h0.w, h1.x, h1.y, h1.z, h1.w};  // digits 255-8t-b
      const int sum = ((c[0] + c[1]) + (c[2] + c[3])) + ((c[4] + c[5]) + (c[6] + c[7]));
      int incl = sum;
#pragma unroll
      for (int off = 1; off < 32; off <<= 1) {
        const int y = __shfl_up_sync(kFull, incl, off);
        if (t >= off) incl += y;
      }
      const int excl = incl - sum;
      const unsigned owner = __ballot_sync(kFull, excl < rem && rem <= incl);
      if (t == __ffs(owner) - 1) {
        int before = excl;
#pragma unroll
        for (int b = 0; b < 8; ++b) {
          if (before < rem && rem <= before + c[b]) {
            s_prefix = prefix | ((unsigned long long)(255 - 8 * t - b) << shift);
            s_rem = rem - before;
            s_eq = c[b];
          }
          before += c[b];
        }
      }
    }
    __syncthreads();
    prefix = s_prefix;
    rem = s_rem;
    eq = s_eq;
    himask |= 0xffULL << shift;
    if (rem == eq || shift == 0) break;
    buf ^= 1;
  }
  }
  if (rem == eq) {  // every candidate of the bin is kept
    for (int g = t; g < G; g += nt) sflag[g] = (key[g] & himask) >= prefix;
    return;
  }
  const unsigned long long T = prefix;  // exact key with ties: index-order ranks among them
  int carry = 0;
  for (int base = 0; base < G; base += nt) {
    const int g = base + t;
    const int e = (g < G && key[g] == T) ? 1 : 0;
    const int ex = block_exclusive_scan(e, warp_tot, &total);
    if (g < G) sflag[g] = key[g] > T || (e && carry + ex < rem);
    carry += total;
  }
}

// One layer's selection by the whole block; K1 partials are read through L2 (in
// the fused form other CTAs of the same launch wrote them). Partials are per
// group: [nparts][G] (FILTER: [G], complete row sums), folded in part order.
// shared memory: keys[G] (u64), flags[G] (u8)
__host__ __device__ inline size_t select_bytes(int G) { return ((size_t)G * 9 + 15) / 16 * 16; }
constexpr int kFoldCols = 8192;  // column totals staged per norm chunk (64 KB): one chunk for 512 x 3x3 groups

__device__ void select_layer(const DevLayer& gly, int pass, const double* __restrict__ partials,
                             double* __restrict__ norms, const FlagPtrs& flags, void* smem, int l,
                             const KeepArgs* ka) {
  // layer fields in registers: the byte stores below may alias the layer table
  const int G = gly.G[pass], grp = gly.group[pass], keep = gly.keep[pass];
  const int nparts = grp == kFilter ? 1 : gly.nparts;
  const int kc = (grp == kChannel && gly.percol) ? gly.k : 1;  // per-column partials: fold kh*kw columns
  const int pstride = kc > 1 ? gly.L : G;
  const long long goff = gly.goff[pass];
  const double* __restrict__ part = partials + gly.poff[pass];
  unsigned long long* skey = reinterpret_cast<unsigned long long*>(smem);
  uint8_t* sflag = reinterpret_cast<uint8_t*>(skey + G);
  const int nt = blockDim.x;
  const int t = threadIdx.x;
  const bool structured = ka != nullptr && pass == gly.ncons - 1;
  uint8_t* stage = reinterpret_cast<uint8_t*>(smem) + select_bytes(G) +
                   structured_smem(gly.rows, gly.L, gly.cin);
  if (structured) stage_prev(*ka, gly, stage);
#ifdef HSX_PROBE_SELECT
  long long tm[6];
  tm[0] = clock64();
#define SEL_MARK(i) do { __syncthreads(); tm[i] = clock64(); } while (0)
#else
#define SEL_MARK(i) do { } while (0)
#endif
  // 1) norms, in column chunks of kFoldCols: each column's nparts partials are
  // summed in part order (coalesced across threads, all of a thread's loads in
  // flight together: the tail runs beside streaming CTAs, where every dependent
  // L2 round trip costs ~1 us), then each group adds its kc column totals in
  // column order from shared memory. Fixed order: deterministic.
  double* colsum = reinterpret_cast<double*>(reinterpret_cast<uint8_t*>(smem) + select_bytes(G) +
                                             structured_bytes(gly.rows, gly.L, gly.cin));
  const int chunk_g = max(1, kFoldCols / kc);
  for (int g0 = 0; g0 < G; g0 += chunk_g) {
    const int ng = min(chunk_g, G - g0), nc = ng * kc;
    const double* __restrict__ pc = part + (long long)g0 * kc;
    if (nparts <= 4) {  // 4 columns x <= 4 parts per thread in flight together
      for (int c0 = t; c0 < nc; c0 += 4 * nt) {
        double v[4][4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
#pragma unroll
          for (int q = 0; q < 4; ++q)
            v[u][q] = (q < nparts && c0 + u * nt < nc) ? __ldcg(pc + (long long)q * pstride + c0 + u * nt) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          double s2 = v[u][0];
#pragma unroll
          for (int q = 1; q < 4; ++q)
            if (q < nparts) s2 += v[u][q];
          if (c0 + u * nt < nc) colsum[c0 + u * nt] = s2;
        }
      }
    } else {
      for (int c = t; c < nc; c += nt) {
        double s2 = 0.0;
        for (int p0 = 0; p0 < nparts; p0 += 16) {
          double v[16];
#pragma unroll
          for (int u = 0; u < 16; ++u) v[u] = p0 + u < nparts ? __ldcg(pc + (long long)(p0 + u) * pstride + c) : 0.0;
#pragma unroll
          for (int u = 0; u < 16; ++u)
            if (p0 + u < nparts) s2 += v[u];
        }
        colsum[c] = s2;
      }
    }
    __syncthreads();
    for (int g = t; g < ng; g += nt) {
      double s2 = colsum[g * kc];
      for (int jx = 1; jx < kc; ++jx) s2 += colsum[g * kc + jx];
      const double nrm = sqrt(s2);
      norms[goff + g0 + g] = nrm;
      skey[g0 + g] = (unsigned long long)__double_as_longlong(nrm);
    }
    __syncthreads();
  }
  __syncthreads();
  SEL_MARK(1);
  // 2) top-k flags
  radix_top_k(skey, G, keep, sflag);
  __syncthreads();
  SEL_MARK(2);
  uint8_t* __restrict__ fl = flags.f[pass] + goff;
  for (int g = t; g < G; g += nt) fl[g] = sflag[g];
  SEL_MARK(3);
  if (structured)  // one node: keep sets of the rectangle
    structured_keep_sets(*ka, l, gly, pass, sflag, reinterpret_cast<uint8_t*>(smem) + select_bytes(G), stage);
#ifdef HSX_PROBE_SELECT
  SEL_MARK(4);
  if (t == 0)
    printf("select l=%d G=%d nparts=%d kc=%d nt=%d: norms %lld topk %lld flags %lld keepsets %lld cycles\n", l, G,
           nparts, kc, nt, tm[1] - tm[0], tm[2] - tm[1], tm[3] - tm[2], tm[4] - tm[3]);
#endif
}

// Chained mode (k1done != nullptr): K2 is launched right behind K1 (programmatic
// dependent launch) and does not wait for K1's grid to complete before it starts:
// it lets its own dependents launch, each CTA waits for its layer's tiles only
// (K1 counts them into k1done with release semantics: fence + atomic), selects,
// and only then waits for K1's grid — so K2's completion still implies K1's and
// everything before it, while the selections of the layers K1 finished early run
// under K1's drain. K1 has started every CTA before K2 can launch (its CTAs
// trigger at entry), so the wait always makes progress.
__global__ void __launch_bounds__(1024) k_select(const DevLayer* __restrict__ layers,
                                                 const int* __restrict__ list, int pass,
                                                 const double* __restrict__ partials,
                                                 double* __restrict__ norms, FlagPtrs flags, KeepArgs ka,
                                                 int structured, unsigned int* __restrict__ k1done,
                                                 unsigned int* __restrict__ ready) {
  extern __shared__ unsigned long long skey[];
  const int l = list[blockIdx.x];
  if (k1done == nullptr) {
    PDL_ENTRY();
    select_layer(layers[l], pass, partials, norms, flags, skey, l, structured ? &ka : nullptr);
    return;
  }
  pdl_trigger();
  const DevLayer& ly = layers[l];
  unsigned* c = k1done + ly.pidx;
  if (threadIdx.x == 0) {
    unsigned v;
    for (;;) {
      // system scope: under a split two-rank K1 half of the counts (and partials) come
      // from the peer GPU
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(c) : "memory");
      if (v >= (unsigned)ly.ncitems) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
  select_layer(ly, pass, partials, norms, flags, skey, l, structured ? &ka : nullptr);
  __syncthreads();
  if (threadIdx.x == 0) {
    atomicSub(c, (unsigned)ly.ncitems);  // back to 0 for the next K1 (graph replays too)
    if (ready) {                          // a chained K3 projects this layer now
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(ready + l), "r"(1u) : "memory");
    }
  }
  pdl_wait();
}

// ---------------------------------------------------------------------------
// K1 candidate (+ group-norm partials).  consensus.py:142-160, tensors.py:75-93
// ---------------------------------------------------------------------------

// fp64 candidate; explicit _rn intrinsics (no FMA contraction) so the value is
// bit-identical to numpy's (rho1 * s + rho2 * (z - v)) / gamma.
struct Coef {
  double rho1, rho2, gamma, rgamma;
};

__device__ __forceinline__ Coef coef_of(const DevLayer& ly) {
  return Coef{ly.rho1, ly.rho2, ly.gamma, ly.rgamma};
}

// num / den, correctly rounded: q = RN(num * y) with y = RN(1/den), then one FMA
// residual correction (Markstein). Exactness vs IEEE division is checked bit for
// bit by tests/test_gpu_parity.py::test_candidate_division_is_ieee (hsx_selftest_division).
__device__ __forceinline__ double div_rn(double num, double den, double y) {
  double q = __dmul_rn(num, y);
  double r = __fma_rn(-q, den, num);
  return __fma_rn(r, y, q);
}

// fp64 candidate; explicit _rn intrinsics (no FMA contraction) so the value is
// numpy's (rho1 * s + rho2 * (z - v)) / gamma.
__device__ __forceinline__ double cand_of(double s, double z, double v, const Coef& cf) {
  double num = __dadd_rn(__dmul_rn(cf.rho1, s), __dmul_rn(cf.rho2, __dsub_rn(z, v)));
  return div_rn(num, cf.gamma, cf.rgamma);
}

// input modes of K1 (template parameter): the sum S is given (P > 1 through
// NCCL), is theta + u (P == 1: the intra all-reduce is the identity), is read
// from the P ranks' theta + u buffers over NVLink (kModePeers: the intra
// all-reduce fused into K1, folded in rank order like the reference's serial
// fold), or the candidate is S itself (kModeIdent: per-tensor projection API)
// (kModePeers2: exactly two ranks — a 4-slot ring stage like the local modes, so
// three CTAs fit per SM instead of two)
// (kModeSumDist: S is the P ranks' reduce-scatter slices, read from the owner of
// each quad over NVLink instead of all-gathered first)
enum { kModeThetaU = 0, kModeSum = 1, kModeIdent = 2, kModePeers = 3, kModePeers2 = 4, kModeSumDist = 5 };

__host__ __device__ constexpr bool peer_mode(int m) { return m == kModePeers || m == kModePeers2; }
__host__ __device__ constexpr int peer_slots(int m) { return m == kModePeers2 ? 2 : kMaxPeers; }

template <int MODE>
struct K1 {
  static constexpr int NB = peer_mode(MODE) ? peer_slots(MODE) + 2 : 4;  // ring slots per stage
  static constexpr int ZS = peer_mode(MODE) ? peer_slots(MODE) : 2;      // slot of z (v follows)
  // ring depth: two peers keep 5 stages in flight (more NVLink bytes in flight per
  // thread; 6 x 4 x 4 KB = 96 KB, two CTAs per SM)
  static constexpr int D = MODE == kModePeers2 ? 6 : kDepth;
};

// source pointers of one layer (offset already applied)
struct K1Src {
  const float* a;
  const float* b;
  const float* z;
  const float* v;
  const float* peer[kMaxPeers];
  long long bl[kMaxPeers];  // kModeSumDist: slice starts relative to this source's base
  int np;
};

// staged peer operand: 1 while this CTA's current item reads the peer's send directly
// (its staging copy had not landed), 0 otherwise (also for every unstaged launch)
__shared__ int s_k1_alt;

template <int MODE>
__device__ __forceinline__ K1Src k1_src(const CandArgs& p, long long base) {
  K1Src s;
  s.a = s.b = nullptr;
  s.np = 0;
  if (peer_mode(MODE) || MODE == kModeSumDist) {
    s.np = p.peers.n;
#pragma unroll
    for (int j = 0; j < kMaxPeers; ++j) s.peer[j] = j < s.np ? p.peers.p[j] + base : nullptr;
    if (MODE == kModeSumDist) {
#pragma unroll
      for (int j = 0; j < kMaxPeers; ++j) s.bl[j] = j < s.np ? p.sbound[j] - base : (1LL << 62);
    }
  } else {
    s.a = (MODE == kModeThetaU ? p.theta : p.s) + base;
    s.b = MODE == kModeThetaU ? (s_k1_alt ? p.u_alt : p.u) + base : nullptr;
  }
  s.z = MODE != kModeIdent ? p.z + base : nullptr;
  s.v = MODE != kModeIdent ? p.v + base : nullptr;
  return s;
}

// issue the quad at element e of every source into stage d (FULL: 16-B copies,
// the quad is known to be in range)
template <int MODE, bool FULL>
__device__ __forceinline__ void k1_issue(float4* ring, int d, const K1Src& s, long long e, long long n,
                                         unsigned long long pol) {
  constexpr int NB = K1<MODE>::NB;
  auto cp = [&](int slot, const float* src) {
    if (FULL)
      cp16h(ring_slot<NB>(ring, d, slot), src + e, pol);
    else
      cp_quad_h(ring_slot<NB>(ring, d, slot), src, e, n, pol);
  };
  // the peers' sends (one or more over NVLink) carry no L2 policy (with the evict-first
  // hint, HSX_PEER_HINT build, K1 read them at the same 470 GB/s, r2za)
  auto cpp = [&](int slot, const float* src) {
#ifdef HSX_PEER_HINT
    cp(slot, src);
#else
    if (FULL)
      cp16(ring_slot<NB>(ring, d, slot), src + e);
    else
      cp_quad(ring_slot<NB>(ring, d, slot), src, e, n);
#endif
  };
  if (peer_mode(MODE)) {
#pragma unroll
    for (int j = 0; j < peer_slots(MODE); ++j)
      if (j < s.np) cpp(j, s.peer[j]);
  } else if (MODE == kModeSumDist) {
    // the slice owner of this quad (slice bounds are multiples of 32 elements and
    // layers start 32-aligned, so a quad never straddles two slices)
    int o = 0;
#pragma unroll
    for (int j = 1; j < kMaxPeers; ++j) o += e >= s.bl[j] ? 1 : 0;
    const float* src = o == 0 ? s.peer[0] : o == 1 ? s.peer[1] : o == 2 ? s.peer[2] : s.peer[3];
    cpp(0, src);
  } else {
    cp(0, s.a);
    if (MODE == kModeThetaU) cp(1, s.b);
  }
  if (MODE != kModeIdent) {
    cp(K1<MODE>::ZS, s.z);
    cp(K1<MODE>::ZS + 1, s.v);
  }
}

// the four fp64 candidates of stage d
template <int MODE>
__device__ __forceinline__ void k1_cand(float4* ring, int d, int np, const Coef& cf, double c[4]) {
  constexpr int NB = K1<MODE>::NB;
  double s[4];
  if (peer_mode(MODE)) {
    const float4 x0 = *ring_slot<NB>(ring, d, 0);
    s[0] = x0.x; s[1] = x0.y; s[2] = x0.z; s[3] = x0.w;
#pragma unroll
    for (int j = 1; j < peer_slots(MODE); ++j) {
      if (j < np) {
        const float4 x = *ring_slot<NB>(ring, d, j);
        s[0] = __dadd_rn(s[0], (double)x.x); s[1] = __dadd_rn(s[1], (double)x.y);
        s[2] = __dadd_rn(s[2], (double)x.z); s[3] = __dadd_rn(s[3], (double)x.w);
      }
    }
  } else {
    const float4 a = *ring_slot<NB>(ring, d, 0);
    if (MODE == kModeThetaU) {
      const float4 b = *ring_slot<NB>(ring, d, 1);
      s[0] = __dadd_rn((double)a.x, (double)b.x); s[1] = __dadd_rn((double)a.y, (double)b.y);
      s[2] = __dadd_rn((double)a.z, (double)b.z); s[3] = __dadd_rn((double)a.w, (double)b.w);
    } else {
      s[0] = a.x; s[1] = a.y; s[2] = a.z; s[3] = a.w;
    }
  }
  if (MODE == kModeIdent) {
#pragma unroll
    for (int i = 0; i < 4; ++i) c[i] = s[i];
    return;
  }
  const float4 z = *ring_slot<NB>(ring, d, K1<MODE>::ZS), v = *ring_slot<NB>(ring, d, K1<MODE>::ZS + 1);
  c[0] = cand_of(s[0], z.x, v.x, cf);
  c[1] = cand_of(s[1], z.y, v.y, cf);
  c[2] = cand_of(s[2], z.z, v.z, cf);
  c[3] = cand_of(s[3], z.w, v.w, cf);
}

template <int MODE>
__device__ __forceinline__ double cand_elem(const CandArgs& p, long long gi, const Coef& cf) {
  double s;
  if (peer_mode(MODE)) {
    s = (double)p.peers.p[0][gi];
    for (int j = 1; j < p.peers.n; ++j) s = __dadd_rn(s, (double)p.peers.p[j][gi]);
  } else if (MODE == kModeThetaU) {
    s = __dadd_rn((double)p.theta[gi], (double)(s_k1_alt ? p.u_alt : p.u)[gi]);
  } else if (MODE == kModeSumDist) {
    int o = 0;
    for (int j = 1; j < p.peers.n; ++j) o += gi >= p.sbound[j] ? 1 : 0;
    s = (double)p.peers.p[o][gi];
  } else {
    s = (double)p.s[gi];
  }
  if (MODE == kModeIdent) return s;
  return cand_of(s, (double)p.z[gi], (double)p.v[gi], cf);
}

__device__ __forceinline__ int group_of(int grp, unsigned o, unsigned col, unsigned c) {
  return grp == kFilter ? (int)o : (grp == kChannel ? (int)c : (int)col);
}

// keep test of layer-local element e against passes [0, npass) (renorm passes only)
__device__ __forceinline__ bool kept_by(const DevLayer& ly, const uint8_t* const* flags, int npass,
                                        long long e) {
  unsigned o = fdiv((unsigned)e, ly.divL);
  unsigned col = (unsigned)e - o * (unsigned)ly.L;
  unsigned c = fdiv(col, ly.divk);
  bool keep = true;
  for (int q = 0; q < npass; ++q) keep = keep && flags[q][ly.goff[q] + group_of(ly.group[q], o, col, c)];
  return keep;
}

// K1a: elementwise candidate over [begin, end) of one layer (dense layers; every
// layer in frozen mode, where prunable layers get cand * global mask,
// consensus.py:177-180). Inputs stream through the per-thread cp.async ring.
template <int MODE>
__device__ void cand_elementwise(const CandArgs& p, const DevLayer& ly, long long begin, long long end,
                                 int frozen, float4* ring) {
  const bool masked = frozen && ly.ncons > 0 && p.fmask != nullptr;
  const long long nq = (end - begin + 3) >> 2;
  const int t = threadIdx.x;
  const Coef cf = coef_of(ly);
  const long long n = ly.n, off = ly.off, mword = ly.mword;
  const int count = t < nq ? (int)((nq - t + kThreads - 1) / kThreads) : 0;
  const K1Src src = k1_src<MODE>(p, off);
  float* zn = p.zn + off;
  const uint32_t* fm = masked ? p.fmask + mword : nullptr;
  const unsigned long long pf = l2pol(kL2First), pl = l2pol(kL2Last);
  ring_run<K1<MODE>::D>(
      count,
      [&](int d, int i) { k1_issue<MODE, false>(ring, d, src, begin + 4 * (t + (long long)i * kThreads), n, pf); },
      [&](int d, int i) {
        const long long e = begin + 4 * (t + (long long)i * kThreads);
        double c[4];
        k1_cand<MODE>(ring, d, src.np, cf, c);
        const uint32_t bits = fm ? fm[e >> 5] : 0u;
        float4 out;
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          double ci = c[i2];
          if (fm) ci = ((bits >> ((e + i2) & 31)) & 1u) ? ci : ci * 0.0;
          f4set(out, i2, (float)ci);
        }
        if (e + 3 < n) {
          st4(zn + e, out);  // z_node: re-read by K3 / K6 / K7 this step (normal priority)
        } else {
          for (int i2 = 0; i2 < 4 && e + i2 < n; ++i2) zn[e + i2] = f4get(out, i2);
        }
      });
}

// K1b quad tiles (CHANNEL / SHAPE groups, c_in*kh*kw % 4 == 0 — every ResNet conv
// but the 7x7 stem): a tile is rows x cq column quads (cq <= 64, 4*cq a multiple
// of kh*kw so a tile holds whole channels); thread t owns quad (t & 63) and row
// phase (t >> 6), so its fp64 column sums of squares stay in registers while
// its rows stream through the cp.async ring; the 4 phases fold in shared memory
// in a fixed order, then the kh*kw columns of each channel, and the tile writes
// one fp64 partial per group: partials[part][G].
constexpr int kTileQuads = 64;

// a quad tile of pass p.pass whose fold does not use the ring (no fused selection):
// the next such tile's first ring stages may go in flight under this tile's fold
__device__ __forceinline__ bool xtile_ok(const CandArgs& p, const Item& it) {
  const DevLayer& ly = p.layers[it.layer];
  return ly.ncons > p.pass && ly.tiling == 1 && !((ly.fsel >> p.pass) & 1);
}

// the first D-1 ring stages of quad tile `it` (this thread's share)
template <int MODE>
__device__ __forceinline__ void tile_quads_prologue(const CandArgs& p, const Item& it, float4* ring) {
  const DevLayer& ly = p.layers[it.layer];
  const int W = ly.cw, RP = kThreads / W, L = ly.L, cq = ly.cq;
  const int jj = threadIdx.x & (W - 1);
  const int j = it.chunk * cq + jj;
  const long long r0 = it.begin + threadIdx.x / W;
  const int count = (jj < cq && j < (L >> 2) && r0 < it.end) ? (int)((it.end - r0 + RP - 1) / RP) : 0;
  const K1Src src = k1_src<MODE>(p, ly.off + 4 * j);
  const long long stride = (long long)RP * L;
  const unsigned long long pf = l2pol(kL2First);
  ring_prologue<K1<MODE>::D>(
      count, [&](int d, int i) { k1_issue<MODE, true>(ring, d, src, r0 * L + i * stride, 0, pf); });
}

// xnext != nullptr (cross-tile mode): the prologue of this tile was issued by the
// previous one iff *pre; once this tile's loads are consumed, thread 0 claims the
// CTA's next item (claim()), and if it is a quad tile its first stages are issued
// before the fold; *xnext = the claimed index, *pre = whether they were issued.
template <int MODE, class Claim>
__device__ void cand_tile_quads(const CandArgs& p, const DevLayer& ly, const Item& it, float4* ring,
                                double* cs, bool* pre, int* xnext, Claim claim) {
  const int W = ly.cw;          // lanes per row (power of two)
  const int RP = kThreads / W;  // row phases
  const int pass = p.pass;
  const int L = ly.L;
  const int Q = L >> 2;
  const int cq = ly.cq;
  const int jj = threadIdx.x & (W - 1);
  const int ph = threadIdx.x / W;
  const int j = it.chunk * cq + jj;
  const long long r0 = it.begin + ph, r1 = it.end;
  const int count = (jj < cq && j < Q && r0 < r1) ? (int)((r1 - r0 + RP - 1) / RP) : 0;
  const long long off = ly.off;
  const K1Src src = k1_src<MODE>(p, off + 4 * j);
  float* zn = p.zn + off + 4 * j;
  float* znp = p.zn_peer ? p.zn_peer + off + 4 * j : nullptr;
  const Coef cf = coef_of(ly);
  const long long stride = (long long)RP * L;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  const unsigned long long pf = l2pol(kL2First), pl = l2pol(kL2Last);
  auto issue = [&](int d, int i) { k1_issue<MODE, true>(ring, d, src, r0 * L + i * stride, 0, pf); };
  if (!(xnext && *pre)) ring_prologue<K1<MODE>::D>(count, issue);
  ring_loop<K1<MODE>::D>(
      count, issue,
      [&](int d, int i) {
        const long long e = r0 * L + i * stride;
        double c[4];
        k1_cand<MODE>(ring, d, src.np, cf, c);
        if (pass > 0) {
          const long long ee = e + 4 * j;
#pragma unroll
          for (int i2 = 0; i2 < 4; ++i2)
            if (!kept_by(ly, p.flags, pass, ee + i2)) c[i2] = 0.0;
        } else {
          const float4 o = make_float4((float)c[0], (float)c[1], (float)c[2], (float)c[3]);
          st4(zn + e, o);
          if (znp) st4(znp + e, o);  // split K1: the peer's z_node too (NVLink store)
        }
        a0 = __dadd_rn(a0, __dmul_rn(c[0], c[0]));
        a1 = __dadd_rn(a1, __dmul_rn(c[1], c[1]));
        a2 = __dadd_rn(a2, __dmul_rn(c[2], c[2]));
        a3 = __dadd_rn(a3, __dmul_rn(c[3], c[3]));
      });
  if (xnext) {
    __shared__ int s_claim;
    __syncthreads();
    if (threadIdx.x == 0) s_claim = claim();
    __syncthreads();
    const int nx = s_claim;
    *xnext = nx;
    *pre = nx < p.n_items && xtile_ok(p, p.items[nx]);
    if (*pre) tile_quads_prologue<MODE>(p, p.items[nx], ring);  // in flight under the fold
  }
  double* mine = cs + ph * (4 * W) + 4 * jj;
  __syncthreads();  // (without xnext) cs aliases the ring: every thread is done with its last stage
  mine[0] = a0; mine[1] = a1; mine[2] = a2; mine[3] = a3;
  __syncthreads();
  const int col0 = it.chunk * 4 * cq;
  const int ncol = min(4 * cq, L - col0);
  const bool percol = ly.group[pass] == kShape || ly.k == 1 || ly.percol;
  const int G = ly.G[pass];
  double* out = p.partials + ly.poff[pass] + (long long)it.part * (percol ? L : G);
  double* outp = p.partials_peer ? p.partials_peer + (out - p.partials) : nullptr;
  const int t = threadIdx.x;
  double s = 0.0;
  if (t < ncol) {  // one column per thread: the row phases in order
    s = cs[t];
    for (int q = 1; q < RP; ++q) s += cs[q * 4 * W + t];
  }
  if (percol) {
    if (t < ncol) {
      out[col0 + t] = s;
      if (outp) outp[col0 + t] = s;
    }
    return;
  }
  __syncthreads();
  if (t < ncol) cs[t] = s;
  __syncthreads();
  const int k = ly.k;
  const int c0 = col0 / k;  // whole channels per tile
  if (t < ncol / k) {
    double g = 0.0;
    for (int jx = 0; jx < k; ++jx) g += cs[t * k + jx];
    out[c0 + t] = g;
    if (outp) outp[c0 + t] = g;
  }
}

// K1b row tiles (FILTER groups, composite plans mixing FILTER, rows not a
// multiple of 4 elements — e.g. the 7x7 stem): one shared-memory sub-tile of
// rows per item; squares staged in shared memory, then reduced by one thread
// per column (CHANNEL / SHAPE: per-column partials [part][L], folded into
// channels by K2) or one warp per row (FILTER: per-row sums).
template <int MODE>
__device__ void cand_tile_rows(const CandArgs& p, const DevLayer& ly, const Item& it, double* sq) {
  const int pass = p.pass;
  const int grp = ly.group[pass];
  const int L = ly.L;
  const Coef cf = coef_of(ly);
  const long long r0 = it.begin / L;
  const int nr = (int)((it.end - it.begin) / L);
  const int E = nr * L;
  const long long ebase = r0 * (long long)L;
  const long long gbase = ly.off + ebase;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int i = threadIdx.x; i < E; i += kThreads) {
    double c = cand_elem<MODE>(p, gbase + i, cf);
    if (pass > 0 && !kept_by(ly, p.flags, pass, ebase + i)) c = 0.0;
    if (pass == 0) {
      p.zn[gbase + i] = (float)c;
      if (p.zn_peer) p.zn_peer[gbase + i] = (float)c;
    }
    sq[i] = __dmul_rn(c, c);
  }
  __syncthreads();
  if (grp == kFilter) {
    for (int r = warp; r < nr; r += kThreads / 32) {
      double s = 0.0;
      for (int i = lane; i < L; i += 32) s += sq[r * L + i];
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) s += __shfl_xor_sync(kFull, s, off);
      if (lane == 0) {
        p.partials[ly.poff[pass] + r0 + r] = s;
        if (p.partials_peer) p.partials_peer[ly.poff[pass] + r0 + r] = s;
      }
    }
  } else if (grp == kShape || ly.k == 1 || ly.percol) {
    for (int col = threadIdx.x; col < L; col += kThreads) {
      double s = 0.0;
      for (int r = 0; r < nr; ++r) s += sq[r * L + col];
      p.partials[ly.poff[pass] + (long long)it.part * L + col] = s;
      if (p.partials_peer) p.partials_peer[ly.poff[pass] + (long long)it.part * L + col] = s;
    }
  } else {
    const int k = ly.k, G = ly.G[pass];
    for (int c = threadIdx.x; c < G; c += kThreads) {  // channel: rows, then its kh*kw columns
      double s = 0.0;
      for (int r = 0; r < nr; ++r)
        for (int jx = 0; jx < k; ++jx) s += sq[r * L + c * k + jx];
      p.partials[ly.poff[pass] + (long long)it.part * G + c] = s;
      if (p.partials_peer) p.partials_peer[ly.poff[pass] + (long long)it.part * G + c] = s;
    }
  }
}

#ifdef HSX_TRACE
// timeline instrumentation (trace builds only: make trace): per item slot
// [start ns, tile done ns, tail done ns, smid | layer << 16]
__device__ unsigned long long g_trace[16384 * 4];
__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned smid() {
  unsigned r;
  asm volatile("mov.u32 %0, %smid;" : "=r"(r));
  return r;
}
#define TRACE_AT(slot, j, val) \
  do {                         \
    if (threadIdx.x == 0 && (slot) < 16384) g_trace[(slot) * 4 + (j)] = (val); \
  } while (0)
#else
#define TRACE_AT(slot, j, val) \
  do {                         \
  } while (0)
#endif

template <int MODE, class Claim>
__device__ __forceinline__ void cand_item(const CandArgs& p, int frozen, const Item& it, float4* ring,
                                          double* xcs, bool* pre, int* xnext, Claim claim) {
  const DevLayer& ly = p.layers[it.layer];
  if (frozen || ly.ncons == 0) {
    if (p.pass > 0) return;
    if (it.begin & 3) {  // ranges of layers with c_in*kh*kw % 4 != 0: scalar path
      const bool masked = frozen && ly.ncons > 0 && p.fmask != nullptr;
      const Coef cf = coef_of(ly);
      for (long long e = it.begin + threadIdx.x; e < it.end; e += kThreads) {
        double c = cand_elem<MODE>(p, ly.off + e, cf);
        if (masked && !((p.fmask[ly.mword + (e >> 5)] >> (e & 31)) & 1u)) c = c * 0.0;
        p.zn[ly.off + e] = (float)c;
      }
      return;
    }
    cand_elementwise<MODE>(p, ly, it.begin, it.end, frozen, ring);
    return;
  }
  if (ly.ncons <= p.pass) return;
  if (ly.tiling == 1)
    cand_tile_quads<MODE>(p, ly, it, ring, xnext ? xcs : reinterpret_cast<double*>(ring), pre, xnext, claim);
  else
    cand_tile_rows<MODE>(p, ly, it, reinterpret_cast<double*>(ring));
#ifdef HSX_TRACE
  TRACE_AT((&it - p.items), 1, gtime());
#endif
  if (!((ly.fsel >> p.pass) & 1)) {
    if (p.k1done) {  // chained K2: this tile's partials are released to the layer's selection
      __syncthreads();
      if (threadIdx.x == 0) {
        if (p.k1done_peer) {
          // split K1: the tile's z_node and partials went to both ranks; both
          // selections count it (system scope: the peer's K2 reads over its acquire)
          __threadfence_system();
          atomicAdd_system(p.k1done_peer + ly.pidx, 1u);
        } else {
          __threadfence();
        }
        atomicAdd(p.k1done + ly.pidx, 1u);
      }
    }
    return;
  }
  // fused K2: the layer's last tile to finish selects its groups (its partials
  // are complete once every tile has released them: fence, then the counter)
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(p.cand_done + ly.pidx, 1u) == (unsigned)ly.ncitems - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  select_layer(ly, p.pass, p.partials, p.norms, p.fw, ring, it.layer, p.structured ? &p.ka : nullptr);
  if (threadIdx.x == 0) p.cand_done[ly.pidx] = 0;  // ready for the next launch
}

// Persistent CTAs (grid = resident CTAs, or one per item if fewer): CTA b starts
// on item b and then pulls the next unclaimed item from a global counter, so the
// unequal tiles (ragged column chunks, short dense items, selection tails) balance
// dynamically instead of leaving a partial second wave. Results do not depend on
// which CTA runs an item (partials are indexed by item), so they stay
// deterministic. The last CTA to leave re-zeroes the counters.
template <int MODE>
__global__ void __launch_bounds__(kThreads, 3) k_candidate(CandArgs p, int frozen) {
  PDL_ENTRY();
  extern __shared__ float4 ring[];
  __shared__ int next;
  int idx = blockIdx.x;
  unsigned epoch = 0;
  // cross-tile pipelining (dynamic launches, persistent grid, no staging)
  const bool single = gridDim.x >= (unsigned)p.n_items;
  const bool xt = p.xtile && !frozen && !p.sready && !single;
  // fold scratch in cross-tile mode: the ring's last stage (D-1), which the next tile's
  // prologue (stages 0 .. D-2) leaves free until the fold is done (8 KB <= one stage)
  double* xcs = reinterpret_cast<double*>(ring + (K1<MODE>::D - 1) * K1<MODE>::NB * kThreads);
  bool pre = false;
  unsigned int* const sched = p.sched;  // (captured by value: a reference to the kernel
                                         // parameter would force a local copy of it)
  auto claim = [sched]() -> int { return (int)gridDim.x + (int)atomicAdd(sched, 1u); };
  if (threadIdx.x == 0) {
    s_k1_alt = 0;
    if (p.sready) epoch = *reinterpret_cast<volatile unsigned*>(p.sepoch);  // bumped only by the last CTA
  }
  __syncthreads();
  while (idx < p.n_items) {
#ifdef HSX_TRACE
    TRACE_AT(idx, 0, gtime());
    TRACE_AT(idx, 3, smid() | ((unsigned long long)p.items[idx].layer << 16));
#endif
    if (p.sready) {
      // staged peer operand: wait for this item's staging copy (the staging kernel runs
      // ahead on a side stream); if it has not landed within the timeout, read the
      // peer's send directly for this item (never a deadlock, same values either way)
      if (threadIdx.x == 0) {
        const unsigned long long t0 = global_ns();
        unsigned v;
        int alt = 0;
        for (;;) {
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p.sready + idx) : "memory");
          if (v == epoch + 1u) break;
          if (global_ns() - t0 > 200000ull) {
            alt = 1;
            break;
          }
          __nanosleep(64);
        }
        s_k1_alt = alt;
      }
      __syncthreads();
    }
    // cross-tile (xt): a quad tile claims the next item itself and may have issued
    // its first stages already (pre); other items claim below
    int nx = -1;
    cand_item<MODE>(p, frozen, p.items[idx], ring, xcs, &pre, xt ? &nx : nullptr, claim);
    if (xt) {
      if (nx < 0) {
        pre = false;
        __syncthreads();
        if (threadIdx.x == 0) next = claim();
        __syncthreads();
        nx = next;
      }
#ifdef HSX_TRACE
      TRACE_AT(idx, 2, gtime());
#endif
      __syncthreads();  // fold scratch / row flags reused by the next item
      idx = nx;
      continue;
    }
#ifdef HSX_TRACE
    TRACE_AT(idx, 2, gtime());
#endif
    if (gridDim.x >= (unsigned)p.n_items) break;
    __syncthreads();  // ring / fold scratch reused by the next item
    if (threadIdx.x == 0) next = (int)gridDim.x + (int)atomicAdd(p.sched, 1u);
    __syncthreads();
    idx = next;
  }
  if (gridDim.x < (unsigned)p.n_items && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(p.sched + 1, 1u) == gridDim.x - 1) {
      p.sched[0] = 0;
      p.sched[1] = 0;
    }
  }
  if (p.sready && threadIdx.x == 0) {  // the last CTA out moves the staging epoch on
    __threadfence();
    if (atomicAdd(p.sepoch + 1, 1u) == gridDim.x - 1) {
      p.sepoch[1] = 0;
      p.sepoch[0] = epoch + 1u;
    }
  }
}

// Staging copy of the peer's send for a staged K1: persistent CTAs take K1's dynamic
// items in order (the order K1 takes them), copy each item's region of the peer's
// buffer into the local stage buffer with float4 loads, and publish sready[item] =
// epoch + 1 (release). Quad tiles: rows [begin, end) x quads [chunk cq, +cq) of the
// layer; element items: [begin, end) of the layer.
__global__ void __launch_bounds__(kThreads) k_stage(const float* __restrict__ peer, float* __restrict__ stage,
                                                    const DevLayer* __restrict__ layers,
                                                    const Item* __restrict__ items, int n_items,
                                                    unsigned int* sready, const unsigned int* sepoch,
                                                    unsigned int* counter) {
  __shared__ int next;
  __shared__ unsigned epoch;
  if (threadIdx.x == 0) epoch = *reinterpret_cast<const volatile unsigned*>(sepoch);
  int idx = blockIdx.x;
  __syncthreads();
  while (idx < n_items) {
    const Item it = items[idx];
    const DevLayer& ly = layers[it.layer];
    const long long off = ly.off;
    if (it.tile == 1) {
      // eight float4 loads in flight per thread (NVLink latency): ~32 KB per CTA
      const int Q = ly.L >> 2;
      const int q0 = it.chunk * ly.cq;
      const int nq = min(ly.cq, Q - q0);
      const long long nrow = it.end - it.begin;
      const long long total = nrow * nq;
      constexpr int U = 8;
      for (long long i0 = threadIdx.x; i0 < total; i0 += (long long)U * kThreads) {
        float4 x[U];
        long long ea[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const long long i = i0 + (long long)u * kThreads;
          ea[u] = -1;
          if (i < total) {
            const long long r = it.begin + i / nq;
            ea[u] = off + r * ly.L + 4LL * (q0 + (int)(i % nq));
            x[u] = __ldcg(reinterpret_cast<const float4*>(peer + ea[u]));
          }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (ea[u] >= 0) *reinterpret_cast<float4*>(stage + ea[u]) = x[u];
      }
    } else {
      const long long b = off + it.begin, e = off + it.end;
      const long long b4 = (b + 3) & ~3LL, e4 = e & ~3LL;
      if (b4 < e4) {
        for (long long i = b4 + 4LL * threadIdx.x; i < e4; i += 4LL * kThreads)
          *reinterpret_cast<float4*>(stage + i) = __ldcg(reinterpret_cast<const float4*>(peer + i));
        for (long long i = b + threadIdx.x; i < b4; i += kThreads) stage[i] = peer[i];
        for (long long i = e4 + threadIdx.x; i < e; i += kThreads) stage[i] = peer[i];
      } else {
        for (long long i = b + threadIdx.x; i < e; i += kThreads) stage[i] = peer[i];
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sready + idx), "r"(epoch + 1u) : "memory");
      next = (int)gridDim.x + (int)atomicAdd(counter, 1u);
    }
    __syncthreads();
    idx = next;
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(counter + 1, 1u) == gridDim.x - 1) {
      counter[0] = 0;
      counter[1] = 0;
    }
  }
}

void launch_stage(const float* peer, float* stage, const DevLayer* layers, const Item* items, int n_items,
                  unsigned int* sready, const unsigned int* sepoch, unsigned int* counter, int grid, cudaStream_t st) {
  if (n_items <= 0) return;
  k_stage<<<std::min(grid, n_items), kThreads, 0, st>>>(peer, stage, layers, items, n_items, sready, sepoch, counter);
}

template <int MODE>
static void launch_candidate_mode(const CandArgs& a, int n_items, int frozen, size_t smem, cudaStream_t st) {
  allow_smem(k_candidate<MODE>, smem);
  // resident CTAs per device (per instantiation and shared-memory size)
  static int resident_of[kMaxDevices];
  static size_t resident_smem[kMaxDevices];
  const int dev = current_device();
  if (resident_of[dev] <= 0 || resident_smem[dev] != smem) {
    int per_sm = 0, sms = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_candidate<MODE>, kThreads, smem);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    resident_of[dev] = std::max(1, per_sm) * std::max(1, sms);
    resident_smem[dev] = smem;
  }
  const int resident = resident_of[dev];
  static const bool persistent = [] {
    const char* v = std::getenv("HSX_K1_PERSISTENT");
    return !(v && v[0] == '0');
  }();
  CandArgs b = a;
  b.n_items = n_items;
  const int slots = std::max(1, resident - std::max(0, a.reserve));
  const int grid = (persistent && a.sched) ? std::min(n_items, slots) : n_items;
  launch_pdl(k_candidate<MODE>, grid, kThreads, smem, st, b, frozen);
}

void launch_candidate(const CandArgs& a, int n_items, int frozen, size_t smem, cudaStream_t st) {
  if (n_items <= 0) return;
  // two ranks: their sum is theta + u's fp64 fold with the two sends as the operands
  // (rank order), so the theta + u kernel runs it — a 4-slot ring, three CTAs per SM
  // and no per-peer loop (B200: 18% faster than the peer kernel on local data);
  // HSX_K1_PEERS2=2 (opt-in: reading over NVLink it measured 3% slower than the
  // general peer kernel, r2y), =1: the 2-slot peer kernel, default 0: the general one
  static const int peers2 = [] {
    const char* v = std::getenv("HSX_K1_PEERS2");
    return v ? std::atoi(v) : 0;  // over NVLink the theta + u kernel measured 3% slower (r2y): opt-in (=2)
  }();
  if (a.sdist) {
    launch_candidate_mode<kModeSumDist>(a, n_items, frozen, smem, st);
  } else if (a.peers.n == 2 && peers2 == 2) {
    CandArgs b = a;
    b.theta = a.peers.p[0];
    b.u = a.peers.p[1];
    b.s = nullptr;
    b.peers.n = 0;
    launch_candidate_mode<kModeThetaU>(b, n_items, frozen, smem, st);
  } else if (a.peers.n == 2 && peers2 == 1)
    launch_candidate_mode<kModePeers2>(a, n_items, frozen,
                                       std::max(smem, (size_t)K1<kModePeers2>::D * K1<kModePeers2>::NB * kThreads * 16),
                                       st);
  else if (a.peers.n > 0)
    launch_candidate_mode<kModePeers>(a, n_items, frozen, smem + (size_t)kDepth * (kMaxPeers - 2) * kThreads * 16, st);
  else if (a.identity)
    launch_candidate_mode<kModeIdent>(a, n_items, frozen, smem, st);
  else if (a.s)
    launch_candidate_mode<kModeSum>(a, n_items, frozen, smem, st);
  else
    launch_candidate_mode<kModeThetaU>(a, n_items, frozen, smem, st);
}

__global__ void k_div_selftest(const double* __restrict__ num, long long n, double den, double y,
                               double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = div_rn(num[i], den, y);
}

void launch_div_selftest(const double* num, long long n, double den, double* out, cudaStream_t st) {
  if (n <= 0) return;
  int grid = (int)std::min<long long>((n + 255) / 256, 148LL * 8);
  k_div_selftest<<<grid, 256, 0, st>>>(num, n, den, 1.0 / den, out);
}

void launch_select(const DevLayer* layers, const int* list, int n, int pass, const double* partials,
                   double* norms, FlagPtrs flags, const KeepArgs& ka, int structured, size_t smem, cudaStream_t st,
                   unsigned int* k1done, unsigned int* ready) {
  if (n <= 0) return;
  allow_smem(k_select, smem);
  static const int nt = [] {
    const char* v = std::getenv("HSX_SELECT_THREADS");
    // 512 (B200 sweep, profiles/r1i_sweep_select_threads.txt): cheaper barriers than
    // 1024 for G <= 2048 groups, enough loads in flight for the partial fold
    const int x = v ? std::atoi(v) : 512;
    return (x >= 64 && x <= 1024 && x % 32 == 0) ? x : 512;
  }();
  launch_pdl(k_select, n, nt, smem, st, layers, list, pass, partials, norms, flags, ka, structured, k1done, ready);
}

size_t structured_smem_bytes(int rows, int L, int cin) { return structured_bytes(rows, L, cin); }
size_t select_smem_bytes(int G) { return select_bytes(G) + (size_t)kFoldCols * sizeof(double); }

// ---------------------------------------------------------------------------
// K3 project + local mask.  sparsity.py:71-94, 113-115; consensus.py:181-182
// A thread owns a quad of elements (one row when L % 4 == 0): one float4 load,
// a loop-invariant kept nibble for its four columns; 8 lanes' nibbles OR-fold
// into one mask word.
// ---------------------------------------------------------------------------

// Layer fields the streaming kernels use, loaded once into registers (stores
// through the float arenas would otherwise force reloads of the layer table).
struct LayerRegs {
  long long off, n, mword, okeep, ikeep;
  int L, k, ncons, qtile;
  FastDiv divL, divk;
  __device__ __forceinline__ LayerRegs(const DevLayer* __restrict__ layers, int l) {
    const DevLayer& ly = layers[l];
    off = ly.off; n = ly.n; mword = ly.mword; okeep = ly.okeep; ikeep = ly.ikeep;
    L = ly.L; k = ly.k; ncons = ly.ncons; qtile = ly.qtile; divL = ly.divL; divk = ly.divk;
  }
};

// Row-quad tiles (prunable layers with c_in*kh*kw % 32 == 0): an item is rows
// [begin, end) x quad chunk `chunk` (64 quads); thread t owns quad
// chunk*64 + (t & 63) and walks rows begin + (t >> 6) + 4i. Column maps are
// loop-invariant registers; row maps of the tile sit in shared memory.
constexpr int kRowPhases = kThreads / kTileQuads;  // 4
constexpr int kMaxTileRows = 128;

struct TileCtx {
  int j, jj, ph;
  long long r0, r1;
  int count;
  bool valid;
  __device__ __forceinline__ TileCtx(const Item& it, int L) {
    jj = threadIdx.x & (kTileQuads - 1);
    ph = threadIdx.x / kTileQuads;
    j = it.chunk * kTileQuads + jj;
    r0 = it.begin + ph;
    r1 = it.end;
    valid = 4 * j < L;
    count = (valid && r0 < r1) ? (int)((r1 - r0 + kRowPhases - 1) / kRowPhases) : 0;
  }
  __device__ __forceinline__ long long row(int i) const { return r0 + (long long)i * kRowPhases; }
};

// CHECK (structured keep sets, one node): flag the layer when a kept element is
// exactly zero — its mask is then not the rectangle R x C the selection derived
// the keep sets from, and k_keep_fixup re-derives it from the bits
__device__ __forceinline__ void flag_irregular(const KeepArgs& a, int pidx, bool bad) {
  if (__any_sync(kFull, bad) && (threadIdx.x & 31) == 0) {
    atomicOr(a.irr + pidx, 1);
    atomicOr(a.irr_any, 1);
  }
}

// TMA (unchained launches): the tile's rows of z_node arrive by 1-D bulk copies
// (cp.async.bulk, one per kept row segment of up to 1 KB, issued by one thread) into
// a two-stage ring of 16-row stages completed on mbarriers, instead of one 16-B
// cp.async per quad and thread.
constexpr int kProjStageRows = 16;
constexpr size_t kProjTmaSmem = 2 * kProjStageRows * kTileQuads * 16;  // 32 KB

template <bool CHECK, bool TMA = false>
__device__ __forceinline__ void project_item(const KeepArgs& a, float* __restrict__ zn,
                                             uint32_t* __restrict__ mask, const Item& it, float4* ring) {
  __shared__ uint8_t s_rk[kMaxTileRows];
  const LayerRegs ly(a.layers, it.layer);
  const DevLayer& dl = a.layers[it.layer];
  const int lane = threadIdx.x & 31;
  if (it.tile == 1) {
    // row-quad tile: 8 lanes (same row, 8 consecutive quads) make one mask word
    const TileCtx tc(it, ly.L);
    const int nrow = (int)(it.end - it.begin);
    // all lanes of a warp share a row phase and walk the same rows; quads past the
    // row end are a suffix of the last chunk in whole 8-lane groups (L % 32 == 0):
    // they run the loop with nothing kept (no read, no store) so the mask-word
    // shuffles are full-warp, and a warp with no valid quad skips the loop
    const bool warp_valid = 4 * (it.chunk * kTileQuads + ((threadIdx.x & ~31) & (kTileQuads - 1))) < ly.L;
    const int count = (warp_valid && tc.r0 < tc.r1) ? (int)((tc.r1 - tc.r0 + kRowPhases - 1) / kRowPhases) : 0;
    const bool valid = tc.valid;
    const bool word_lane = (lane & 7) == 0 && valid;
    // (no L2 policy here: with the mask-word shuffles in the loop ptxas reuses the
    // policy's uniform descriptor register for BRA.DIV -> illegal instruction)
    // quad i of this thread sits at e0 + i * estep, its mask word at m0 + i * mstep
    // (L % 32 == 0), its row flag at s_rk[ph + 4 i]: walked by running pointers
    const long long e0 = tc.r0 * ly.L + 4 * (valid ? tc.j : 0), estep = (long long)kRowPhases * ly.L;
    const int mstep = kRowPhases * (ly.L >> 5);
    const float* ls = zn + ly.off + e0;    // next quad to load
    const unsigned ring0 = smem_u32(ring_slot<1>(ring, 0, 0));
    if (!TMA) {
      // the first kDepth-1 quads go in flight before the keep flags are gathered (a
      // chain of dependent flag loads): read whatever is kept
#pragma unroll
      for (int d = 0; d < kDepth - 1; ++d) {
        if (d < count)
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ring0 + d * kThreads * 16), "l"(ls)
                       : "memory");
        cp_commit();
        ls += estep;
      }
    }
    // kept = AND over the passes' group flags: rows (FILTER) in shared memory,
    // this thread's four columns (CHANNEL / SHAPE) in a nibble
    for (int r = threadIdx.x; r < nrow; r += kThreads) {
      uint8_t kp = 1;
      for (int q = 0; q < ly.ncons; ++q)
        if (dl.group[q] == kFilter) kp &= a.flags.f[q][dl.goff[q] + it.begin + r];
      s_rk[r] = kp;
    }
    const FastDiv divk = dl.divk;
    unsigned ckb = 0;
    if (valid) {
      ckb = 0xFu;
      for (int q = 0; q < ly.ncons; ++q) {
        const int grp = dl.group[q];
        if (grp == kFilter) continue;
        const uint8_t* f = a.flags.f[q] + dl.goff[q];
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const unsigned col = 4 * tc.j + b;
          if (!f[grp == kChannel ? fdiv(col, divk) : col]) ckb &= ~(1u << b);
        }
      }
    }
    if (TMA) {
      __shared__ __align__(8) uint64_t s_full[2];
      if (threadIdx.x == 0) {
        mbar_init(&s_full[0], 1);
        mbar_init(&s_full[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
      }
      // no kept column in this chunk: nothing is read (every quad is zeroed)
      const bool anycol = __syncthreads_or(ckb != 0);
      const int q0 = it.chunk * kTileQuads;
      const unsigned seg = (unsigned)min(kTileQuads, (ly.L >> 2) - q0) * 16u;
      unsigned char* buf = reinterpret_cast<unsigned char*>(ring);
      const float* rows = zn + ly.off + it.begin * ly.L + 4 * q0;
      const int nst = (nrow + kProjStageRows - 1) / kProjStageRows;
      auto issue_stage = [&](int g) {  // thread 0: the kept rows of stage g
        const int b = g & 1, r0 = g * kProjStageRows, r1 = min(r0 + kProjStageRows, nrow);
        unsigned bytes = 0;
        for (int r = r0; r < r1; ++r) bytes += s_rk[r] ? seg : 0u;
        mbar_arrive_tx(&s_full[b], bytes);
        for (int r = r0; r < r1; ++r)
          if (s_rk[r])
            bulk_g2s(buf + ((size_t)b * kProjStageRows + (r - r0)) * (kTileQuads * 16), rows + (long long)r * ly.L,
                     seg, &s_full[b]);
      };
      if (threadIdx.x == 0 && anycol) {
        issue_stage(0);
        if (nst > 1) issue_stage(1);
      }
      unsigned bad = 0;
      float* qc = zn + ly.off + e0;
      uint32_t* mc = mask + ly.mword + (e0 >> 5);
      const int sh = 4 * (lane & 7);
      for (int g = 0; g < nst; ++g) {
        if (anycol) mbar_wait(&s_full[g & 1], (unsigned)(g >> 1) & 1u);
        const unsigned char* sb = buf + (size_t)(g & 1) * kProjStageRows * (kTileQuads * 16) + tc.jj * 16;
#pragma unroll
        for (int k = 0; k < kProjStageRows / kRowPhases; ++k) {
          if (4 * g + k >= count) break;  // warp-uniform
          const int rr = tc.ph + kRowPhases * k;
          float4 v = *reinterpret_cast<const float4*>(sb + rr * (kTileQuads * 16));
          const unsigned kn = s_rk[g * kProjStageRows + rr] ? ckb : 0u;
          const unsigned nib = kn & ((unsigned)(v.x != 0.f) | ((unsigned)(v.y != 0.f) << 1) |
                                     ((unsigned)(v.z != 0.f) << 2) | ((unsigned)(v.w != 0.f) << 3));
          if (CHECK) bad |= kn & ~nib;
          if (kn != 0xFu && valid) {
            if (!(kn & 1u)) v.x = 0.f;
            if (!(kn & 2u)) v.y = 0.f;
            if (!(kn & 4u)) v.z = 0.f;
            if (!(kn & 8u)) v.w = 0.f;
            st4(qc, v);
          }
          unsigned w = nib << sh;
          w |= __shfl_xor_sync(kFull, w, 1);
          w |= __shfl_xor_sync(kFull, w, 2);
          w |= __shfl_xor_sync(kFull, w, 4);
          if (word_lane) *mc = w;
          qc += estep;
          mc += mstep;
        }
        if (g + 2 < nst) {
          __syncthreads();  // every thread is done with this stage's buffer
          if (threadIdx.x == 0 && anycol) {
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            issue_stage(g + 2);
          }
        }
      }
      if (CHECK) flag_irregular(a, dl.pidx, bad != 0);
      return;
    }
    __syncthreads();
    // from stage kDepth-1 on a quad with nothing kept is not read (the copy zero-fills
    // it without touching memory): only the kept quads' z_node is needed for the
    // nonzero test
    const uint8_t* lrk = s_rk + tc.ph + kRowPhases * (kDepth - 1);  // row flag of the next quad to load
    auto issue = [&](int d, int) {
      const bool any = ckb && *lrk;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(ring0 + d * kThreads * 16), "l"(ls),
                   "r"(any ? 16 : 0)
                   : "memory");
      ls += estep;
      lrk += kRowPhases;
    };
    unsigned bad = 0;  // CHECK: kept but zero
    float* qc = zn + ly.off + e0;          // quad being consumed
    uint32_t* mc = mask + ly.mword + (e0 >> 5);
    const uint8_t* crk = s_rk + tc.ph;
    const int sh = 4 * (lane & 7);
    auto consume = [&](int d, int) {
      float4 v = *ring_slot<1>(ring, d, 0);
      const unsigned kn = *crk ? ckb : 0u;  // kept nibble (0 past the row end)
      const unsigned nib = kn & ((unsigned)(v.x != 0.f) | ((unsigned)(v.y != 0.f) << 1) |
                                 ((unsigned)(v.z != 0.f) << 2) | ((unsigned)(v.w != 0.f) << 3));
      if (CHECK) bad |= kn & ~nib;
      if (kn != 0xFu && valid) {
        if (!(kn & 1u)) v.x = 0.f;
        if (!(kn & 2u)) v.y = 0.f;
        if (!(kn & 4u)) v.z = 0.f;
        if (!(kn & 8u)) v.w = 0.f;
        st4(qc, v);
      }
      unsigned w = nib << sh;
      w |= __shfl_xor_sync(kFull, w, 1);
      w |= __shfl_xor_sync(kFull, w, 2);
      w |= __shfl_xor_sync(kFull, w, 4);
      if (word_lane) *mc = w;
      qc += estep;
      mc += mstep;
      crk += kRowPhases;
    };
    ring_loop(count, issue, consume);
    if (CHECK) flag_irregular(a, dl.pidx, bad != 0);
    return;
  }
  // contiguous ranges of other prunable layers: one warp per 32-element word; the
  // passes' group kinds and flag bases in registers
  int gq[kMaxPasses];
  const uint8_t* fq[kMaxPasses];
#pragma unroll
  for (int q = 0; q < kMaxPasses; ++q) {
    gq[q] = q < ly.ncons ? dl.group[q] : -1;
    fq[q] = q < ly.ncons ? a.flags.f[q] + dl.goff[q] : nullptr;
  }
  const FastDiv divk = dl.divk;
  const int warp = threadIdx.x >> 5;
  const long long w0 = it.begin >> 5, w1 = (it.end + 31) >> 5;
  bool bad = false;
  for (long long w = w0 + warp; w < w1; w += kThreads / 32) {
    long long e = (w << 5) + lane;
    bool kp = false;
    float x = 0.f;
    if (e < ly.n) {
      const unsigned o = fdiv((unsigned)e, ly.divL);
      const unsigned col = (unsigned)e - o * (unsigned)ly.L;
      const unsigned c = fdiv(col, divk);
      kp = true;
#pragma unroll
      for (int q = 0; q < kMaxPasses; ++q)
        if (gq[q] >= 0) kp = kp && fq[q][group_of(gq[q], o, col, c)];
      x = zn[ly.off + e];
      if (!kp) zn[ly.off + e] = 0.f;
    }
    const bool bit = kp && x != 0.0f;
    if (CHECK) bad |= kp && !bit;
    const unsigned bits = __ballot_sync(kFull, bit);
    if (lane == 0) mask[ly.mword + w] = bits;
  }
  if (CHECK) flag_irregular(a, dl.pidx, bad);
}

__device__ void fixup_layer(const KeepArgs& a, int l, uint8_t* fsm);

// Chained (ready != nullptr, behind a chained K2): like the chained K2, the CTA lets
// its dependents launch at once, waits for its layer's selection (ready[layer],
// published by K2 with release semantics), projects, and waits for the grid before
// it at the end; the layer's last item re-zeroes its counter and flag.
template <bool CHECK, bool TMA>
__global__ void __launch_bounds__(kThreads, 5) k_project(KeepArgs a, float* __restrict__ zn,
                                                         uint32_t* __restrict__ mask, unsigned int* ready,
                                                         unsigned int* pdone, ChainK67 c67) {
  extern __shared__ float4 ring[];
  const Item it = a.items[blockIdx.x];  // a register copy: a reference into global memory is
  if (ready == nullptr) {               // reloaded after every store through zn / mask
    PDL_ENTRY();
    project_item<CHECK, TMA>(a, zn, mask, it, ring);
    return;
  }
  pdl_trigger();
  if (threadIdx.x == 0) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ready + it.layer) : "memory");
      if (v) break;
      __nanosleep(128);
    }
  }
  __syncthreads();
  project_item<CHECK>(a, zn, mask, it, ring);
  __shared__ bool last_item, last_layer;
  __syncthreads();
  const DevLayer& dl = a.layers[it.layer];
  if (threadIdx.x == 0) {
    __threadfence();
    last_item = atomicAdd(pdone + dl.pidx, 1u) == (unsigned)dl.npitems - 1;
  }
  __syncthreads();
  if (last_item) {
    __threadfence();
    if (threadIdx.x == 0) {
      pdone[dl.pidx] = 0;
      ready[it.layer] = 0;
    }
    if (c67.ready3) {
      // the layer's keep-set fixup here (not a launch of its own), then the chained
      // K67 may take the layer; the last layer lays the flat buffer out again if a
      // layer turned out irregular
      fixup_layer(a, it.layer, reinterpret_cast<uint8_t*>(ring));
      __syncthreads();
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(c67.ready3 + it.layer), "r"(1u) : "memory");
        last_layer = atomicAdd(pdone + a.n_prunable, 1u) == (unsigned)a.n_prunable - 1;
      }
      __syncthreads();
      if (last_layer) {
        __threadfence();
        if (*reinterpret_cast<volatile int*>(a.irr_any)) layout_flat(a);
        __syncthreads();
        if (threadIdx.x == 0) {
          pdone[a.n_prunable] = 0;
          *a.irr_any = 0;
        }
        if (c67.pub_sum) {
          // the summary is final: publish it to the host now (the K67 behind this
          // launch keeps the stream busy, so no copy op can sit between them)
          __threadfence();
          for (int i = threadIdx.x; i < c67.n_sum; i += blockDim.x)
            c67.pub_sum[i] = __ldcg(reinterpret_cast<const long long*>(a.summary) + i);
          __threadfence_system();
          __syncthreads();
          if (threadIdx.x == 0) {
            const unsigned v = atomicAdd(c67.seq_ctr, 1u) + 1u;
            asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(c67.pub_seq), "r"(v) : "memory");
          }
        }
      }
    }
  }
  pdl_wait();
  // everything before this launch is complete: the chained K67's dense-layer items
  // (which read K1's output directly) may start
  if (c67.upstream && threadIdx.x == 0) {
    __threadfence();
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(c67.upstream), "r"(1u) : "memory");
  }
}

__device__ void fixup_layer(const KeepArgs& a, int l, uint8_t* fsm);

// K2 + K3 in one launch (single-constraint plans): CTAs [0, nsel) select one layer
// each and publish ready[layer]; the K3 CTAs behind them wait for their layer's
// flag (acquire), so the projection of the layers selected first overlaps the
// selection of the big ones instead of waiting for the slowest. Selection CTAs
// have the lowest indices and never wait (dispatched first: no deadlock). The
// last K3 item of a layer re-zeroes its flag and counter for the next launch.
__global__ void __launch_bounds__(kThreads) k_select_project(SelProjArgs sp, KeepArgs a, float* __restrict__ zn,
                                                            uint32_t* __restrict__ mask) {
  PDL_ENTRY();
  extern __shared__ float4 ring[];
  if ((int)blockIdx.x < sp.nsel) {
    const int l = sp.list[blockIdx.x];
    select_layer(a.layers[l], 0, sp.partials, sp.norms, a.flags, ring, l, sp.structured ? &a : nullptr);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(sp.ready + l), "r"(1u) : "memory");
    }
    return;
  }
  const Item it = a.items[blockIdx.x - sp.nsel];
  const int l = it.layer;
  if (threadIdx.x == 0) {
    unsigned v;
    for (;;) {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(sp.ready + l) : "memory");
      if (v) break;
      __nanosleep(256);
    }
  }
  __syncthreads();
  project_item<true>(a, zn, mask, it, ring);
  // the layer's last K3 item runs the layer's fixup (k_keep_fixup fused); the last
  // layer to finish re-lays the flat buffer out if any layer had a kept zero
  __shared__ bool last_item, last_layer;
  __syncthreads();
  const DevLayer& dl = a.layers[l];
  if (threadIdx.x == 0) {
    __threadfence();
    last_item = atomicAdd(sp.pdone + dl.pidx, 1u) == (unsigned)dl.npitems - 1;
  }
  __syncthreads();
  if (!last_item) return;
  __threadfence();
  if (threadIdx.x == 0) {
    sp.pdone[dl.pidx] = 0;
    sp.ready[l] = 0;
  }
  fixup_layer(a, l, reinterpret_cast<uint8_t*>(ring));
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last_layer = atomicAdd(sp.pdone + a.n_prunable, 1u) == (unsigned)a.n_prunable - 1;
  }
  __syncthreads();
  if (!last_layer) return;
  __threadfence();
  if (*reinterpret_cast<volatile int*>(a.irr_any)) layout_flat(a);
  if (threadIdx.x == 0) {
    sp.pdone[a.n_prunable] = 0;
    *a.irr_any = 0;
  }
}

void launch_select_project(const SelProjArgs& sp, const KeepArgs& a, int n_items, float* zn, uint32_t* mask,
                           size_t smem, cudaStream_t st) {
  const size_t need = std::max(smem, (size_t)kDepth * kThreads * sizeof(float4));
  allow_smem(k_select_project, need);
  launch_pdl(k_select_project, sp.nsel + n_items, kThreads, need, st, sp, a, zn, mask);
}

void launch_project(const KeepArgs& a, int n_items, float* zn, uint32_t* mask, int check, cudaStream_t st,
                    unsigned int* ready, unsigned int* pdone, ChainK67 c67, size_t fix_smem) {
  if (n_items <= 0) return;
  const size_t smem = (size_t)kDepth * kThreads * sizeof(float4);
  // TMA row copies (unchained launches; HSX_K3_TMA=0: per-thread cp.async quads)
  static const bool tma = [] {
    const char* v = std::getenv("HSX_K3_TMA");
    return v && v[0] == '1';
  }();
  if (tma && ready == nullptr) {
    const size_t sm = std::max(smem, kProjTmaSmem);
    if (check) {
      allow_smem(k_project<true, true>, std::max(sm, fix_smem));
      launch_pdl(k_project<true, true>, n_items, kThreads, std::max(sm, fix_smem), st, a, zn, mask, ready, pdone, c67);
    } else {
      allow_smem(k_project<false, true>, sm);
      launch_pdl(k_project<false, true>, n_items, kThreads, sm, st, a, zn, mask, ready, pdone, c67);
    }
    return;
  }
  if (check)
    launch_pdl(k_project<true, false>, n_items, kThreads, std::max(smem, fix_smem), st, a, zn, mask, ready, pdone,
               c67);
  else
    launch_pdl(k_project<false, false>, n_items, kThreads, smem, st, a, zn, mask, ready, pdone, c67);
}

// ---------------------------------------------------------------------------
// K4 mask union over leaders (transport.py:455-457): NCCL has no OR, so the
// leaders all-gather packed bits and OR them here.
// ---------------------------------------------------------------------------

__global__ void k_mask_or(MaskPtrs g, long long words, uint32_t* __restrict__ out, int vec) {
  PDL_ENTRY();
  const long long n4 = vec ? (words >> 2) : 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n4;
       i += (long long)gridDim.x * blockDim.x) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (int r = 0; r < g.n; ++r) {
      uint4 x = reinterpret_cast<const uint4*>(g.p[r])[i];
      acc.x |= x.x; acc.y |= x.y; acc.z |= x.z; acc.w |= x.w;
    }
    reinterpret_cast<uint4*>(out)[i] = acc;
  }
  for (long long i = n4 * 4 + blockIdx.x * (long long)blockDim.x + threadIdx.x; i < words;
       i += (long long)gridDim.x * blockDim.x) {
    uint32_t acc = 0;
    for (int r = 0; r < g.n; ++r) acc |= g.p[r][i];
    out[i] = acc;
  }
}

void launch_mask_or(const MaskPtrs& g, long long words, uint32_t* out, cudaStream_t st) {
  if (words <= 0 || g.n <= 0) return;
  int vec = 1;  // 16-B aligned sources (arenas and all-gather slices of words % 4 == 0)
  for (int r = 0; r < g.n; ++r) vec &= (reinterpret_cast<uintptr_t>(g.p[r]) & 15) == 0;
  long long n = vec ? (words >> 2) : words;
  int grid = (int)std::min<long long>(std::max<long long>((n + 255) / 256, 1), 148LL * 16);
  launch_pdl(k_mask_or, grid, 256, 0, st, g, words, out, vec);
}

// ---------------------------------------------------------------------------
// K5 keep sets from the union mask, one launch: items are word ranges of one
// layer; marks with a skip over the rest of each (o, c) kernel run.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) k_keep_sets(KeepArgs a) {
  PDL_ENTRY();
  extern __shared__ uint8_t sflag[];
  const Item it = a.items[blockIdx.x];
  const int l = it.layer;
  const DevLayer& ly = a.layers[l];
  const long long w0 = it.begin >> 5, w1 = (it.end + 31) >> 5;
  const long long r_lo = it.begin / ly.L;
  const long long r_hi = (std::min(it.end, ly.n) - 1) / ly.L;  // inclusive
  const int nr = (int)(r_hi - r_lo + 1);
  uint8_t* s_in = sflag;
  uint8_t* s_out = sflag + ly.cin;
  // rows of whole mask words (c_in kh kw % 32 == 0, every ResNet conv but the stem):
  // a row's "any" is its words' OR and the columns' "any" is the OR of the words at
  // each word position, so the marking is per word (a row flag + one shared-memory
  // atomicOr), and only the OR-ed column words are decoded into channels bit by bit
  const bool wordwise = (ly.L & 31) == 0;
  const int W = ly.L >> 5;
  uint32_t* s_col = reinterpret_cast<uint32_t*>(sflag + ((ly.cin + nr + 15) & ~15));
  for (int i = threadIdx.x; i < ly.cin + nr; i += kThreads) sflag[i] = 0;
  if (wordwise)
    for (int i = threadIdx.x; i < W; i += kThreads) s_col[i] = 0;
  __syncthreads();
  // a) marks and popcounts
  unsigned long long pop = 0, drift = 0;
  for (long long w = w0 + threadIdx.x; w < w1; w += kThreads) {
    long long e0 = w << 5;
    long long nvalid = ly.n - e0;
    uint32_t valid = nvalid >= 32 ? kFull : ((1u << nvalid) - 1u);
    uint32_t x;
    if (a.usrc.n) {  // fused union: OR of the leaders' words (over NVLink), stored once
      x = 0;
      for (int j = 0; j < a.usrc.n; ++j) x |= __ldcg(a.usrc.p[j] + ly.mword + w);
      a.uni_out[ly.mword + w] = x;
      x &= valid;
    } else {
      x = a.uni[ly.mword + w] & valid;
    }
    pop += __popc(x);
    if (a.prev) drift += __popc((x ^ a.prev[ly.mword + w]) & valid);
    if (wordwise) {
      if (x) {
        const unsigned o = fdiv((unsigned)e0, ly.divL);
        s_out[o - r_lo] = 1;
        atomicOr(s_col + ((unsigned)w - o * (unsigned)W), x);
      }
      continue;
    }
    while (x) {
      int b = __ffs(x) - 1;
      unsigned e = (unsigned)(e0 + b);
      unsigned o = fdiv(e, ly.divL);
      unsigned col = e - o * (unsigned)ly.L;
      unsigned c = fdiv(col, ly.divk);
      unsigned jx = col - c * (unsigned)ly.k;
      s_out[o - r_lo] = 1;
      s_in[c] = 1;
      int skip = b + (int)((unsigned)ly.k - jx);  // rest of this (o, c) kernel run
      x = skip >= 32 ? 0u : (x & ~((1u << skip) - 1u));
    }
  }
  __syncthreads();
  if (wordwise) {  // channels of the OR-ed column words
    for (int cw = threadIdx.x; cw < W; cw += kThreads) {
      uint32_t x = s_col[cw];
      while (x) {
        const int b = __ffs(x) - 1;
        const unsigned col = 32u * cw + b;
        const unsigned c = fdiv(col, ly.divk);
        s_in[c] = 1;
        const int skip = b + (int)((unsigned)ly.k - (col - c * (unsigned)ly.k));  // rest of the channel
        x = skip >= 32 ? 0u : (x & ~((1u << skip) - 1u));
      }
    }
    __syncthreads();
  }
  for (int i = threadIdx.x; i < ly.cin; i += kThreads)
    if (s_in[i]) a.iflag[ly.ikeep + i] = 1;
  for (int i = threadIdx.x; i < nr; i += kThreads)
    if (s_out[i]) a.oflag[ly.okeep + r_lo + i] = 1;
  __syncthreads();  // the tail reuses the mark flags' shared memory for positions
  keep_mark_done(a, l, ly, it.chunk, pop, drift);
}

void launch_keep_sets(const KeepArgs& a, int n_items, size_t smem, cudaStream_t st) {
  if (n_items <= 0) return;
  allow_smem(k_keep_sets, smem);
  launch_pdl(k_keep_sets, n_items, kThreads, smem, st, a);
}

// After the structured derivation (one CTA per prunable layer): a layer whose
// mask has a kept zero (irr bit 0, set by K3) is derived exactly from its mask
// bits; a layer whose previous mask was irregular (bit 1) gets its drift
// counted from the bits. The common case (neither) returns at once; when some
// layer was re-derived, the last CTA lays out the flat buffer again.
// smem: c_in + rows bytes.
// Per-layer part of the fixup (all of the layer's K3 items are done): exact keep
// sets / popcounts from the mask bits when the layer has a kept zero now (bit 0)
// or had one in the previous mask (bit 1, the drift reference); shifts the flag.
__device__ void fixup_layer(const KeepArgs& a, int l, uint8_t* fsm) {
  const DevLayer& gly = a.layers[l];
  const int pidx = gly.pidx;
  const int irr = a.irr[pidx];
  if (irr & 3) {
    const int cin = gly.cin, rows = gly.rows, k = gly.k, L = gly.L;
    const long long n = gly.n, mword = gly.mword, ikeep = gly.ikeep, okeep = gly.okeep;
    const FastDiv divL = gly.divL, divk = gly.divk;
    uint8_t* s_in = fsm;
    uint8_t* s_out = fsm + cin;
    const bool exact = irr & 1;
    for (int i = threadIdx.x; i < cin + rows; i += blockDim.x) fsm[i] = 0;
    __syncthreads();
    unsigned long long pop = 0, drift = 0;
    const long long nw = (n + 31) >> 5;
    for (long long w = threadIdx.x; w < nw; w += blockDim.x) {
      const long long e0 = w << 5;
      const long long nvalid = n - e0;
      const uint32_t valid = nvalid >= 32 ? kFull : ((1u << nvalid) - 1u);
      uint32_t x = a.uni[mword + w] & valid;
      pop += __popc(x);
      if (a.prev) drift += __popc((x ^ a.prev[mword + w]) & valid);
      while (exact && x) {  // marks, skipping the rest of each (o, c) kernel run
        const int b = __ffs(x) - 1;
        const unsigned e = (unsigned)(e0 + b);
        const unsigned o = fdiv(e, divL);
        const unsigned col = e - o * (unsigned)L;
        const unsigned c = fdiv(col, divk);
        const unsigned jx = col - c * (unsigned)k;
        s_out[o] = 1;
        s_in[c] = 1;
        const int skip = b + (int)((unsigned)k - jx);
        x = skip >= 32 ? 0u : (x & ~((1u << skip) - 1u));
      }
    }
    {
      const ulonglong2 t = block_sum2(pop, drift);
      pop = t.x;
      drift = t.y;
    }
    if (exact) {
      __syncthreads();
      const int2 nio = scan_keep<true>(s_in, cin, s_out, rows, a.pos_in + ikeep, a.pos_out + okeep);
      if (threadIdx.x == 0) {
        long long* row = a.summary + (long long)l * kSumCols;
        row[0] = nio.y;
        row[1] = nio.x;
        row[2] = (long long)nio.y * nio.x * k;
        row[5] = (long long)pop;
      }
    }
    if (threadIdx.x == 0) a.summary[(long long)l * kSumCols + 4] = (long long)drift;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    a.irr[pidx] = (irr & 1) << 1;  // this mask is the next one's previous
  }
}

__global__ void __launch_bounds__(kThreads) k_keep_fixup(KeepArgs a, const int* __restrict__ prunable) {
  PDL_ENTRY();
  extern __shared__ __align__(16) uint8_t fsm[];
  const int l = prunable[blockIdx.x];
  const int any = *reinterpret_cast<volatile int*>(a.irr_any);
  fixup_layer(a, l, fsm);
  if (!any) return;
  // some layer was re-derived: the last CTA lays the flat buffer out again
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.done, 1u) == (unsigned)a.n_prunable - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  layout_flat(a);
  if (threadIdx.x == 0) {
    *a.done = 0;
    *a.irr_any = 0;
  }
}

void launch_keep_fixup(const KeepArgs& a, const int* prunable, int n, size_t smem, cudaStream_t st) {
  if (n <= 0) return;
  allow_smem(k_keep_fixup, smem);
  launch_pdl(k_keep_fixup, n, kThreads, smem, st, a, prunable);
}

// ---------------------------------------------------------------------------
// K6 compact + intra dual; K7 decompact + inter dual.
// consensus.py:476-505, 535; shrinkage.py:61-82
// A thread owns element quads: the dense streams move as float4; the compact
// payload offset of element (o, c*k + j) is
//   coff + pos_out[o] * |K_in| * k + pos_in[c] * k + j
// (the row part per tile row in shared memory, the column part of a tile
// thread's quad in registers); a -1 position drops the coordinate.
// ---------------------------------------------------------------------------

// payload index of element e of a non-tiled prunable layer (-1: dropped)
__device__ __forceinline__ int elem_dst(const ElemArgs& a, const LayerRegs& ly, int rowlen, long long e) {
  const unsigned o = fdiv((unsigned)e, ly.divL);
  const unsigned col = (unsigned)e - o * (unsigned)ly.L;
  const unsigned c = fdiv(col, ly.divk), jx = col - c * (unsigned)ly.k;
  const int po = a.pos_out[ly.okeep + o], pi = a.pos_in[ly.ikeep + c];
  return (po < 0 || pi < 0) ? -1 : po * rowlen + pi * ly.k + (int)jx;
}

// payload indices of the quad at e of a contiguous item (dense or non-tiled prunable)
__device__ __forceinline__ int4 dst4_linear(const ElemArgs& a, const LayerRegs& ly, int rowlen, long long e) {
  if (ly.ncons == 0) {
    int b = (int)e;
    return make_int4(b, e + 1 < ly.n ? b + 1 : -1, e + 2 < ly.n ? b + 2 : -1, e + 3 < ly.n ? b + 3 : -1);
  }
  int4 d;
  d.x = elem_dst(a, ly, rowlen, e);
  d.y = e + 1 < ly.n ? elem_dst(a, ly, rowlen, e + 1) : -1;
  d.z = e + 2 < ly.n ? elem_dst(a, ly, rowlen, e + 2) : -1;
  d.w = e + 3 < ly.n ? elem_dst(a, ly, rowlen, e + 3) : -1;
  return d;
}

// column part of the payload offsets of a tile thread's quad (columns 4j .. 4j+3)
__device__ __forceinline__ int4 col_pos4(const ElemArgs& a, const LayerRegs& ly, int j, bool valid) {
  if (!valid) return make_int4(-1, -1, -1, -1);
  int v[4];
#pragma unroll
  for (int b = 0; b < 4; ++b) {
    const unsigned col = 4 * j + b, c = fdiv(col, ly.divk), jx = col - c * (unsigned)ly.k;
    const int pi = a.pos_in[ly.ikeep + c];
    v[b] = pi >= 0 ? pi * ly.k + (int)jx : -1;
  }
  return make_int4(v[0], v[1], v[2], v[3]);
}

// row parts of a tile's rows: pos_out[o] * |K_in| * k, or -1
__device__ __forceinline__ void row_base(const ElemArgs& a, const LayerRegs& ly, const Item& it, int rowlen,
                                         int* s_rb) {
  for (int r = threadIdx.x; r < it.end - it.begin; r += kThreads) {
    const int po = a.pos_out[ly.okeep + it.begin + r];
    s_rb[r] = po >= 0 ? po * rowlen : -1;
  }
}

__device__ __forceinline__ int4 add_base(int rb, int4 cp) {
  if (rb < 0) return make_int4(-1, -1, -1, -1);
  return make_int4(cp.x < 0 ? -1 : rb + cp.x, cp.y < 0 ? -1 : rb + cp.y, cp.z < 0 ? -1 : rb + cp.z,
                   cp.w < 0 ? -1 : rb + cp.w);
}

// fp64 sums of NS per-thread values over the block (xor-shuffle, then the warps in
// order: deterministic), written by thread 0 to out[0..NS)
template <int NS>
__device__ __forceinline__ void block_partials(double (&acc)[NS], double* __restrict__ out) {
  __shared__ double red[kThreads / 32][NS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) acc[q] += __shfl_xor_sync(kFull, acc[q], off);
    if (lane == 0) red[warp][q] = acc[q];
  }
  __syncthreads();
  if (threadIdx.x == 0) {
#pragma unroll
    for (int q = 0; q < NS; ++q) {
      double x = red[0][q];
      for (int w = 1; w < kThreads / 32; ++w) x += red[w][q];
      out[q] = x;
    }
  }
}

__device__ __forceinline__ double sqd(double x) { return x * x; }

// K6: flat[payload] <- z_node + v  (+ u <- u + (theta - z_node)) for one item.
// flat_out == nullptr: the intra dual alone (a follower's K6f). RESID: the item's
// sums of (theta - z_node)^2, theta^2, u'^2 (consensus.py:541-545) -> rpart slots 0-2.
template <bool RESID>
__global__ void __launch_bounds__(kThreads) k_compact(ElemArgs a) {
  PDL_ENTRY();
  extern __shared__ float4 ring[];
  __shared__ int s_rb[kMaxTileRows];
  const Item it = a.items[blockIdx.x];
  const LayerRegs ly(a.layers, it.layer);
  const long long coff = a.summary[(long long)it.layer * kSumCols + 3];
  const int rowlen = (int)a.summary[(long long)it.layer * kSumCols + 1] * ly.k;  // |K_in| * k
  const float* __restrict__ ZN = a.zn + ly.off;
  const float* __restrict__ VI = a.vin ? a.vin + ly.off : nullptr;
  const float* __restrict__ TH = a.u ? a.theta + ly.off : nullptr;
  float* __restrict__ UU = a.u ? a.u + ly.off : nullptr;
  float* __restrict__ flat = a.flat_out ? a.flat_out + coff : nullptr;
  double acc[3] = {0.0, 0.0, 0.0};
  // z_node is read again by K7 (keep resident), theta / u / v stream (evict first);
  // the compact buffer is written evict_last for K7's gather
  const unsigned long long pf = l2pol(kL2First), pl = l2pol(kL2Last);
  auto load4 = [&](int d, long long e) {
    cp_quad_h(ring_slot<4>(ring, d, 0), ZN, e, ly.n, pl);
    if (VI && flat) cp_quad_h(ring_slot<4>(ring, d, 1), VI, e, ly.n, pf);
    if (TH) {
      cp_quad_h(ring_slot<4>(ring, d, 2), TH, e, ly.n, pf);
      cp_quad_h(ring_slot<4>(ring, d, 3), UU, e, ly.n, pf);
    }
  };
  auto emit = [&](int d, long long e, int4 dd) {
    float4 zn = *ring_slot<4>(ring, d, 0);
    if (TH) {
      float4 th = *ring_slot<4>(ring, d, 2), uu = *ring_slot<4>(ring, d, 3);
      float4 un = make_float4(dual1(uu.x, th.x, zn.x), dual1(uu.y, th.y, zn.y), dual1(uu.z, th.z, zn.z),
                              dual1(uu.w, th.w, zn.w));
      if (RESID) {  // out-of-range lanes of a tail quad were zero-filled: they add 0
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const double t = f4get(th, i2);
          acc[0] += sqd(t - (double)f4get(zn, i2));
          acc[1] += sqd(t);
          acc[2] += sqd((double)f4get(un, i2));
        }
      }
      if (e + 3 < ly.n) {
        stcs4(UU + e, un);
      } else {
        for (int i2 = 0; i2 < 4 && e + i2 < ly.n; ++i2) UU[e + i2] = f4get(un, i2);
      }
    }
    if (!flat) return;
    float4 vv = VI ? *ring_slot<4>(ring, d, 1) : make_float4(0.f, 0.f, 0.f, 0.f);
    if (dd.x >= 0) flat[dd.x] = zn.x + vv.x;
    if (dd.y >= 0) flat[dd.y] = zn.y + vv.y;
    if (dd.z >= 0) flat[dd.z] = zn.z + vv.z;
    if (dd.w >= 0) flat[dd.w] = zn.w + vv.w;
  };
  if (it.tile == 1) {
    const TileCtx tc(it, ly.L);
    if (flat) row_base(a, ly, it, rowlen, s_rb);
    const int4 cp = flat ? col_pos4(a, ly, tc.j, tc.valid) : make_int4(-1, -1, -1, -1);
    __syncthreads();
    ring_run(tc.count, [&](int d, int i) { load4(d, tc.row(i) * ly.L + 4 * tc.j); },
             [&](int d, int i) {
               const long long r = tc.row(i);
               emit(d, r * ly.L + 4 * tc.j, flat ? add_base(s_rb[r - it.begin], cp) : cp);
             });
  } else {
    const long long nq = (it.end - it.begin + 3) >> 2;
    const int t = threadIdx.x;
    const int count = t < nq ? (int)((nq - t + kThreads - 1) / kThreads) : 0;
    ring_run(count, [&](int d, int i) { load4(d, it.begin + 4 * (t + (long long)i * kThreads)); },
             [&](int d, int i) {
               const long long e = it.begin + 4 * (t + (long long)i * kThreads);
               emit(d, e, flat ? dst4_linear(a, ly, rowlen, e) : make_int4(-1, -1, -1, -1));
             });
  }
  if (RESID) block_partials<3>(acc, a.rpart + (long long)blockIdx.x * kResidSlots);
}

void launch_compact(const ElemArgs& a, int n_items, cudaStream_t st) {
  if (n_items <= 0) return;
  const size_t smem = (size_t)kDepth * 4 * kThreads * sizeof(float4);
  if (a.rpart) {
    allow_smem(k_compact<true>, smem);
    launch_pdl(k_compact<true>, n_items, kThreads, smem, st, a);
  } else {
    allow_smem(k_compact<false>, smem);
    launch_pdl(k_compact<false>, n_items, kThreads, smem, st, a);
  }
}

// K7: z <- zero-filled gather of flat / divisor (+ v <- v + (z_node - z)); the
// gather streams through the ring: dropped coordinates are zero-filled by
// cp.async without touching memory. RESID: also streams the previous z (read
// before it is overwritten) and the previous z_node, and sums (z_node - z)^2,
// (z_node - z_node_prev)^2, z_node^2, v'^2, (z - z_prev)^2, z^2
// (consensus.py:552-563) -> rpart slots 3-8. RESID with flat_in == nullptr: a
// non-sync iteration (z, v unchanged, dz = 0, nothing stored).
// AVG2 (F1, two leaders): the leader average fused in — the compact values are
// gathered from both leaders' flat buffers (the other one over NVLink), folded in
// rank order in fp64 and divided by the divisor exactly as k_average does, written
// to the node's payload buffer zhat_out for the followers (when given) and
// decompacted in the same pass: bitwise the K8 -> K7 sequence without the K8 pass.
template <bool RESID, bool AVG2>
__global__ void __launch_bounds__(kThreads) k_decompact(ElemArgs a) {
  PDL_ENTRY();
  constexpr int NB = (RESID ? 5 : 3) + (AVG2 ? 1 : 0);
  constexpr int AS = NB - 1;             // AVG2: slot of the second leader's values
  constexpr int D = RESID ? 3 : kDepth;  // 5 streams x 3 stages: 60 KB, three CTAs per SM
  extern __shared__ float4 ring[];
  __shared__ int s_rb[kMaxTileRows];
  const Item it = a.items[blockIdx.x];
  const LayerRegs ly(a.layers, it.layer);
  const long long coff = a.summary[(long long)it.layer * kSumCols + 3];
  const int rowlen = (int)a.summary[(long long)it.layer * kSumCols + 1] * ly.k;  // |K_in| * k
  const bool sync = !RESID || a.flat_in != nullptr;
  const float* __restrict__ flat = sync ? a.flat_in + coff : nullptr;
  const float* __restrict__ flat2 = AVG2 ? a.flat_in2 + coff : nullptr;
  float* __restrict__ zhat = AVG2 && a.zhat_out ? a.zhat_out + coff : nullptr;
  const double adiv = a.avg_div;
  const float* __restrict__ ZN = a.v ? a.zn + ly.off : nullptr;
  float* __restrict__ VV = a.v ? a.v + ly.off : nullptr;
  float* __restrict__ ZO = a.z + ly.off;
  const float* __restrict__ ZP = RESID ? a.zn_prev + ly.off : nullptr;
  const float div = a.divisor;
  double acc[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const unsigned long long pf = l2pol(kL2First);
  auto load = [&](int d, long long e, int4 dd) {
    if (sync) {
      float* g = reinterpret_cast<float*>(ring_slot<NB>(ring, d, 0));
      cp4z(g + 0, flat + (dd.x >= 0 ? dd.x : 0), dd.x >= 0);
      cp4z(g + 1, flat + (dd.y >= 0 ? dd.y : 0), dd.y >= 0);
      cp4z(g + 2, flat + (dd.z >= 0 ? dd.z : 0), dd.z >= 0);
      cp4z(g + 3, flat + (dd.w >= 0 ? dd.w : 0), dd.w >= 0);
      if (AVG2) {
        float* h = reinterpret_cast<float*>(ring_slot<NB>(ring, d, AS));
        cp4z(h + 0, flat2 + (dd.x >= 0 ? dd.x : 0), dd.x >= 0);
        cp4z(h + 1, flat2 + (dd.y >= 0 ? dd.y : 0), dd.y >= 0);
        cp4z(h + 2, flat2 + (dd.z >= 0 ? dd.z : 0), dd.z >= 0);
        cp4z(h + 3, flat2 + (dd.w >= 0 ? dd.w : 0), dd.w >= 0);
      }
    }
    if (ZN) {  // last uses in the step: evict first
      cp_quad_h(ring_slot<NB>(ring, d, 1), ZN, e, ly.n, pf);
      cp_quad_h(ring_slot<NB>(ring, d, 2), VV, e, ly.n, pf);
    }
    if (RESID) {
      cp_quad_h(ring_slot<NB>(ring, d, RESID ? 3 : 0), ZP, e, ly.n, pf);
      cp_quad_h(ring_slot<NB>(ring, d, RESID ? 4 : 0), ZO, e, ly.n, pf);
    }
  };
  auto emit = [&](int d, long long e, int4 dd) {
    float4 zo;
    if (sync) {
      zo = *ring_slot<NB>(ring, d, 0);
      if (AVG2) {
        const float4 z2 = *ring_slot<NB>(ring, d, AS);
        zo = make_float4((float)__ddiv_rn(__dadd_rn((double)zo.x, (double)z2.x), adiv),
                         (float)__ddiv_rn(__dadd_rn((double)zo.y, (double)z2.y), adiv),
                         (float)__ddiv_rn(__dadd_rn((double)zo.z, (double)z2.z), adiv),
                         (float)__ddiv_rn(__dadd_rn((double)zo.w, (double)z2.w), adiv));
        if (zhat) {  // the node's averaged payload for the intra broadcast
          if (dd.x >= 0) zhat[dd.x] = zo.x;
          if (dd.y >= 0) zhat[dd.y] = zo.y;
          if (dd.z >= 0) zhat[dd.z] = zo.z;
          if (dd.w >= 0) zhat[dd.w] = zo.w;
        }
      } else if (div != 1.0f) {
        zo = make_float4(zo.x / div, zo.y / div, zo.z / div, zo.w / div);
      }
    } else {
      zo = *ring_slot<NB>(ring, d, RESID ? 4 : 0);
    }
    float4 vn;
    if (ZN) {
      float4 zn = *ring_slot<NB>(ring, d, 1), vv = *ring_slot<NB>(ring, d, 2);
      vn = sync ? make_float4(dual1(vv.x, zn.x, zo.x), dual1(vv.y, zn.y, zo.y), dual1(vv.z, zn.z, zo.z),
                              dual1(vv.w, zn.w, zo.w))
                : vv;
      if (RESID) {  // zero-filled tail lanes add 0
        const float4 zp = *ring_slot<NB>(ring, d, RESID ? 3 : 0), zold = *ring_slot<NB>(ring, d, RESID ? 4 : 0);
#pragma unroll
        for (int i2 = 0; i2 < 4; ++i2) {
          const double n = f4get(zn, i2), z = f4get(zo, i2);
          acc[0] += sqd(n - z);
          acc[1] += sqd(n - (double)f4get(zp, i2));
          acc[2] += sqd(n);
          acc[3] += sqd((double)f4get(vn, i2));
          if (sync) acc[4] += sqd(z - (double)f4get(zold, i2));
          acc[5] += sqd(z);
        }
      }
    }
    if (!sync) return;
    if (e + 3 < ly.n) {
      stcs4(ZO + e, zo);
      if (ZN) stcs4(VV + e, vn);
    } else {
      for (int i2 = 0; i2 < 4 && e + i2 < ly.n; ++i2) {
        ZO[e + i2] = f4get(zo, i2);
        if (ZN) VV[e + i2] = f4get(vn, i2);
      }
    }
  };
  if (it.tile == 1) {
    const TileCtx tc(it, ly.L);
    if (sync) row_base(a, ly, it, rowlen, s_rb);
    const int4 cp = sync ? col_pos4(a, ly, tc.j, tc.valid) : make_int4(-1, -1, -1, -1);
    __syncthreads();
    ring_run<D>(tc.count,
             [&](int d, int i) {
               const long long r = tc.row(i);
               load(d, r * ly.L + 4 * tc.j, sync ? add_base(s_rb[r - it.begin], cp) : cp);
             },
             [&](int d, int i) {
               const long long r = tc.row(i);
               emit(d, r * ly.L + 4 * tc.j, AVG2 ? add_base(s_rb[r - it.begin], cp) : cp);
             });
  } else {
    const long long nq = (it.end - it.begin + 3) >> 2;
    const int t = threadIdx.x;
    const int count = t < nq ? (int)((nq - t + kThreads - 1) / kThreads) : 0;
    ring_run<D>(count,
             [&](int d, int i) {
               const long long e = it.begin + 4 * (t + (long long)i * kThreads);
               load(d, e, sync ? dst4_linear(a, ly, rowlen, e) : make_int4(-1, -1, -1, -1));
             },
             [&](int d, int i) {
               const long long e = it.begin + 4 * (t + (long long)i * kThreads);
               emit(d, e, AVG2 ? dst4_linear(a, ly, rowlen, e) : make_int4(-1, -1, -1, -1));
             });
  }
  if (RESID) block_partials<6>(acc, a.rpart + (long long)blockIdx.x * kResidSlots + 3);
}

template <bool AVG2>
static void launch_decompact_a(const ElemArgs& a, int n_items, cudaStream_t st) {
  constexpr int X = AVG2 ? 1 : 0;
  if (a.rpart) {
    const size_t smem = (size_t)3 * (5 + X) * kThreads * sizeof(float4);
    allow_smem(k_decompact<true, AVG2>, smem);
    launch_pdl(k_decompact<true, AVG2>, n_items, kThreads, smem, st, a);
  } else {
    const size_t smem = (size_t)kDepth * (3 + X) * kThreads * sizeof(float4);
    allow_smem(k_decompact<false, AVG2>, smem);
    launch_pdl(k_decompact<false, AVG2>, n_items, kThreads, smem, st, a);
  }
}

void launch_decompact(const ElemArgs& a, int n_items, cudaStream_t st) {
  if (n_items <= 0) return;
  if (a.flat_in2)
    launch_decompact_a<true>(a, n_items, st);
  else
    launch_decompact_a<false>(a, n_items, st);
}

// K6+K7 of one node (M == 1), fused: the leader average is the identity, so the
// compact round trip z = decompress(compress(z_node + v)) is z = z_node + v on the
// kept rectangle K_out x K_in and 0 elsewhere — computed in place without the
// flat buffer (bitwise what K6 then K7 produce: the same fp32 add, / 1):
//   u <- u + (theta - z_node); z <- kept ? z_node + v : 0; v <- v + (z_node - z)
// RESID: the K6 (0-2) and K7 (3-8) residual slots in one pass (z_prev, z_node_prev
// streamed too).
// Chained (a.c67.ready3 != nullptr, behind a chained K3 that ran the fixups): the
// CTA lets its dependents launch, waits for its layer's projection (ready3[layer];
// dense layers: the upstream flag K3 sets once K1 and K2 are complete), runs, and
// waits for the grid before it at the end; the layer's last item / the launch's last
// item re-zero the flags for the next step.
template <bool RESID>
__global__ void __launch_bounds__(kThreads) k_local_sync(ElemArgs a) {
  const bool chained = a.c67.ready3 != nullptr;
  if (!chained) {
    PDL_ENTRY();
  } else {
    pdl_trigger();
    if (threadIdx.x == 0) {
      const Item& itc = a.items[blockIdx.x];
      const unsigned* f = a.layers[itc.layer].ncons > 0 ? a.c67.ready3 + itc.layer : a.c67.upstream;
      unsigned v;
      for (;;) {
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(f) : "memory");
        if (v) break;
        __nanosleep(128);
      }
    }
    __syncthreads();
  }
  constexpr int NB = RESID ? 6 : 4;
  constexpr int D = RESID ? 3 : kDepth;  // 6 x 3 x 4 KB = 72 KB / 4 x 4 x 4 KB = 64 KB
  extern __shared__ float4 ring[];
  __shared__ int s_rb[kMaxTileRows];
  const Item it = a.items[blockIdx.x];
  const LayerRegs ly(a.layers, it.layer);
  const int rowlen = (int)a.summary[(long long)it.layer * kSumCols + 1] * ly.k;  // |K_in| * k
  const float* __restrict__ ZN = a.zn + ly.off;
  const float* __restrict__ TH = a.theta + ly.off;
  float* __restrict__ UU = a.u + ly.off;
  float* __restrict__ VV = a.v + ly.off;
  float* __restrict__ ZO = a.z + ly.off;
  const float* __restrict__ ZP = RESID ? a.zn_prev + ly.off : nullptr;
  double acc[9] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const unsigned long long pf = l2pol(kL2First);
  auto load = [&](int d, long long e) {
    cp_quad_h(ring_slot<NB>(ring, d, 0), ZN, e, ly.n, pf);
    cp_quad_h(ring_slot<NB>(ring, d, 1), VV, e, ly.n, pf);
    cp_quad_h(ring_slot<NB>(ring, d, 2), TH, e, ly.n, pf);
    cp_quad_h(ring_slot<NB>(ring, d, 3), UU, e, ly.n, pf);
    if (RESID) {
      cp_quad_h(ring_slot<NB>(ring, d, RESID ? 4 : 0), ZP, e, ly.n, pf);
      cp_quad_h(ring_slot<NB>(ring, d, RESID ? 5 : 0), ZO, e, ly.n, pf);
    }
  };
  auto emit = [&](int d, long long e, int4 dd) {
    const float4 zn = *ring_slot<NB>(ring, d, 0), vv = *ring_slot<NB>(ring, d, 1);
    const float4 th = *ring_slot<NB>(ring, d, 2), uu = *ring_slot<NB>(ring, d, 3);
    const float4 un = make_float4(dual1(uu.x, th.x, zn.x), dual1(uu.y, th.y, zn.y), dual1(uu.z, th.z, zn.z),
                                  dual1(uu.w, th.w, zn.w));
    const float4 zo = make_float4(dd.x >= 0 ? zn.x + vv.x : 0.f, dd.y >= 0 ? zn.y + vv.y : 0.f,
                                  dd.z >= 0 ? zn.z + vv.z : 0.f, dd.w >= 0 ? zn.w + vv.w : 0.f);
    const float4 vn = make_float4(dual1(vv.x, zn.x, zo.x), dual1(vv.y, zn.y, zo.y), dual1(vv.z, zn.z, zo.z),
                                  dual1(vv.w, zn.w, zo.w));
    if (RESID) {  // zero-filled tail lanes add 0
      const float4 zp = *ring_slot<NB>(ring, d, RESID ? 4 : 0), zold = *ring_slot<NB>(ring, d, RESID ? 5 : 0);
#pragma unroll
      for (int i2 = 0; i2 < 4; ++i2) {
        const double t = f4get(th, i2), n = f4get(zn, i2), z = f4get(zo, i2);
        acc[0] += sqd(t - n);
        acc[1] += sqd(t);
        acc[2] += sqd((double)f4get(un, i2));
        acc[3] += sqd(n - z);
        acc[4] += sqd(n - (double)f4get(zp, i2));
        acc[5] += sqd(n);
        acc[6] += sqd((double)f4get(vn, i2));
        acc[7] += sqd(z - (double)f4get(zold, i2));
        acc[8] += sqd(z);
      }
    }
    if (e + 3 < ly.n) {
      stcs4(UU + e, un);
      stcs4(ZO + e, zo);
      stcs4(VV + e, vn);
    } else {
      for (int i2 = 0; i2 < 4 && e + i2 < ly.n; ++i2) {
        UU[e + i2] = f4get(un, i2);
        ZO[e + i2] = f4get(zo, i2);
        VV[e + i2] = f4get(vn, i2);
      }
    }
  };
  if (it.tile == 1) {
    const TileCtx tc(it, ly.L);
    row_base(a, ly, it, rowlen, s_rb);
    const int4 cp = col_pos4(a, ly, tc.j, tc.valid);
    __syncthreads();
    ring_run<D>(tc.count, [&](int d, int i) { load(d, tc.row(i) * ly.L + 4 * tc.j); },
                [&](int d, int i) {
                  const long long r = tc.row(i);
                  emit(d, r * ly.L + 4 * tc.j, add_base(s_rb[r - it.begin], cp));
                });
  } else {
    const long long nq = (it.end - it.begin + 3) >> 2;
    const int t = threadIdx.x;
    const int count = t < nq ? (int)((nq - t + kThreads - 1) / kThreads) : 0;
    ring_run<D>(count, [&](int d, int i) { load(d, it.begin + 4 * (t + (long long)i * kThreads)); },
                [&](int d, int i) {
                  const long long e = it.begin + 4 * (t + (long long)i * kThreads);
                  emit(d, e, dst4_linear(a, ly, rowlen, e));
                });
  }
  if (RESID) block_partials<9>(acc, a.rpart + (long long)blockIdx.x * kResidSlots);
  if (chained) {
    // after the grid wait the chained K3 is complete (its last upstream store too), so
    // the last item to get here may re-zero the flags: every item is past its wait
    pdl_wait();
    __syncthreads();
    if (threadIdx.x == 0) {
      const int l = it.layer;
      if (a.layers[l].ncons > 0 && atomicAdd(a.c67.cnt + l, 1u) == (unsigned)a.c67.count[l] - 1) {
        a.c67.cnt[l] = 0;
        a.c67.ready3[l] = 0;
      }
      if (atomicAdd(a.c67.all, 1u) == gridDim.x - 1) {
        *a.c67.all = 0;
        *a.c67.upstream = 0;
      }
    }
  }
}

void launch_local_sync(const ElemArgs& a, int n_items, cudaStream_t st) {
  if (n_items <= 0) return;
  if (a.rpart) {
    const size_t smem = (size_t)3 * 6 * kThreads * sizeof(float4);
    allow_smem(k_local_sync<true>, smem);
    launch_pdl(k_local_sync<true>, n_items, kThreads, smem, st, a);
  } else {
    const size_t smem = (size_t)kDepth * 4 * kThreads * sizeof(float4);
    allow_smem(k_local_sync<false>, smem);
    launch_pdl(k_local_sync<false>, n_items, kThreads, smem, st, a);
  }
}

// ---------------------------------------------------------------------------
// Phase 5 (consensus.py:537-598): per-layer fold of the item partials, the
// residual report (consensus.py:239-288) and residual balancing
// (consensus.py:189-219) with the penalties updated in the device layer table,
// then the dual rescale u *= u_scale, v *= v_scale of the layers that changed.
// ---------------------------------------------------------------------------

// vec[l][q]: one CTA per layer, warp q folds slot q — lane i sums items i, i+32, ...
// in order (loads batched), then a fixed xor-shuffle tree: deterministic
__global__ void __launch_bounds__(32 * kResidSlots) k_resid_fold(ResidArgs a) {
  PDL_ENTRY();
  const int l = blockIdx.x, q = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double x = 0.0;
  if (q < 3 || a.leader) {
    const int f = a.first[l], c = a.count[l];
    const double* __restrict__ src = a.rpart + (long long)f * kResidSlots + q;
    for (int j0 = lane; j0 < c; j0 += 32 * 8) {
      double v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = j0 + 32 * u < c ? src[(long long)(j0 + 32 * u) * kResidSlots] : 0.0;
#pragma unroll
      for (int u = 0; u < 8; ++u) x += v[u];
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) x += __shfl_xor_sync(kFull, x, off);
  }
  if (lane == 0) a.vec[(long long)l * kResidSlots + q] = x;
}

void launch_resid_fold(const ResidArgs& a, cudaStream_t st) {
  if (a.n_layers <= 0) return;
  launch_pdl(k_resid_fold, a.n_layers, 32 * kResidSlots, 0, st, a);
}

// One CTA: thread per layer. With a.global: the report of every layer, the
// totals folded in layer order by thread 0 (the reference's accumulation order),
// then (adapt) the new penalties. Without: penalties adapted from a received report.
__global__ void __launch_bounds__(512) k_report(ResidArgs a) {
  PDL_ENTRY();
  __shared__ double tot[4];
  const int L = a.n_layers;
  const double world = (double)a.num_nodes * a.per_node;
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    DevLayer& ly = a.layers[l];
    double* rp = a.report + (long long)l * 8;
    if (a.global) {
      const double* g = a.global + (long long)l * kResidSlots;
      const double n = (double)ly.n;
      const double r_intra = sqrt(g[0]);
      const double s_intra = __dmul_rn(ly.rho1, sqrt(__dmul_rn((double)a.per_node, g[4])));
      const double r_inter = sqrt(g[3]);
      const double s_inter = __dmul_rn(ly.rho2, sqrt(g[7]));
      const double e_i = __dmul_rn(sqrt(__dmul_rn(n, world)), a.eps_abs);
      const double e_o = __dmul_rn(sqrt(__dmul_rn(n, (double)a.num_nodes)), a.eps_abs);
      rp[0] = r_intra;
      rp[1] = s_intra;
      rp[2] = r_inter;
      rp[3] = s_inter;
      rp[4] = __dadd_rn(e_i, __dmul_rn(a.eps_rel, fmax(sqrt(g[1]), sqrt(__dmul_rn((double)a.per_node, g[5])))));
      rp[5] = __dadd_rn(e_i, __dmul_rn(__dmul_rn(a.eps_rel, ly.rho1), sqrt(g[2])));
      rp[6] = __dadd_rn(e_o, __dmul_rn(a.eps_rel, fmax(sqrt(g[5]), sqrt(g[8]))));
      rp[7] = __dadd_rn(e_o, __dmul_rn(__dmul_rn(a.eps_rel, ly.rho2), sqrt(g[6])));
      if (a.flat) rp[2] = rp[3] = rp[6] = rp[7] = 0.0;  // baselines.py:249 (no inter level)
    }
  }
  __syncthreads();
  if (a.global && threadIdx.x == 0) {
    double s[4] = {0.0, 0.0, 0.0, 0.0};
    for (int l = 0; l < L; ++l) {
      const double* rp = a.report + (long long)l * 8;
      s[0] = __dadd_rn(s[0], __dadd_rn(__dmul_rn(rp[0], rp[0]), __dmul_rn(rp[2], rp[2])));
      s[1] = __dadd_rn(s[1], __dadd_rn(__dmul_rn(rp[1], rp[1]), __dmul_rn(rp[3], rp[3])));
      s[2] = __dadd_rn(s[2], __dadd_rn(__dmul_rn(rp[4], rp[4]), __dmul_rn(rp[6], rp[6])));
      s[3] = __dadd_rn(s[3], __dadd_rn(__dmul_rn(rp[5], rp[5]), __dmul_rn(rp[7], rp[7])));
    }
    double* t = a.report + (long long)L * 8;
    for (int q = 0; q < 4; ++q) t[q] = tot[q] = sqrt(s[q]);
    t[4] = (tot[0] <= tot[2] && tot[1] <= tot[3]) ? 1.0 : 0.0;
  }
  __syncthreads();
  for (int l = threadIdx.x; l < L; l += blockDim.x) {
    DevLayer& ly = a.layers[l];
    const double* rp = a.report + (long long)l * 8;
    double su = 1.0, sv = 1.0;
    if (a.adapt) {
      const double old = ly.rho1, old2 = ly.rho2;
      double r1 = old, r2 = old2;
      if (rp[0] > __dmul_rn(a.mu, rp[1]))
        r1 = fmin(__dmul_rn(old, a.tau_inc), a.rho1_max);
      else if (rp[1] > __dmul_rn(a.mu, rp[0]))
        r1 = __ddiv_rn(old, a.tau_dec);
      if (rp[2] > __dmul_rn(a.mu, rp[3]))
        r2 = fmin(__dmul_rn(old2, a.tau_inc), a.rho2_max);
      else if (rp[3] > __dmul_rn(a.mu, rp[2]))
        r2 = __ddiv_rn(old2, a.tau_dec);
      if (r1 != old) su = __ddiv_rn(old, r1);
      if (r2 != old2) sv = __ddiv_rn(old2, r2);
      if (r1 != old || r2 != old2) {  // consensus.py:157-159, same expression order as the host
        ly.rho1 = r1;
        ly.rho2 = r2;
        const double gamma =
            __dadd_rn(__dadd_rn(__ddiv_rn(a.wd, (double)a.num_nodes), __dmul_rn((double)a.per_node, r1)), r2);
        ly.gamma = gamma;
        ly.rgamma = __drcp_rn(gamma);
      }
    }
    a.scales[l] = su;
    a.scales[L + l] = sv;
  }
}

void launch_report(const ResidArgs& a, cudaStream_t st) {
  if (a.n_layers <= 0) return;
  launch_pdl(k_report, 1, 512, 0, st, a);
}

// u *= scale_u[l], v *= scale_v[l] over the stream items of layers whose scale != 1
__global__ void __launch_bounds__(kThreads) k_scale_duals(const DevLayer* __restrict__ layers,
                                                         const Item* __restrict__ items,
                                                         const double* __restrict__ scales, int n_layers,
                                                         float* __restrict__ u, float* __restrict__ v) {
  PDL_ENTRY();
  const Item it = items[blockIdx.x];
  const double su = scales[it.layer], sv = scales[n_layers + it.layer];
  if (su == 1.0 && sv == 1.0) return;
  const DevLayer& ly = layers[it.layer];
  const long long b = it.begin, e = it.end;  // contiguous element items (8192, quad-aligned)
  const long long nq = (e - b) >> 2;
  constexpr int U = 8;
  float4* __restrict__ u4 = reinterpret_cast<float4*>(u + ly.off + b);
  float4* __restrict__ v4 = reinterpret_cast<float4*>(v + ly.off + b);
  auto sc = [](float4 x, double s) {
    return make_float4((float)((double)x.x * s), (float)((double)x.y * s), (float)((double)x.z * s),
                       (float)((double)x.w * s));
  };
  for (long long q0 = threadIdx.x; q0 < nq; q0 += (long long)U * kThreads) {
    float4 xu[U], xv[U];
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long q = q0 + (long long)j * kThreads;
      if (q < nq) {
        if (su != 1.0) xu[j] = u4[q];
        if (sv != 1.0) xv[j] = v4[q];
      }
    }
#pragma unroll
    for (int j = 0; j < U; ++j) {
      const long long q = q0 + (long long)j * kThreads;
      if (q < nq) {
        if (su != 1.0) u4[q] = sc(xu[j], su);
        if (sv != 1.0) v4[q] = sc(xv[j], sv);
      }
    }
  }
  for (long long i = b + 4 * nq + threadIdx.x; i < e; i += kThreads) {
    if (su != 1.0) u[ly.off + i] = (float)((double)u[ly.off + i] * su);
    if (sv != 1.0) v[ly.off + i] = (float)((double)v[ly.off + i] * sv);
  }
}

void launch_scale_duals(const DevLayer* layers, const Item* items, int n_items, const double* scales,
                        int n_layers, float* u, float* v, cudaStream_t st) {
  if (n_items <= 0) return;
  launch_pdl(k_scale_duals, n_items, kThreads, 0, st, layers, items, scales, n_layers, u, v);
}

// ---------------------------------------------------------------------------
// Leader average over NVLink (the leader all-reduce AVG, transport.py:453-462,
// as a contiguous stream): out[i] = fp32((sum_j src_j[i], rank order, fp64) / div)
// for i < the payload size read from the device summary (no host sync). Also the
// followers' copy of their leader's averaged payload (n = 1, div = 1).
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) k_average(PeerPtrs src, const long long* __restrict__ total_p,
                                                      double div, float* __restrict__ out) {
  PDL_ENTRY();
  const long long total = *total_p;
  const long long n4 = total >> 2;
  const long long stride = (long long)gridDim.x * kThreads;
  constexpr int U = 4;
  for (long long i0 = blockIdx.x * (long long)kThreads + threadIdx.x; i0 < n4; i0 += stride * U) {
    float4 x[U][kMaxPeers];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      const long long i = i0 + uu * stride;
#pragma unroll
      for (int j = 0; j < kMaxPeers; ++j)
        if (j < src.n && i < n4) x[uu][j] = __ldcg(reinterpret_cast<const float4*>(src.p[j]) + i);
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      const long long i = i0 + uu * stride;
      if (i >= n4) break;
      double s0 = x[uu][0].x, s1 = x[uu][0].y, s2 = x[uu][0].z, s3 = x[uu][0].w;
#pragma unroll
      for (int j = 1; j < kMaxPeers; ++j) {
        if (j >= src.n) break;
        s0 = __dadd_rn(s0, (double)x[uu][j].x); s1 = __dadd_rn(s1, (double)x[uu][j].y);
        s2 = __dadd_rn(s2, (double)x[uu][j].z); s3 = __dadd_rn(s3, (double)x[uu][j].w);
      }
      reinterpret_cast<float4*>(out)[i] = make_float4((float)__ddiv_rn(s0, div), (float)__ddiv_rn(s1, div),
                                                      (float)__ddiv_rn(s2, div), (float)__ddiv_rn(s3, div));
    }
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)kThreads + threadIdx.x; i < total; i += stride) {
    double s = src.p[0][i];
    for (int j = 1; j < src.n; ++j) s = __dadd_rn(s, (double)src.p[j][i]);
    out[i] = (float)__ddiv_rn(s, div);
  }
}

void launch_average(const PeerPtrs& src, const long long* total, long long max_elems, double div, float* out,
                    cudaStream_t st) {
  if (src.n <= 0 || max_elems <= 0) return;
  int grid = (int)std::min<long long>(std::max<long long>((max_elems / 4 + kThreads - 1) / kThreads, 1), 148LL * 8);
  launch_pdl(k_average, grid, kThreads, 0, st, src, total, div, out);
}

// ---------------------------------------------------------------------------
// Slice collectives over NVLink for groups of >= 3 ranks (reduce-scatter +
// all-gather move 2(n-1)/n of the buffer per rank instead of (n-1)):
//   part >= 0: out[i] = fp32((sum_j src_j[i], rank order, fp64) / div) on slice
//              `part` of [0, total) (slices of ceil(total / n) rounded to 32);
//   part <  0: out[i] = src_{owner(i)}[i] on [0, total) (gather the slices).
// total is a host value or, when total_p != NULL, read on the device.
// ---------------------------------------------------------------------------

__global__ void __launch_bounds__(kThreads) k_slices(PeerPtrs src, const long long* __restrict__ total_p,
                                                     long long total_h, int part, double div,
                                                     float* __restrict__ out) {
  PDL_ENTRY();
  const long long total = total_p ? *total_p : total_h;
  const long long slice = ((total + src.n - 1) / src.n + 31) / 32 * 32;
  long long b = 0, e = total;
  if (part >= 0) {
    b = std::min<long long>((long long)part * slice, total);
    e = std::min<long long>(b + slice, total);
  }
  const long long stride = (long long)gridDim.x * kThreads;
  const long long q0 = b >> 2, q1 = e >> 2;  // slice bounds are multiples of 32
  for (long long q = q0 + blockIdx.x * (long long)kThreads + threadIdx.x; q < q1; q += stride) {
    float4 r;
    if (part >= 0) {
      float4 x = __ldcg(reinterpret_cast<const float4*>(src.p[0]) + q);
      double s0 = x.x, s1 = x.y, s2 = x.z, s3 = x.w;
      for (int j = 1; j < src.n; ++j) {
        x = __ldcg(reinterpret_cast<const float4*>(src.p[j]) + q);
        s0 = __dadd_rn(s0, (double)x.x); s1 = __dadd_rn(s1, (double)x.y);
        s2 = __dadd_rn(s2, (double)x.z); s3 = __dadd_rn(s3, (double)x.w);
      }
      r = make_float4((float)__ddiv_rn(s0, div), (float)__ddiv_rn(s1, div), (float)__ddiv_rn(s2, div),
                      (float)__ddiv_rn(s3, div));
    } else {
      const int owner = (int)std::min<long long>((4 * q) / slice, src.n - 1);
      r = __ldcg(reinterpret_cast<const float4*>(src.p[owner]) + q);
    }
    reinterpret_cast<float4*>(out)[q] = r;
  }
  // tail of the last slice (total not a multiple of 4)
  for (long long i = 4 * q1 + blockIdx.x * (long long)kThreads + threadIdx.x; i < e; i += stride) {
    if (part >= 0) {
      double sum = src.p[0][i];
      for (int j = 1; j < src.n; ++j) sum = __dadd_rn(sum, (double)src.p[j][i]);
      out[i] = (float)__ddiv_rn(sum, div);
    } else {
      const int owner = (int)std::min<long long>(i / slice, src.n - 1);
      out[i] = src.p[owner][i];
    }
  }
}

void launch_slices(const PeerPtrs& src, const long long* total_p, long long total_h, long long max_elems,
                   int part, double div, float* out, cudaStream_t st) {
  if (src.n <= 0 || max_elems <= 0) return;
  const long long span = part >= 0 ? (max_elems + src.n - 1) / src.n : max_elems;
  int grid = (int)std::min<long long>(std::max<long long>((span / 4 + kThreads - 1) / kThreads, 1), 148LL * 8);
  launch_pdl(k_slices, grid, kThreads, 0, st, src, total_p, total_h, part, div, out);
}

// ---------------------------------------------------------------------------
// Group barrier over NVLink: member i publishes `epoch` into slot `slots[me]` of
// every other member's flag array (release, system scope) and waits until its
// own slots of all other members reach `epoch` (acquire). Stream-ordered: the
// kernels before it have completed, the kernels after it read peers' buffers.
// A member that has not arrived after the timeout (HSX_BARRIER_TIMEOUT_S, default
// 600 s; 0 waits forever, like an NCCL collective) is not a sticky trap: the waiter
// counts the timeout in g_barrier_timeouts and lets the stream continue, and the
// host raises ProtocolError when it next reads the counter (hsx_barrier_timeouts).
// ---------------------------------------------------------------------------

__device__ unsigned int g_barrier_timeouts;

__global__ void k_barrier(BarrierArgs b) {
  const int i = threadIdx.x;
  if (b.mode != 2 && i < b.n && i != b.me) {
    __threadfence_system();
    int* dst = b.flags[i] + b.slots[b.me];
    asm volatile("st.release.sys.global.s32 [%0], %1;" ::"l"(dst), "r"(b.epoch) : "memory");
  }
  __syncwarp();
  if (b.mode != 1 && i < b.n && i != b.me && (b.mode == 0 || i == b.root)) {
    const int* src = b.flags[b.me] + b.slots[i];
    const unsigned long long t0 = global_ns();
    int v;
    while (true) {
      asm volatile("ld.acquire.sys.global.s32 %0, [%1];" : "=r"(v) : "l"(src) : "memory");
      if (v - b.epoch >= 0) break;
      if (b.timeout_ns && global_ns() - t0 > b.timeout_ns) {
        atomicAdd(&g_barrier_timeouts, 1u);
        break;
      }
      __nanosleep(64);
    }
  }
  __syncwarp();
  __threadfence_system();
}

static unsigned long long barrier_timeout_ns() {
  static const unsigned long long ns = [] {
    const char* v = std::getenv("HSX_BARRIER_TIMEOUT_S");
    const double s = v ? std::atof(v) : 600.0;
    return s > 0 ? (unsigned long long)(s * 1e9) : 0ull;
  }();
  return ns;
}

int barrier_timeouts(unsigned int* count, int reset) {
  if (cudaMemcpyFromSymbol(count, g_barrier_timeouts, sizeof(unsigned int)) != cudaSuccess) return -1;
  if (reset) {
    const unsigned int zero = 0;
    if (cudaMemcpyToSymbol(g_barrier_timeouts, &zero, sizeof(unsigned int)) != cudaSuccess) return -1;
  }
  return 0;
}

void launch_barrier(const BarrierArgs& b, cudaStream_t st) {
  BarrierArgs a = b;
  a.timeout_ns = barrier_timeout_ns();
  k_barrier<<<1, 32, 0, st>>>(a);
}

// ---------------------------------------------------------------------------
// K0 send = theta + u; K6f u += theta - z_node (arena-wide streaming)
// ---------------------------------------------------------------------------

static int stream_grid(long long n4) {
  long long g = (n4 + kThreads - 1) / kThreads;
  return (int)std::min<long long>(std::max<long long>(g, 1), 148LL * 8);
}

__global__ void __launch_bounds__(kThreads) k_add(const float* __restrict__ a,
                                                  const float* __restrict__ b,
                                                  float* __restrict__ out, long long n) {
  PDL_ENTRY();
  const long long n4 = n >> 2;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n4; i += stride) {
    float4 x = ldcs4(a + 4 * i), y = ldcs4(b + 4 * i);
    st4(out + 4 * i, make_float4(x.x + y.x, x.y + y.y, x.z + y.z, x.w + y.w));
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += stride)
    out[i] = a[i] + b[i];
}

void launch_add(const float* a, const float* b, float* out, long long n, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_add, stream_grid(n >> 2), kThreads, 0, st, a, b, out, n);
}

__global__ void __launch_bounds__(kThreads) k_dual(const float* __restrict__ th,
                                                   float* __restrict__ u,
                                                   const float* __restrict__ zn, long long n) {
  PDL_ENTRY();
  const long long n4 = n >> 2;
  const long long stride = (long long)gridDim.x * kThreads;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n4; i += stride) {
    float4 t = ldcs4(th + 4 * i), x = ldcs4(u + 4 * i), z = ldcs4(zn + 4 * i);
    stcs4(u + 4 * i, make_float4(dual1(x.x, t.x, z.x), dual1(x.y, t.y, z.y), dual1(x.z, t.z, z.z),
                                 dual1(x.w, t.w, z.w)));
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += stride)
    u[i] = dual1(u[i], th[i], zn[i]);
}

void launch_dual(const float* theta, float* u, const float* zn, long long n, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_dual, stream_grid(n >> 2), kThreads, 0, st, theta, u, zn, n);
}

// ---------------------------------------------------------------------------
// small mask helpers for the per-tensor API
// ---------------------------------------------------------------------------

__global__ void k_nonzero(const float* __restrict__ t, long long n, uint8_t* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    out[i] = fabsf(t[i]) > 0.0f ? 1 : 0;
}

__global__ void k_pack(const uint8_t* __restrict__ m, long long n, uint32_t* __restrict__ bits) {
  const long long words = (n + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const long long warp0 = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
  const long long nwarps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long w = warp0; w < words; w += nwarps) {
    long long e = (w << 5) + lane;
    unsigned b = __ballot_sync(kFull, e < n && m[e] != 0);
    if (lane == 0) bits[w] = b;
  }
}

__global__ void k_unpack(const uint32_t* __restrict__ bits, long long n, uint8_t* __restrict__ m) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    m[i] = (bits[i >> 5] >> (i & 31)) & 1u;
}

__global__ void k_count_diff(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                             long long n, unsigned long long* c) {
  unsigned long long cnt = 0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    cnt += (a[i] != 0) != (b[i] != 0);
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) cnt += __shfl_xor_sync(kFull, cnt, off);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(c, cnt);
}

static int small_grid(long long n) {
  return (int)std::min<long long>(std::max<long long>((n + 255) / 256, 1), 148LL * 8);
}

void launch_nonzero(const float* t, long long n, uint8_t* out, cudaStream_t st) {
  if (n > 0) k_nonzero<<<small_grid(n), 256, 0, st>>>(t, n, out);
}
void launch_pack(const uint8_t* m, long long n, uint32_t* bits, cudaStream_t st) {
  if (n > 0) k_pack<<<small_grid(n), 256, 0, st>>>(m, n, bits);
}
void launch_unpack(const uint32_t* bits, long long n, uint8_t* m, cudaStream_t st) {
  if (n > 0) k_unpack<<<small_grid(n), 256, 0, st>>>(bits, n, m);
}
void launch_count_diff(const uint8_t* a, const uint8_t* b, long long n, unsigned long long* c,
                       cudaStream_t st) {
  if (n > 0) k_count_diff<<<small_grid(n), 256, 0, st>>>(a, b, n, c);
}

}  // namespace hsx

#ifdef HSX_TRACE
extern "C" int hsx_debug_trace(void* out, int n) {
  return (int)cudaMemcpyFromSymbol(out, hsx::g_trace, (size_t)n * 4 * sizeof(unsigned long long));
}
#endif

namespace hsx {
// ---------------------------------------------------------------------------
// Phase-1 boundary: one proximal-SGD step of the reference's
// solver (workloads.py:316-320), fused over every layer:
//   combined = grad + rho1_l * (theta - z_node + u); vel = momentum * vel + combined;
//   theta -= lr * vel
// in fp64 (the reference's order), rounded once to fp32; first: vel starts at 0
// (the solver zeroes it per outer iteration, :312); send != nullptr: also writes
// theta + u for the intra sum (K0 fused into the last step). rho1 comes from the
// device layer table, so device-side penalty adaptation is seen directly.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) k_prox_sgd(const DevLayer* __restrict__ layers,
                                                      const Item* __restrict__ items, const float* __restrict__ g,
                                                      float* __restrict__ th, const float* __restrict__ zn,
                                                      const float* __restrict__ u, float* __restrict__ vel,
                                                      float* __restrict__ send, double lr, double mom, int first) {
  PDL_ENTRY();
  const Item it = items[blockIdx.x];
  const DevLayer& ly = layers[it.layer];
  const double rho1 = ly.rho1;
  const long long off = ly.off;
  for (long long e = it.begin + threadIdx.x; e < it.end; e += kThreads) {
    const long long i = off + e;
    const double w = th[i];
    const double comb = __dadd_rn((double)g[i], __dmul_rn(rho1, __dadd_rn(__dsub_rn(w, (double)zn[i]), (double)u[i])));
    const double v = first ? comb : __dadd_rn(__dmul_rn(mom, (double)vel[i]), comb);
    const float wn = (float)__dsub_rn(w, __dmul_rn(lr, v));
    vel[i] = (float)v;
    th[i] = wn;
    if (send) send[i] = (float)__dadd_rn((double)wn, (double)u[i]);
  }
}

void launch_prox_sgd(const DevLayer* layers, const Item* items, int n_items, const float* g, float* th,
                     const float* zn, const float* u, float* vel, float* send, double lr, double mom, int first,
                     cudaStream_t st) {
  if (n_items <= 0) return;
  launch_pdl(k_prox_sgd, n_items, kThreads, 0, st, layers, items, g, th, zn, u, vel, send, lr, mom, first);
}

// ---------------------------------------------------------------------------
// Dense synchronous SGD baseline (baselines.py:77-98): per step every rank packs
// g = grad + wd * params (fp64 math, :88), the all-rank AVG, then velocity =
// momentum * velocity + avg, params -= lr * velocity (:90-92). Flat arena-wide
// float4 grid-stride kernels (HBM-bound: 12 B / 16 B per element + 4 B per peer).
// ---------------------------------------------------------------------------

__device__ __forceinline__ float dense_g(float g, float p, double wd) {
  return (float)__dadd_rn((double)g, __dmul_rn(wd, (double)p));
}

__device__ __forceinline__ void dense_upd(double avg, float& p, float& v, double lr, double mom, int first) {
  const double vn = first ? __dadd_rn(0.0, avg) : __dadd_rn(__dmul_rn(mom, (double)v), avg);
  v = (float)vn;
  p = (float)__dsub_rn((double)p, __dmul_rn(lr, vn));
}

__global__ void __launch_bounds__(kThreads) k_dense_pack(const float* __restrict__ g, const float* __restrict__ p,
                                                         double wd, float* __restrict__ send, long long n) {
  PDL_ENTRY();
  const long long n4 = n >> 2, stride = (long long)gridDim.x * kThreads;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n4; i += stride) {
    const float4 a = __ldcs(reinterpret_cast<const float4*>(g) + i), b = reinterpret_cast<const float4*>(p)[i];
    __stcg(reinterpret_cast<float4*>(send) + i,
           make_float4(dense_g(a.x, b.x, wd), dense_g(a.y, b.y, wd), dense_g(a.z, b.z, wd), dense_g(a.w, b.w, wd)));
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += stride)
    send[i] = dense_g(g[i], p[i], wd);
}

// avg = (sum_j src_j, rank order, fp64) / div over the peers' send buffers (the
// all-rank AVG fused with the update: one pass, no reduced buffer); n_peers == 1
// with div == 1 applies an already averaged buffer (the NCCL path)
__global__ void __launch_bounds__(kThreads) k_dense_apply(PeerPtrs src, double div, float* __restrict__ p,
                                                          float* __restrict__ v, double lr, double mom, int first,
                                                          long long n) {
  PDL_ENTRY();
  const long long n4 = n >> 2, stride = (long long)gridDim.x * kThreads;
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n4; i += stride) {
    float4 x[kMaxPeers];
#pragma unroll
    for (int j = 0; j < kMaxPeers; ++j)
      if (j < src.n) x[j] = __ldcg(reinterpret_cast<const float4*>(src.p[j]) + i);
    double s0 = x[0].x, s1 = x[0].y, s2 = x[0].z, s3 = x[0].w;
#pragma unroll
    for (int j = 1; j < kMaxPeers; ++j) {
      if (j >= src.n) break;
      s0 = __dadd_rn(s0, (double)x[j].x); s1 = __dadd_rn(s1, (double)x[j].y);
      s2 = __dadd_rn(s2, (double)x[j].z); s3 = __dadd_rn(s3, (double)x[j].w);
    }
    float4 pp = reinterpret_cast<float4*>(p)[i], vv = first ? make_float4(0.f, 0.f, 0.f, 0.f)
                                                            : reinterpret_cast<float4*>(v)[i];
    dense_upd(__ddiv_rn(s0, div), pp.x, vv.x, lr, mom, first);
    dense_upd(__ddiv_rn(s1, div), pp.y, vv.y, lr, mom, first);
    dense_upd(__ddiv_rn(s2, div), pp.z, vv.z, lr, mom, first);
    dense_upd(__ddiv_rn(s3, div), pp.w, vv.w, lr, mom, first);
    reinterpret_cast<float4*>(p)[i] = pp;
    reinterpret_cast<float4*>(v)[i] = vv;
  }
  for (long long i = 4 * n4 + blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += stride) {
    double s = src.p[0][i];
    for (int j = 1; j < src.n; ++j) s = __dadd_rn(s, (double)src.p[j][i]);
    float pp = p[i], vv = first ? 0.f : v[i];
    dense_upd(__ddiv_rn(s, div), pp, vv, lr, mom, first);
    p[i] = pp;
    v[i] = vv;
  }
}

static int dense_grid(long long n) {
  return (int)std::min<long long>(std::max<long long>((n / 4 + kThreads - 1) / kThreads, 1), 148LL * 8);
}

void launch_dense_pack(const float* g, const float* p, double wd, float* send, long long n, cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_dense_pack, dense_grid(n), kThreads, 0, st, g, p, wd, send, n);
}

void launch_dense_apply(const PeerPtrs& src, double div, float* p, float* v, double lr, double mom, int first,
                        long long n, cudaStream_t st) {
  if (n <= 0 || src.n <= 0) return;
  launch_pdl(k_dense_apply, dense_grid(n), kThreads, 0, st, src, div, p, v, lr, mom, first, n);
}

// ---------------------------------------------------------------------------
// Top-K gradient compression with error feedback (baselines.py:101-148).
// Per layer: acc = residual + grad + wd * params (fp64, in place in the fp64
// residual arena); an exact MSD radix select (8 passes of 8 bits over the key
// bits(|acc|), layers whose chosen bin holds exactly the remaining count stop
// early) gives the k-th largest key T and the number of ties to take; the
// selection (key > T, plus the lowest-index ties: the stable argsort of -|x|,
// :71-74) is written in ascending index order as (fp32 value, int32 index) pairs
// and zeroed in the residual (flat - kept, :142-144). The all-gathered pairs are
// scatter-added rank by rank into an fp64 buffer (:137-139), then / W and the
// momentum update (:145-146), which also clears the buffer.
// ---------------------------------------------------------------------------

__device__ __forceinline__ unsigned long long tk_key(double x) {
  return (unsigned long long)__double_as_longlong(fabs(x));
}

__global__ void k_topk_init(TkLayer* __restrict__ tl, TkState* __restrict__ st, unsigned* __restrict__ hist,
                            int L) {
  PDL_ENTRY();
  for (int l = blockIdx.x; l < L; l += gridDim.x) {
    if (threadIdx.x == 0) {
      st[l].prefix = 0ull;
      st[l].mask = 0ull;
      st[l].k_rem = tl[l].k;
      st[l].done = 0;
    }
    hist[(long long)l * 256 + threadIdx.x] = 0u;
  }
}

// ACC: fold grad + wd * params into the residual first (pass 0)
template <bool ACC>
__global__ void __launch_bounds__(kThreads) k_topk_hist(const TkTile* __restrict__ tiles, const TkLayer* __restrict__ tl,
                                                        const TkState* __restrict__ st, unsigned* __restrict__ hist,
                                                        double* __restrict__ res, const float* __restrict__ g,
                                                        const float* __restrict__ p, double wd, int shift) {
  PDL_ENTRY();
  __shared__ unsigned sh[256];
  const TkTile t = tiles[blockIdx.x];
  const TkState s = st[t.layer];
  if (!ACC && s.done) return;
  sh[threadIdx.x] = 0u;
  __syncthreads();
  const long long off = tl[t.layer].off;
  for (long long e = t.begin + threadIdx.x; e < t.end; e += kThreads) {
    double a;
    if (ACC) {
      a = __dadd_rn(res[off + e], __dadd_rn((double)g[off + e], __dmul_rn(wd, (double)p[off + e])));
      res[off + e] = a;
    } else {
      a = res[off + e];
    }
    const unsigned long long k = tk_key(a);
    if ((k & s.mask) == s.prefix) atomicAdd(&sh[(k >> shift) & 255u], 1u);
  }
  __syncthreads();
  const unsigned c = sh[threadIdx.x];
  if (c) atomicAdd(&hist[(long long)t.layer * 256 + threadIdx.x], c);
}

// one CTA (256 threads) per layer: the bin holding the k_rem-th largest key
__global__ void __launch_bounds__(256) k_topk_resolve(TkState* __restrict__ st, unsigned* __restrict__ hist,
                                                      int shift) {
  PDL_ENTRY();
  __shared__ long long suf[256];
  __shared__ int best;
  const int l = blockIdx.x, b = threadIdx.x;
  TkState s = st[l];
  unsigned* h = hist + (long long)l * 256;
  const long long c = h[b];
  h[b] = 0u;
  if (s.done) return;
  suf[b] = c;
  if (b == 0) best = -1;
  __syncthreads();
  for (int d = 1; d < 256; d <<= 1) {  // suffix sums: suf[b] = sum_{b' >= b} hist[b']
    const long long add = b + d < 256 ? suf[b + d] : 0;
    __syncthreads();
    suf[b] += add;
    __syncthreads();
  }
  if (suf[b] >= s.k_rem && (b == 255 || suf[b + 1] < s.k_rem)) best = b;
  __syncthreads();
  if (b == 0 && best >= 0) {
    const long long above = best == 255 ? 0 : suf[best + 1];
    s.k_rem -= above;
    s.prefix |= (unsigned long long)best << shift;
    s.mask |= 255ull << shift;
    s.done = (suf[best] - above == s.k_rem) ? 1 : 0;
    st[l] = s;
  }
}

__device__ __forceinline__ void tk_class(unsigned long long k, const TkState& s, int& gt, int& eq) {
  const unsigned long long m = k & s.mask;
  gt = m > s.prefix;
  eq = m == s.prefix;
}

__global__ void __launch_bounds__(kThreads) k_topk_count(const TkTile* __restrict__ tiles, const TkLayer* __restrict__ tl,
                                                         const TkState* __restrict__ st, const double* __restrict__ res,
                                                         int2* __restrict__ cnt) {
  PDL_ENTRY();
  const TkTile t = tiles[blockIdx.x];
  const TkState s = st[t.layer];
  const long long off = tl[t.layer].off;
  int gt = 0, eq = 0;
  for (long long e = t.begin + threadIdx.x; e < t.end; e += kThreads) {
    int a, b;
    tk_class(tk_key(res[off + e]), s, a, b);
    gt += a;
    eq += b;
  }
  for (int o = 16; o > 0; o >>= 1) {
    gt += __shfl_xor_sync(kFull, gt, o);
    eq += __shfl_xor_sync(kFull, eq, o);
  }
  __shared__ int sg[kThreads / 32], se[kThreads / 32];
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = gt;
    se[threadIdx.x >> 5] = eq;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0, b = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      a += sg[w];
      b += se[w];
    }
    cnt[blockIdx.x] = make_int2(a, b);
  }
}

// one thread per layer: exclusive (ties before, output before) per tile, in tile order
__global__ void k_topk_scan(const TkLayer* __restrict__ tl, const TkState* __restrict__ st,
                            const int2* __restrict__ cnt, int2* __restrict__ base, int L) {
  PDL_ENTRY();
  const int l = blockIdx.x * blockDim.x + threadIdx.x;
  if (l >= L) return;
  const long long k_rem = st[l].k_rem;
  long long eq_before = 0, out_before = 0;
  for (int i = tl[l].tile0; i < tl[l].tile0 + tl[l].ntiles; ++i) {
    const int2 c = cnt[i];
    base[i] = make_int2((int)eq_before, (int)out_before);
    const long long take = std::min<long long>(std::max<long long>(k_rem - eq_before, 0), c.y);
    eq_before += c.y;
    out_before += c.x + take;
  }
}

__global__ void __launch_bounds__(kThreads) k_topk_write(const TkTile* __restrict__ tiles, const TkLayer* __restrict__ tl,
                                                         const TkState* __restrict__ st, const int2* __restrict__ base,
                                                         double* __restrict__ res, float* __restrict__ vals,
                                                         int* __restrict__ idx) {
  PDL_ENTRY();
  __shared__ int wsum[kThreads / 32];
  __shared__ int carry;
  const TkTile t = tiles[blockIdx.x];
  const TkState s = st[t.layer];
  const TkLayer ly = tl[t.layer];
  const int2 b0 = base[blockIdx.x];
  int eq_run = b0.x, out_run = b0.y;  // block-uniform running totals
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long e0 = t.begin; e0 < t.end; e0 += kThreads) {
    const long long e = e0 + threadIdx.x;
    int gt = 0, eq = 0;
    double a = 0.0;
    if (e < t.end) {
      a = res[ly.off + e];
      tk_class(tk_key(a), s, gt, eq);
    }
    // inclusive scan of (eq << 16 | gt) over the block (<= 256 each: no carry between halves)
    int x = (eq << 16) | gt;
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(kFull, x, o);
      if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    int wbase = 0;
    for (int j = 0; j < w; ++j) wbase += wsum[j];
    x += wbase;
    const int eq_incl = x >> 16, gt_incl = x & 0xffff;
    const int eq_rank = eq_run + eq_incl - eq;  // ties before this element in the layer
    const int take_eq = eq && eq_rank < s.k_rem;
    // output slot: gt before + ties taken before (ties before capped at k_rem)
    const long long ties_taken_before = std::min<long long>(std::max<long long>(s.k_rem - eq_run, 0),
                                                            (long long)(eq_incl - eq));
    if (gt || take_eq) {
      const long long pos = (long long)out_run + (gt_incl - gt) + ties_taken_before;
      vals[ly.koff + pos] = (float)a;
      idx[ly.koff + pos] = (int)e;
      res[ly.off + e] = __dsub_rn(a, a);  // flat - kept (:144)
    }
    if (threadIdx.x == kThreads - 1) carry = x;
    __syncthreads();
    const int tot = carry;
    const int eq_tot = tot >> 16, gt_tot = tot & 0xffff;
    const long long taken = std::min<long long>(std::max<long long>(s.k_rem - eq_run, 0), (long long)eq_tot);
    out_run += gt_tot + (int)taken;
    eq_run += eq_tot;
    __syncthreads();
  }
}

// dense[off[layer] + idx] += val for one rank's pairs (indices unique within a rank)
__global__ void __launch_bounds__(kThreads) k_topk_scatter(const TkLayer* __restrict__ tl, int L,
                                                           const float* __restrict__ vals, const int* __restrict__ idx,
                                                           long long ktotal, double* __restrict__ dense) {
  PDL_ENTRY();
  for (long long j = blockIdx.x * (long long)kThreads + threadIdx.x; j < ktotal; j += (long long)gridDim.x * kThreads) {
    int lo = 0, hi = L - 1;  // last layer with koff <= j
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (tl[mid].koff <= j) lo = mid; else hi = mid - 1;
    }
    const long long i = tl[lo].off + idx[j];
    dense[i] = __dadd_rn(dense[i], (double)vals[j]);
  }
}

__global__ void __launch_bounds__(kThreads) k_topk_apply(double* __restrict__ dense, double div, float* __restrict__ p,
                                                         float* __restrict__ v, double lr, double mom, int first,
                                                         long long n) {
  PDL_ENTRY();
  for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
    const double avg = __ddiv_rn(dense[i], div);
    dense[i] = 0.0;
    float pp = p[i], vv = first ? 0.f : v[i];
    dense_upd(avg, pp, vv, lr, mom, first);
    p[i] = pp;
    v[i] = vv;
  }
}

int launch_topk_select(const TkTile* tiles, int n_tiles, const TkLayer* tl, int L, TkState* st, unsigned* hist,
                       int2* cnt, int2* base, double* res, const float* g, const float* p, double wd, float* vals,
                       int* idx, cudaStream_t stq) {
  if (L <= 0 || n_tiles <= 0) return 0;
  int launches = 0;
  launch_pdl(k_topk_init, std::min(L, 148 * 4), 256, 0, stq, const_cast<TkLayer*>(tl), st, hist, L);
  ++launches;
  for (int pass = 0; pass < 8; ++pass) {
    const int shift = 56 - 8 * pass;
    if (pass == 0)
      launch_pdl(k_topk_hist<true>, n_tiles, kThreads, 0, stq, tiles, tl, (const TkState*)st, hist, res, g, p, wd, shift);
    else
      launch_pdl(k_topk_hist<false>, n_tiles, kThreads, 0, stq, tiles, tl, (const TkState*)st, hist, res, g, p, wd,
                 shift);
    launch_pdl(k_topk_resolve, L, 256, 0, stq, st, hist, shift);
    launches += 2;
  }
  launch_pdl(k_topk_count, n_tiles, kThreads, 0, stq, tiles, tl, (const TkState*)st, (const double*)res, cnt);
  launch_pdl(k_topk_scan, (L + 127) / 128, 128, 0, stq, tl, (const TkState*)st, (const int2*)cnt, base, L);
  launch_pdl(k_topk_write, n_tiles, kThreads, 0, stq, tiles, tl, (const TkState*)st, (const int2*)base, res, vals, idx);
  return launches + 3;
}

void launch_topk_scatter(const TkLayer* tl, int L, const float* vals, const int* idx, long long ktotal, double* dense,
                         cudaStream_t st) {
  if (ktotal <= 0) return;
  const int grid = (int)std::min<long long>((ktotal + kThreads - 1) / kThreads, 148LL * 8);
  launch_pdl(k_topk_scatter, grid, kThreads, 0, st, tl, L, vals, idx, ktotal, dense);
}

void launch_topk_apply(double* dense, double div, float* p, float* v, double lr, double mom, int first, long long n,
                       cudaStream_t st) {
  if (n <= 0) return;
  launch_pdl(k_topk_apply, dense_grid(n), kThreads, 0, st, dense, div, p, v, lr, mom, first, n);
}
}  // namespace hsx

extern "C" int hsx_set_l2_hints(int32_t on) {
#ifdef HSX_NO_L2_HINTS
  return on ? 1 : 0;  // built without hints
#else
  return on ? 0 : 1;  // built with hints (a build choice: -DHSX_NO_L2_HINTS)
#endif
}
