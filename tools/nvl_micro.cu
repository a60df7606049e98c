// NVLink read microbenchmarks (tools/nvl_micro.py drives them over torch symmetric
// memory on 2 GPUs): how fast a kernel can stream a peer's buffer depending on the
// load mechanism and the access pattern of K1's tiles.
//   copy_v4        grid-stride float4 loads (4 in flight per thread), contiguous
//   copy_ring      per-thread cp.async 16-B ring (depth 4), K1 tile pattern
//                  (tiles of 128 rows x 1 KB, rows `ld` floats apart)
//   copy_bulk      TMA 1-D bulk copies (cp.async.bulk + mbarrier) of 16 KB stages
//                  into shared memory, 4 stages in flight per CTA, contiguous
//   copy_bulk_rows the same with each stage = 16 row segments of 1 KB (K1 tile rows)
// Every kernel writes what it read to a local buffer (so the compiler keeps it).
#include <cstdint>
#include <cuda_runtime.h>

namespace {

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__global__ void k_copy_v4(const float4* __restrict__ src, float4* __restrict__ dst, long long n4) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i0 = blockIdx.x * (long long)blockDim.x + threadIdx.x; i0 < n4; i0 += 4 * stride) {
    float4 x[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (i < n4) x[u] = __ldcg(src + i);
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const long long i = i0 + u * stride;
      if (i < n4) dst[i] = x[u];
    }
  }
}

// K1-like: tile t = (row block rb, column chunk cc): rows [rb*128, +128) x quads
// [cc*64, +64); thread (jj = t & 63, ph = t >> 6) walks rows ph, ph+4, ...
__global__ void __launch_bounds__(256) k_copy_ring(const float* __restrict__ src, float* __restrict__ dst,
                                                   int rows, int ld, int tiles) {
  extern __shared__ float4 ring[];
  const int jj = threadIdx.x & 63, ph = threadIdx.x >> 6;
  const int chunks = ld / 256;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int rb = t / chunks, cc = t % chunks;
    const long long r0 = (long long)rb * 128 + ph;
    const int count = 32;
    const float* s = src + r0 * ld + cc * 256 + 4 * jj;
    float* d = dst + r0 * ld + cc * 256 + 4 * jj;
    const long long step = 4LL * ld;
    auto issue = [&](int slot, int i) {
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(ring + slot * 256 + threadIdx.x)),
                   "l"(s + i * step)
                   : "memory");
    };
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      issue(q, q);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int i = 0; i < count; ++i) {
      if (i + 3 < count) issue((i + 3) & 3, i + 3);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
      reinterpret_cast<float4*>(d + i * step)[0] = ring[(i & 3) * 256 + threadIdx.x];
    }
    __syncthreads();
  }
}

constexpr int kStages = 4;
constexpr int kStageBytes = 16384;

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
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

// rows_mode 0: stage s of chunk c = bytes [c * kStageBytes, +kStageBytes) of src
// rows_mode 1: stage = 16 row segments of 1 KB: tile rows r, r+1, ... (ld floats apart)
__global__ void __launch_bounds__(256) k_copy_bulk(const float* __restrict__ src, float* __restrict__ dst,
                                                   long long stages_total, int rows_mode, int ld) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[kStages];
  float4* buf = reinterpret_cast<float4*>(smem);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const int chunks = ld / 256;  // 1 KB column chunks per row (rows mode)
  auto src_of = [&](long long g, int seg) -> const float* {
    if (!rows_mode) return src + g * (kStageBytes / 4);
    // global stage g: 16 consecutive rows of one column chunk
    const long long rowgroup = g / chunks;
    const int cc = (int)(g % chunks);
    return src + (rowgroup * 16 + seg) * (long long)ld + cc * 256;
  };
  auto dst_of = [&](long long g, int seg) -> float* {
    if (!rows_mode) return dst + g * (kStageBytes / 4);
    const long long rowgroup = g / chunks;
    const int cc = (int)(g % chunks);
    return dst + (rowgroup * 16 + seg) * (long long)ld + cc * 256;
  };
  auto issue = [&](int s, long long g) {
    mbar_expect_tx(&full[s], kStageBytes);
    if (!rows_mode) {
      bulk_g2s(smem + s * kStageBytes, src_of(g, 0), kStageBytes, &full[s]);
    } else {
      for (int seg = 0; seg < 16; ++seg) bulk_g2s(smem + s * kStageBytes + seg * 1024, src_of(g, seg), 1024, &full[s]);
    }
  };
  // this CTA's stages: g = blockIdx.x + i * gridDim.x
  const long long my = (stages_total - blockIdx.x + gridDim.x - 1) / gridDim.x;
  if (threadIdx.x == 0)
    for (int s = 0; s < kStages && s < my; ++s) issue(s, blockIdx.x + (long long)s * gridDim.x);
  for (long long i = 0; i < my; ++i) {
    const int s = (int)(i % kStages);
    const unsigned phase = (unsigned)((i / kStages) & 1);
    mbar_wait(&full[s], phase);
    const long long g = blockIdx.x + i * gridDim.x;
    // 16 KB = 1024 float4: 4 per thread
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = threadIdx.x + u * 256;  // float4 index in the stage
      float4 v = buf[s * (kStageBytes / 16) + q];
      if (!rows_mode)
        reinterpret_cast<float4*>(dst_of(g, 0))[q] = v;
      else
        reinterpret_cast<float4*>(dst_of(g, q >> 6))[q & 63] = v;
    }
    __syncthreads();  // everyone is done with stage s
    if (threadIdx.x == 0 && i + kStages < my) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(s, blockIdx.x + (i + kStages) * gridDim.x);
    }
  }
}

// K1-like mix: out = remote + a + b + c over the K1 tile pattern (128 rows x 1 KB
// column chunks, rows `ld` floats apart). mode 0: all four streams through the
// per-thread cp.async ring (K1 today); mode 1: the remote stream through TMA bulk
// copies of 16-row stages (3 stages in flight), the local ones through the ring.
constexpr int kMixStage = 16 * 1024;  // 16 rows x 1 KB
__global__ void __launch_bounds__(256) k_mix(const float* __restrict__ rem, const float* __restrict__ la,
                                             const float* __restrict__ lb, const float* __restrict__ lc,
                                             float* __restrict__ out, int rows, int ld, int tiles, int mode) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[3];
  float4* ring = reinterpret_cast<float4*>(smem + (mode ? 3 * kMixStage : 0));  // [4 stages][4 streams][256]
  const int jj = threadIdx.x & 63, ph = threadIdx.x >> 6;
  const int chunks = ld / 256;
  if (mode && threadIdx.x == 0) {
    for (int s = 0; s < 3; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  unsigned phase_bits = 0;
  for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
    const int rb = t / chunks, cc = t % chunks;
    const long long row0 = (long long)rb * 128;
    const long long col = cc * 256;
    const long long r0 = row0 + ph;
    const long long step = 4LL * ld;
    const float* srcs[4] = {rem, la, lb, lc};
    const int nstr = mode ? 3 : 4;
    auto issue = [&](int slot, int i) {
      for (int q = 0; q < nstr; ++q) {
        const float* base = srcs[mode ? q + 1 : q];
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                         smem_u32(ring + (slot * 4 + q) * 256 + threadIdx.x)),
                     "l"(base + (r0 + i * 4) * ld + col + 4 * jj)
                     : "memory");
      }
    };
    // TMA stage k = rows row0 + 16k .. +16 of this column chunk
    auto tma = [&](int k) {
      const int s = k % 3;
      mbar_expect_tx(&full[s], kMixStage);
      for (int seg = 0; seg < 16; ++seg)
        bulk_g2s(smem + s * kMixStage + seg * 1024, rem + (row0 + 16 * k + seg) * ld + col, 1024, &full[s]);
    };
    if (mode && threadIdx.x == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int k = 0; k < 3; ++k) tma(k);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      issue(q, q);
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
    for (int i = 0; i < 32; ++i) {
      if (i + 3 < 32) issue((i + 3) & 3, i + 3);
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group 3;" ::: "memory");
      const int sl = i & 3;
      float4 r;
      if (mode) {
        const int k = i >> 2, s = k % 3;
        if ((i & 3) == 0) {
          mbar_wait(&full[s], (phase_bits >> s) & 1);
        }
        r = reinterpret_cast<const float4*>(smem + s * kMixStage)[((i & 3) * 4 + ph) * 64 + jj];
      } else {
        r = ring[(sl * 4 + 0) * 256 + threadIdx.x];
      }
      const float4 a = ring[(sl * 4 + (mode ? 0 : 1)) * 256 + threadIdx.x];
      const float4 b = ring[(sl * 4 + (mode ? 1 : 2)) * 256 + threadIdx.x];
      const float4 c = ring[(sl * 4 + (mode ? 2 : 3)) * 256 + threadIdx.x];
      reinterpret_cast<float4*>(out + (r0 + i * 4) * ld + col)[jj] =
          make_float4(r.x + a.x + b.x + c.x, r.y + a.y + b.y + c.y, r.z + a.z + b.z + c.z, r.w + a.w + b.w + c.w);
      if (mode && (i & 3) == 3) {
        const int k = i >> 2, s = k % 3;
        phase_bits ^= 1u << s;   // every thread tracks the parity of each stage
        __syncthreads();         // stage s consumed by everyone
        if (threadIdx.x == 0 && k + 3 < 8) {
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          tma(k + 3);
        }
      }
    }
    __syncthreads();
  }
}

}  // namespace

extern "C" {

int nvl_mix(const void* rem, const void* a, const void* b, const void* c, void* out, int rows, int ld, int grid,
            int mode, void* stream) {
  const int tiles = (rows / 128) * (ld / 256);
  const size_t smem = (size_t)(mode ? 3 * kMixStage : 0) + 4 * 4 * 256 * 16;
  cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_mix<<<grid, 256, smem, (cudaStream_t)stream>>>((const float*)rem, (const float*)a, (const float*)b,
                                                   (const float*)c, (float*)out, rows, ld, tiles, mode);
  return (int)cudaGetLastError();
}


int nvl_copy_v4(const void* src, void* dst, long long bytes, int grid, void* stream) {
  k_copy_v4<<<grid, 256, 0, (cudaStream_t)stream>>>((const float4*)src, (float4*)dst, bytes / 16);
  return (int)cudaGetLastError();
}

int nvl_copy_ring(const void* src, void* dst, int rows, int ld, int grid, void* stream) {
  const int tiles = (rows / 128) * (ld / 256);
  const size_t smem = 4 * 256 * 16;
  k_copy_ring<<<grid, 256, smem, (cudaStream_t)stream>>>((const float*)src, (float*)dst, rows, ld, tiles);
  return (int)cudaGetLastError();
}

int nvl_copy_bulk(const void* src, void* dst, long long stages, int rows_mode, int ld, int grid, void* stream) {
  const size_t smem = (size_t)kStages * kStageBytes;
  cudaFuncSetAttribute(k_copy_bulk, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  k_copy_bulk<<<grid, 256, smem, (cudaStream_t)stream>>>((const float*)src, (float*)dst, stages, rows_mode, ld);
  return (int)cudaGetLastError();
}

}  // extern "C"
