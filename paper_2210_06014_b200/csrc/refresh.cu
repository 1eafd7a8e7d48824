// K2  C^(u) = A^(u) B^(u): refresh_dot_mode (_ckern.pyx:21-33 / _pykern.py:16-26) with the
// divergence guard of train.py:101-110 fused into the same pass over A.
//
// HBM-bound (8 flop/B at fp32 for J = R = 32): each warp streams a contiguous 32-row tile of A
// through shared memory with coalesced 128-bit loads, computes the 32 x R outputs with the
// reference's sequential-j accumulation order, and writes C back through shared memory as one
// contiguous, coalesced store.
#include <string.h>
#include <stdlib.h>

#include <cuda.h>
#include <cudaTypedefs.h>

#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int WARPS = 4;
constexpr int TILE = 32;  // rows per warp

struct Dsts {
  float *p[FT_MAX_PEERS];
  int n;
};

__global__ void __launch_bounds__(WARPS * 32)
    refresh_kernel(int64_t I, int J, int R, const float *__restrict__ A,
                   const float *__restrict__ Bt, Dsts dst, uint32_t *guard) {
  __shared__ float bts[FT_MAX_RANK][FT_MAX_RANK + 1];
  __shared__ float tile[WARPS][TILE][FT_MAX_RANK + 1];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int k = threadIdx.x; k < R * J; k += blockDim.x) bts[k / J][k % J] = Bt[k];
  __syncthreads();
  const int64_t row0 = ((int64_t)blockIdx.x * WARPS + w) * TILE;
  if (row0 >= I) return;
  const int rows = (int)(I - row0 < TILE ? I - row0 : TILE);
  const int nA = rows * J;
  const float *src = A + row0 * J;
  uint32_t gmax = 0;
  for (int k = lane; k < nA; k += 32) {
    float v = __ldcs(src + k);
    gmax = max(gmax, abs_bits(v));
    tile[w][k / J][k % J] = v;
  }
  if (guard) guard_max(guard, gmax);
  __syncwarp();
  float out[FT_MAX_RANK];
  if (lane < rows) {
    float a[FT_MAX_RANK];
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j) a[j] = j < J ? tile[w][lane][j] : 0.f;
#pragma unroll
    for (int r = 0; r < FT_MAX_RANK; ++r) {
      float s = 0.f;
      if (r < R) {
        // sequential j, as the reference (padded j >= J contribute exact zeros at the end)
#pragma unroll
        for (int j = 0; j < FT_MAX_RANK; ++j)
          if (j < J) s = __fmaf_rn(a[j], bts[r][j], s);
      }
      out[r] = s;
    }
  }
  __syncwarp();
  if (lane < rows) {
#pragma unroll
    for (int r = 0; r < FT_MAX_RANK; ++r)
      if (r < R) tile[w][lane][r] = out[r];
  }
  __syncwarp();
  // the tile goes to every destination: the local C_u and, for the fused refresh + all-gather,
  // each peer rank's C_u through its CUDA-IPC-mapped pointer (NVLink stores on a multi-GPU node)
  const int nC = rows * R;
  for (int d = 0; d < dst.n; ++d) {
    float *out = dst.p[d] + row0 * R;
    for (int k = lane; k < nC; k += 32) __stcs(out + k, tile[w][k / R][k % R]);
  }
}

// ---- K2 on the 5th-generation tensor cores (tcgen05, kind::tf32) ----------------------------
// C (I x R) = A (I x J) * Bt^T: M = 128 rows of A per tile, N = R, K = J (zero-padded to 32).
// Operands in shared memory, K-major with the 128-byte swizzle (one 128-B row of A per tile row:
// 16-B chunk c of row r at c ^ (r & 7)); accumulator in TMEM (R fp32 columns x 128 lanes).
// 3xTF32 (A_lo Bt_hi + A_hi Bt_lo + A_hi Bt_hi, truncation split as in K3b) keeps fp32
// accuracy.  Per tile: the 128 threads each load one row of A (guard max fused), split it into
// the hi / lo tiles; one elected thread issues 3 x K/8 tcgen05.mma and commits to an mbarrier;
// each warp reads its 32 TMEM lanes (tcgen05.ld 32x32b) and stores its rows of C to every
// destination.  Persistent grid, one tile in flight per CTA, several CTAs per SM.
namespace tc {
constexpr int M = 128;
constexpr int TILE_BYTES = M * 128;   // 128 rows x 32 fp32
constexpr int B_BYTES = 64 * 128;     // 64 rows (P or Q) x 32 fp32
constexpr size_t SMEM = 2 * TILE_BYTES + 2 * B_BYTES + 1024 + 64;  // + alignment slack, barrier

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xffffe000u; }
// shared-memory matrix descriptor, K-major, 128-B swizzle, 8-row groups 1024 B apart
__device__ __forceinline__ uint64_t sw128_desc(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);        // start address
  d |= (uint64_t)1 << 16;                        // leading byte offset (unused for SW128 K-major)
  d |= (uint64_t)(1024 >> 4) << 32;              // stride byte offset: next 8-row group
  d |= (uint64_t)1 << 46;                        // descriptor version (sm_100)
  d |= (uint64_t)2 << 61;                        // SWIZZLE_128B
  return d;
}
__device__ __forceinline__ void mma_tf32_tc(uint32_t tmem_d, uint64_t da, uint64_t db,
                                            uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(accumulate));
}
}  // namespace tc

__global__ void __launch_bounds__(128) refresh_tc_kernel(int64_t I, int J, int R,
                                                         const float *__restrict__ A,
                                                         const float *__restrict__ Bt, Dsts dst,
                                                         uint32_t *guard) {
  using namespace tc;
  extern __shared__ __align__(1024) uint8_t tc_smem[];
  // 1024-B aligned operand tiles (the 128-B swizzle pattern repeats every 8 rows = 1024 B)
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(tc_smem) + 1023) & ~(uintptr_t)1023);
  uint8_t *a_hi = base, *a_lo = base + TILE_BYTES;
  uint8_t *b_hi = base + 2 * TILE_BYTES, *b_lo = b_hi + B_BYTES;
  uint64_t *bar = reinterpret_cast<uint64_t *>(b_lo + B_BYTES);
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 1);
  const int tid = threadIdx.x, w = tid >> 5;

  // Bt (R x J) -> the 64-row B operands P = [Bt_hi ; Bt_lo] and Q = [Bt_hi ; 0] (row r = output
  // column, zero-padded to 32 rows x 32 k), so that D[:, 0:32] = A_hi Bt_hi + A_lo Bt_hi and
  // D[:, 32:64] = A_hi Bt_lo: 3xTF32 in 2 x J/8 MMAs at N = 64 instead of 3 x J/8 at N = 32
  // (an N = 64 tcgen05.mma costs about what an N = 32 one does: tools/umma_probe.cu)
  for (int e = tid; e < 32 * 8; e += 128) {
    const int r = e >> 3, c = e & 7;
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int j = 4 * c + t;
      v[t] = (r < R && j < J) ? __ldg(Bt + r * J + j) : 0.f;
    }
    const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
    uint4 h, l;
    h.x = hi_bits(v[0]), h.y = hi_bits(v[1]), h.z = hi_bits(v[2]), h.w = hi_bits(v[3]);
    l.x = __float_as_uint(v[0] - __uint_as_float(h.x));
    l.y = __float_as_uint(v[1] - __uint_as_float(h.y));
    l.z = __float_as_uint(v[2] - __uint_as_float(h.z));
    l.w = __float_as_uint(v[3] - __uint_as_float(h.w));
    *reinterpret_cast<uint4 *>(b_hi + off) = h;                 // P rows 0-31
    *reinterpret_cast<uint4 *>(b_hi + 32 * 128 + off) = l;      // P rows 32-63
    *reinterpret_cast<uint4 *>(b_lo + off) = h;                 // Q rows 0-31
    *reinterpret_cast<uint4 *>(b_lo + 32 * 128 + off) = make_uint4(0, 0, 0, 0);
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;\n" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  // kind::tf32, D fp32, A / B tf32 K-major, N = 64 (P / Q), M = 128
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const int ksteps = (J + 7) >> 3;
  uint32_t phase = 0, gmax = 0;
  const int64_t ntiles = (I + M - 1) / M;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t row = tile * M + tid;
    {  // this thread's row of A -> hi / lo (swizzled), guard max
      float v[32];
      if (row < I) {
        const float *ar = A + row * J;
        if (J == 32) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 q = __ldcs(reinterpret_cast<const float4 *>(ar) + c);
            v[4 * c] = q.x, v[4 * c + 1] = q.y, v[4 * c + 2] = q.z, v[4 * c + 3] = q.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) v[j] = j < J ? __ldcs(ar + j) : 0.f;
        }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) v[j] = 0.f;
      }
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const uint32_t off = tid * 128 + ((c ^ (tid & 7)) << 4);
        uint4 h, l;
        h.x = hi_bits(v[4 * c]), h.y = hi_bits(v[4 * c + 1]);
        h.z = hi_bits(v[4 * c + 2]), h.w = hi_bits(v[4 * c + 3]);
        l.x = __float_as_uint(v[4 * c] - __uint_as_float(h.x));
        l.y = __float_as_uint(v[4 * c + 1] - __uint_as_float(h.y));
        l.z = __float_as_uint(v[4 * c + 2] - __uint_as_float(h.z));
        l.w = __float_as_uint(v[4 * c + 3] - __uint_as_float(h.w));
        *reinterpret_cast<uint4 *>(a_hi + off) = h;
        *reinterpret_cast<uint4 *>(a_lo + off) = l;
#pragma unroll
        for (int t = 0; t < 4; ++t) gmax = max(gmax, abs_bits(v[4 * c + t]));
      }
    }
    // generic-proxy smem writes -> visible to the tensor core (async proxy)
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
      const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
      uint32_t acc = 0;
      for (int k = 0; k < ksteps; ++k) {  // K = 8 tf32 = 32 B per step inside the 128-B row
        mma_tf32_tc(tmem, sw128_desc(ah + 32 * k), sw128_desc(bh + 32 * k), idesc, acc);
        acc = 1;
      }
      for (int k = 0; k < ksteps; ++k)
        mma_tf32_tc(tmem, sw128_desc(al + 32 * k), sw128_desc(bl + 32 * k), idesc, 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       smem_u32(bar))
                   : "memory");
    }
    // wait for the accumulator
    asm volatile(
        "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase)
        : "memory");
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // TMEM lanes 32w..32w+31 = rows of this warp; columns 0-31 + 32-63 = C[row][0..31]
    uint32_t d[32], d2[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
          "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
          "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]),
          "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]),
          "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
        : "r"(tmem + ((uint32_t)(32 * w) << 16)));
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
        "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
        : "=r"(d2[0]), "=r"(d2[1]), "=r"(d2[2]), "=r"(d2[3]), "=r"(d2[4]), "=r"(d2[5]), "=r"(d2[6]),
          "=r"(d2[7]), "=r"(d2[8]), "=r"(d2[9]), "=r"(d2[10]), "=r"(d2[11]), "=r"(d2[12]), "=r"(d2[13]),
          "=r"(d2[14]), "=r"(d2[15]), "=r"(d2[16]), "=r"(d2[17]), "=r"(d2[18]), "=r"(d2[19]),
          "=r"(d2[20]), "=r"(d2[21]), "=r"(d2[22]), "=r"(d2[23]), "=r"(d2[24]), "=r"(d2[25]),
          "=r"(d2[26]), "=r"(d2[27]), "=r"(d2[28]), "=r"(d2[29]), "=r"(d2[30]), "=r"(d2[31])
        : "r"(tmem + ((uint32_t)(32 * w) << 16) + 32));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int r = 0; r < 32; ++r) d[r] = __float_as_uint(__uint_as_float(d[r]) + __uint_as_float(d2[r]));
    if (row < I) {
      for (int q = 0; q < dst.n; ++q) {
        float *out = dst.p[q] + row * R;
        if (R == 32) {
#pragma unroll
          for (int c = 0; c < 8; ++c)
            __stcs(reinterpret_cast<float4 *>(out) + c,
                   make_float4(__uint_as_float(d[4 * c]), __uint_as_float(d[4 * c + 1]),
                               __uint_as_float(d[4 * c + 2]), __uint_as_float(d[4 * c + 3])));
        } else {
#pragma unroll
          for (int r = 0; r < 32; ++r)
            if (r < R) __stcs(out + r, __uint_as_float(d[r]));
        }
      }
    }
    // TMEM reads and smem tile reads are done before the next tile overwrites them
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  if (guard) guard_max(guard, gmax);
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;\n" ::"r"(tmem));
}

// ---- K2, streaming form (J = R = 32): TMA bulk copies in and out, two tiles in the MMA ------
// A's 128-row tiles are contiguous 16 KB blocks: one elected thread keeps RING - 1 tile loads
// in flight (cp.async.bulk, completion on mbarriers).  Per tile the 128 threads read their row
// from the landed raw tile (chunks in a rotated order: conflict-free), fold the guard max, split
// it into one of two 128-B-swizzled hi / lo operand pairs, and one thread issues the tile's 8
// N = 64 MMAs into one of two TMEM accumulators.  The epilogue of tile t-1 (TMEM -> registers ->
// the warp's swizzled staging slab -> coalesced 512-B row-group stores to every destination,
// peers included) runs while the tensor core works on tile t, and the split of tile t+1 no
// longer waits for tile t's MMAs.
namespace tcs {
constexpr int TM = 128, TBYTES = TM * 128, RING = 6;
// raw ring (5 tile loads in flight: ~80 KB per SM against the HBM latency) + two hi / lo
// operand pairs (tile t + 1 is split while the tensor core works on tile t) + P, Q + the C
// staging tile (one 4 KB slab per warp): ~193 KB, one CTA per SM
constexpr size_t SMEM = 1024 + (size_t)RING * TBYTES + 4 * (size_t)TBYTES + 2 * (64 * 128) +
                        (size_t)TBYTES + 128;
__device__ __forceinline__ void bulk_load(uint32_t dst, const void *src, uint32_t bytes,
                                          uint32_t bar) {
  asm volatile(
      "mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(bar), "r"(bytes)
      : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void bulk_store(void *dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;\n" ::"l"(dst),
               "r"(src), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void wait_parity(uint32_t bar, uint32_t ph) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(bar),
      "r"(ph)
      : "memory");
}
__device__ __forceinline__ void ld_tmem32(uint32_t taddr, uint32_t (&d)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];\n"
      : "=r"(d[0]), "=r"(d[1]), "=r"(d[2]), "=r"(d[3]), "=r"(d[4]), "=r"(d[5]), "=r"(d[6]),
        "=r"(d[7]), "=r"(d[8]), "=r"(d[9]), "=r"(d[10]), "=r"(d[11]), "=r"(d[12]), "=r"(d[13]),
        "=r"(d[14]), "=r"(d[15]), "=r"(d[16]), "=r"(d[17]), "=r"(d[18]), "=r"(d[19]),
        "=r"(d[20]), "=r"(d[21]), "=r"(d[22]), "=r"(d[23]), "=r"(d[24]), "=r"(d[25]),
        "=r"(d[26]), "=r"(d[27]), "=r"(d[28]), "=r"(d[29]), "=r"(d[30]), "=r"(d[31])
      : "r"(taddr)
      : "memory");
}
}  // namespace tcs

__global__ void __launch_bounds__(128, 1) refresh_tcs_kernel(int64_t I, const float *__restrict__ A,
                                                             const float *__restrict__ Bt, Dsts dst,
                                                             uint32_t *guard) {
  using tc::smem_u32;
  using tc::hi_bits;
  using tc::sw128_desc;
  using tc::mma_tf32_tc;
  using namespace tcs;
  extern __shared__ __align__(1024) uint8_t tcs_smem[];
  const uint32_t sraw = smem_u32(tcs_smem), sbase = (sraw + 1023u) & ~1023u;
  uint8_t *gb = tcs_smem + (sbase - sraw);
  const uint32_t ring = sbase, aop = ring + RING * TBYTES;  // [2][a_hi, a_lo]
  const uint32_t bP = aop + 4 * TBYTES, bQ = bP + 64 * 128;
  const uint32_t stage = bQ + 64 * 128;                     // C staging, 4 KB per warp
  const uint32_t bars = stage + TBYTES;                     // ld[RING], mma[2], tmem slot
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gb + (bars - sbase) + 8 * (RING + 2));
  const int tid = threadIdx.x, w = tid >> 5;
  // B operands P = [Bt_hi ; Bt_lo], Q = [Bt_hi ; 0] (as refresh_tc_kernel)
  for (int e = tid; e < 32 * 8; e += 128) {
    const int r = e >> 3, c = e & 7;
    const float4 v = __ldg(reinterpret_cast<const float4 *>(Bt + r * 32) + c);
    const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
    uint4 h, l;
    h.x = hi_bits(v.x), h.y = hi_bits(v.y), h.z = hi_bits(v.z), h.w = hi_bits(v.w);
    l.x = __float_as_uint(v.x - __uint_as_float(h.x));
    l.y = __float_as_uint(v.y - __uint_as_float(h.y));
    l.z = __float_as_uint(v.z - __uint_as_float(h.z));
    l.w = __float_as_uint(v.w - __uint_as_float(h.w));
    *reinterpret_cast<uint4 *>(gb + (bP - sbase) + off) = h;
    *reinterpret_cast<uint4 *>(gb + (bP - sbase) + 32 * 128 + off) = l;
    *reinterpret_cast<uint4 *>(gb + (bQ - sbase) + off) = h;
    *reinterpret_cast<uint4 *>(gb + (bQ - sbase) + 32 * 128 + off) = make_uint4(0, 0, 0, 0);
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(
        smem_u32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int k = 0; k < RING + 2; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bars + 8 * k));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
  const int64_t ntiles = (I + TM - 1) / TM;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  auto tile_of = [&](int it) { return (int64_t)blockIdx.x + (int64_t)it * gridDim.x; };
  auto rows_of = [&](int64_t t) { return (int)(I - t * TM < TM ? I - t * TM : TM); };
  if (tid == 0)
    for (int it = 0; it < RING - 1 && it < nmine; ++it) {
      const int64_t t = tile_of(it);
      bulk_load(ring + it * TBYTES, A + t * TM * 32, (uint32_t)rows_of(t) * 128, bars + 8 * it);
    }
  uint32_t gmax = 0;
  auto epilogue = [&](int it) {  // tile it: TMEM -> C staging -> bulk stores
    const int64_t t = tile_of(it);
    const int rows = rows_of(t);
    wait_parity(bars + 8 * (RING + (it & 1)), (it >> 1) & 1);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    uint32_t d[32], d2[32];
    const uint32_t ta = tmem + ((uint32_t)(32 * w) << 16) + 64 * (it & 1);
    ld_tmem32(ta, d);
    ld_tmem32(ta + 32, d2);
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    // C rows through this warp's staging slab (128-B swizzle: conflict-free both ways), then
    // written back coalesced: four whole rows (512 contiguous bytes) per warp store
    const int lane = tid & 31;
    const uint32_t slab = stage + w * 4096;
#pragma unroll
    for (int c = 0; c < 8; ++c)
      asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(slab + lane * 128 + ((c ^ (lane & 7)) << 4)),
                   "f"(__uint_as_float(d[4 * c]) + __uint_as_float(d2[4 * c])),
                   "f"(__uint_as_float(d[4 * c + 1]) + __uint_as_float(d2[4 * c + 1])),
                   "f"(__uint_as_float(d[4 * c + 2]) + __uint_as_float(d2[4 * c + 2])),
                   "f"(__uint_as_float(d[4 * c + 3]) + __uint_as_float(d2[4 * c + 3])));
    __syncwarp();
    const int c = lane & 7;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int r = 4 * i + (lane >> 3), row = 32 * w + r;
      float4 v;
      asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                   : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                   : "r"(slab + r * 128 + ((c ^ (r & 7)) << 4)));
      if (row < rows) {
#pragma unroll
        for (int q = 0; q < dst.n && q < FT_MAX_PEERS; ++q)
          __stcs(reinterpret_cast<float4 *>(dst.p[q] + (t * TM + row) * 32) + c, v);
      }
    }
    __syncwarp();
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  };
  for (int it = 0; it < nmine; ++it) {
    const int64_t t = tile_of(it);
    const int rows = rows_of(t);
    if (tid == 0 && it + RING - 1 < nmine) {  // keep RING - 1 loads ahead
      const int nx = it + RING - 1;
      const int64_t tn = tile_of(nx);
      bulk_load(ring + (nx % RING) * TBYTES, A + tn * TM * 32, (uint32_t)rows_of(tn) * 128,
                bars + 8 * (nx % RING));
    }
    wait_parity(bars + 8 * (it % RING), (it / RING) & 1);
    // operand pair it & 1 was last read by tile it - 2's MMAs, whose completion epilogue(it - 2)
    // waited for in the previous iteration
    {  // this thread's row -> hi / lo (swizzled) into the operand tiles
      const uint32_t src = ring + (it % RING) * TBYTES + tid * 128;
      const uint32_t ah = aop + (it & 1) * 2 * TBYTES, al = ah + TBYTES;
      float4 v[8];  // all 8 chunks first (rotated order: conflict-free), then split and store
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = (q + tid) & 7;
        v[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        if (tid < rows)
          asm("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
              : "=f"(v[q].x), "=f"(v[q].y), "=f"(v[q].z), "=f"(v[q].w)
              : "r"(src + 16 * c));
      }
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const int c = (q + tid) & 7;
        gmax = max(gmax, max(max(abs_bits(v[q].x), abs_bits(v[q].y)),
                             max(abs_bits(v[q].z), abs_bits(v[q].w))));
        const uint32_t off = tid * 128 + ((c ^ (tid & 7)) << 4);
        const uint32_t hx = hi_bits(v[q].x), hy = hi_bits(v[q].y), hz = hi_bits(v[q].z),
                       hw = hi_bits(v[q].w);
        asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(ah + off), "r"(hx), "r"(hy),
                     "r"(hz), "r"(hw));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(al + off),
                     "f"(v[q].x - __uint_as_float(hx)), "f"(v[q].y - __uint_as_float(hy)),
                     "f"(v[q].z - __uint_as_float(hz)), "f"(v[q].w - __uint_as_float(hw)));
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();  // operand tiles written; raw stage it % RING free for its next load
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    if (tid == 0) {
      const uint32_t ah = aop + (it & 1) * 2 * TBYTES, al = ah + TBYTES;
      const uint32_t d = tmem + 64 * (it & 1);
      for (int k = 0; k < 4; ++k)
        mma_tf32_tc(d, sw128_desc(ah + 32 * k), sw128_desc(bP + 32 * k), idesc, k > 0);
      for (int k = 0; k < 4; ++k)
        mma_tf32_tc(d, sw128_desc(al + 32 * k), sw128_desc(bQ + 32 * k), idesc, 1);
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                       bars + 8 * (RING + (it & 1)))
                   : "memory");
    }
    if (it > 0) epilogue(it - 1);
  }
  if (nmine > 0) epilogue(nmine - 1);
  if (guard) guard_max(guard, gmax);
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tmem));
}

// ---- K2, TMA form (J = R = 32, one destination): warp-specialised, no CTA-wide barriers -------
// warp 0 lane 0 streams A tiles with 2D tensor loads (cp.async.bulk.tensor, 128-B swizzle: the
// landed tile IS the K-major SW128 MMA operand, ragged last tile zero-filled by the TMA unit);
// warp 1 lane 0 issues the MMAs; warps 2-5 (one TMEM lane quadrant each) read their 32 rows from
// the landed tile (conflict-free through the swizzle), fold the guard max and write A_lo =
// A - trunc_tf32(A) into TMEM, then run the epilogue of the previous tile (TMEM -> swizzled
// staging slab -> one 2D tensor store of 32 rows).  3xTF32 per tile: 4 x N = 64 MMAs of the raw
// tile (the tensor core truncates it to A_hi) against P = [Bt_hi ; Bt_lo] plus 4 x N = 32 MMAs
// of A_lo (TMEM) against Bt_hi: 8 MMAs, D[:, 0:32] + D[:, 32:64] = C.  Warps hand off through
// mbarriers only (full / empty per ring stage, lo_ready and acc_full per TMEM stage), so each
// warp runs at its own pace; ~104 KB of shared memory and 256 TMEM columns: two CTAs per SM.
namespace tma {
constexpr int TM = 128, TBYTES = TM * 128, RING = 4, THREADS = 192;
constexpr uint32_t TMEM_COLS = 256, LO = 128;  // D stages at 0 / 64, A_lo stages at 128 / 160
// ring + P + staging (4 worker warps x 2 x 4 KB) + barriers, 1024-B aligned
constexpr size_t SMEM = 1024 + (size_t)RING * TBYTES + 64 * 128 + 8 * 4096 + 256;
__device__ __forceinline__ void load2d(uint32_t dst, const CUtensorMap *m, int c0, int c1,
                                       uint32_t bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, "
      "{%2, %3}], [%4];\n" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(c0), "r"(c1), "r"(bar)
      : "memory");
}
__device__ __forceinline__ void store2d(const CUtensorMap *m, int c0, int c1, uint32_t src) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%1, %2}], [%3];\n" ::"l"(
                   reinterpret_cast<uint64_t>(m)),
               "r"(c0), "r"(c1), "r"(src)
               : "memory");
}
__device__ __forceinline__ void arrive(uint32_t bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(bar) : "memory");
}
__device__ __forceinline__ void commit(uint32_t bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(bar)
               : "memory");
}
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a_tmem, uint64_t db, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a_tmem), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void st_tmem32(uint32_t taddr, const uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
      "%14,%15,%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};\n" ::"r"(taddr),
      "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
      "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]), "r"(v[15]),
      "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]), "r"(v[22]),
      "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]), "r"(v[29]),
      "r"(v[30]), "r"(v[31])
      : "memory");
}
}  // namespace tma

__global__ void __launch_bounds__(tma::THREADS, 2)
    refresh_tma_kernel(int64_t I, const float *__restrict__ Bt,
                       const __grid_constant__ CUtensorMap tmA,
                       const __grid_constant__ CUtensorMap tmC, uint32_t *guard) {
  using tc::smem_u32;
  using tc::hi_bits;
  using tc::sw128_desc;
  using tc::mma_tf32_tc;
  using tcs::wait_parity;
  using tcs::ld_tmem32;
  using namespace tma;
  extern __shared__ __align__(1024) uint8_t tma_smem[];
  const uint32_t sraw = smem_u32(tma_smem), sbase = (sraw + 1023u) & ~1023u;
  uint8_t *gb = tma_smem + (sbase - sraw);
  const uint32_t ring = sbase, bP = ring + RING * TBYTES, stage = bP + 64 * 128;
  const uint32_t bars = stage + 8 * 4096;  // full[RING], empty[RING], lo_ready[2], acc_full[2]
  const uint32_t full = bars, empty = bars + 8 * RING, lo_ready = bars + 16 * RING,
                 acc_full = lo_ready + 16;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(gb + (bars - sbase) + 8 * (2 * RING + 4));
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  for (int e = tid; e < 32 * 8; e += THREADS) {  // P = [Bt_hi ; Bt_lo], SW128 K-major
    const int r = e >> 3, c = e & 7;
    const float4 v = __ldg(reinterpret_cast<const float4 *>(Bt + r * 32) + c);
    const uint32_t off = r * 128 + ((c ^ (r & 7)) << 4);
    uint4 h, l;
    h.x = hi_bits(v.x), h.y = hi_bits(v.y), h.z = hi_bits(v.z), h.w = hi_bits(v.w);
    l.x = __float_as_uint(v.x - __uint_as_float(h.x));
    l.y = __float_as_uint(v.y - __uint_as_float(h.y));
    l.z = __float_as_uint(v.z - __uint_as_float(h.z));
    l.w = __float_as_uint(v.w - __uint_as_float(h.w));
    *reinterpret_cast<uint4 *>(gb + (bP - sbase) + off) = h;
    *reinterpret_cast<uint4 *>(gb + (bP - sbase) + 32 * 128 + off) = l;
  }
  if (w == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int k = 0; k < 2 * RING; ++k)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(bars + 8 * k));
    for (int k = 0; k < 2; ++k) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;\n" ::"r"(lo_ready + 8 * k));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(acc_full + 8 * k));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("prefetch.tensormap [%0];\n" ::"l"(reinterpret_cast<uint64_t>(&tmA)) : "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;
  const int64_t ntiles = (I + TM - 1) / TM;
  const int nmine = ntiles > blockIdx.x ? (int)((ntiles - 1 - blockIdx.x) / gridDim.x) + 1 : 0;
  auto tile_of = [&](int it) { return (int64_t)blockIdx.x + (int64_t)it * gridDim.x; };
  if (w == 0) {
    if (lane == 0)
      for (int it = 0; it < nmine; ++it) {
        const int s = it % RING;
        if (it >= RING) wait_parity(empty + 8 * s, ((it / RING) - 1) & 1);
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(full + 8 * s),
                     "r"(TBYTES)
                     : "memory");
        load2d(ring + s * TBYTES, &tmA, 0, (int)(tile_of(it) * TM), full + 8 * s);
      }
  } else if (w == 1) {
    if (lane == 0) {
      const uint32_t i64 = (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
      const uint32_t i32 = (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
      for (int it = 0; it < nmine; ++it) {
        const int s = it % RING, b = it & 1;
        wait_parity(full + 8 * s, (it / RING) & 1);
        wait_parity(lo_ready + 8 * b, (it >> 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint32_t d = tmem + 64 * b, lo = tmem + LO + 32 * b, a = ring + s * TBYTES;
        for (int k = 0; k < 4; ++k) mma_tf32_tc(d, sw128_desc(a + 32 * k), sw128_desc(bP + 32 * k), i64, k > 0);
        for (int k = 0; k < 4; ++k) mma_ts(d, lo + 8 * k, sw128_desc(bP + 32 * k), i32, 1);
        commit(empty + 8 * s);
        commit(acc_full + 8 * b);
      }
    }
  } else {
    const int q = w & 3;  // TMEM lane quadrant = rows 32q .. 32q + 31 of every tile
    const uint32_t lanes = (uint32_t)(32 * q) << 16;
    uint32_t gmax = 0;
    auto epilogue = [&](int e) {
      const int b = e & 1;
      wait_parity(acc_full + 8 * b, (e >> 1) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      uint32_t d[32], d2[32];
      ld_tmem32(tmem + lanes + 64 * b, d);
      ld_tmem32(tmem + lanes + 64 * b + 32, d2);
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      const uint32_t slab = stage + q * 8192 + b * 4096;
      if (lane == 0 && e >= 2) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
      __syncwarp();
#pragma unroll
      for (int c = 0; c < 8; ++c)
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(slab + lane * 128 + ((c ^ (lane & 7)) << 4)),
                     "f"(__uint_as_float(d[4 * c]) + __uint_as_float(d2[4 * c])),
                     "f"(__uint_as_float(d[4 * c + 1]) + __uint_as_float(d2[4 * c + 1])),
                     "f"(__uint_as_float(d[4 * c + 2]) + __uint_as_float(d2[4 * c + 2])),
                     "f"(__uint_as_float(d[4 * c + 3]) + __uint_as_float(d2[4 * c + 3])));
      asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
      __syncwarp();
      const int64_t row0 = tile_of(e) * TM + 32 * q;
      if (lane == 0) {
        if (row0 < I) store2d(&tmC, 0, (int)row0, slab);
        asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
      }
    };
    for (int it = 0; it < nmine; ++it) {
      const int s = it % RING, b = it & 1;
      wait_parity(full + 8 * s, (it / RING) & 1);
      const uint32_t src = ring + s * TBYTES + (32 * q + lane) * 128;
      uint32_t lo[32];
#pragma unroll
      for (int c = 0; c < 8; ++c) {  // row 32q + lane: chunk c sits at c ^ (lane & 7)
        float4 v;
        asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
                     : "r"(src + ((c ^ (lane & 7)) << 4)));
        gmax = max(gmax, max(max(abs_bits(v.x), abs_bits(v.y)), max(abs_bits(v.z), abs_bits(v.w))));
        lo[4 * c] = __float_as_uint(v.x - __uint_as_float(hi_bits(v.x)));
        lo[4 * c + 1] = __float_as_uint(v.y - __uint_as_float(hi_bits(v.y)));
        lo[4 * c + 2] = __float_as_uint(v.z - __uint_as_float(hi_bits(v.z)));
        lo[4 * c + 3] = __float_as_uint(v.w - __uint_as_float(hi_bits(v.w)));
      }
      st_tmem32(tmem + lanes + LO + 32 * b, lo);
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) arrive(lo_ready + 8 * b);
      if (it > 0) epilogue(it - 1);
    }
    if (nmine > 0) epilogue(nmine - 1);
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
    if (guard) guard_max(guard, gmax);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (w == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "n"(TMEM_COLS));
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &p, 12000, cudaEnableDefault,
                                         &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      p = nullptr;
    return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }();
  return fn;
}
// rows x 32 fp32, 128-B rows, box of box_rows rows, 128-B swizzle; the last few encodings are
// cached (an epoch refreshes the same few matrices over and over)
bool rows32_map(CUtensorMap *m, const float *base, int64_t rows, int box_rows) {
  struct Entry {
    const float *base;
    int64_t rows;
    int box;
    CUtensorMap map;
  };
  static thread_local Entry cache[8] = {};
  static thread_local int next = 0;
  for (const Entry &e : cache)
    if (e.base == base && e.rows == rows && e.box == box_rows) {
      *m = e.map;
      return true;
    }
  const PFN_cuTensorMapEncodeTiled_v12000 enc = tensor_map_encoder();
  if (!enc || rows > INT32_MAX) return false;
  cuuint64_t dims[2] = {32, (cuuint64_t)rows};
  cuuint64_t strides[1] = {128};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  if (enc(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float *>(base), dims, strides, box, es,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cache[next] = Entry{base, rows, box_rows, *m};
  next = (next + 1) & 7;
  return true;
}

// tensor-core refresh unless FT_REFRESH=simt (the fp32 CUDA-core kernel above, which keeps the
// reference's sequential-j accumulation order); both need J, R <= 32
bool use_tc_refresh(int R) {
  static const bool simt = [] {
    const char *e = getenv("FT_REFRESH");
    return e && strcmp(e, "simt") == 0;
  }();
  return !simt && R >= 1;
}

int launch_refresh(int64_t I, int J, int R, const float *A, const float *Bt, const Dsts &d,
                   uint32_t *guard, cudaStream_t s) {
  if (use_tc_refresh(R) && J == 32 && R == 32 && d.n == 1 &&
      (reinterpret_cast<uintptr_t>(A) & 15) == 0 && (reinterpret_cast<uintptr_t>(d.p[0]) & 15) == 0) {
    CUtensorMap ma, mc;
    if (rows32_map(&ma, A, I, tma::TM) && rows32_map(&mc, d.p[0], I, 32)) {
      static bool set_t = false;
      if (!set_t) {
        cudaFuncSetAttribute(refresh_tma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)tma::SMEM);
        set_t = true;
      }
      int64_t g = (I + tma::TM - 1) / tma::TM;
      if (g > 2 * (int64_t)sm_count()) g = 2 * (int64_t)sm_count();
      refresh_tma_kernel<<<(unsigned)g, tma::THREADS, tma::SMEM, s>>>(I, Bt, ma, mc, guard);
      return check_launch("ft_refresh(tcgen05 TMA)");
    }
  }
  if (use_tc_refresh(R) && J == 32 && R == 32 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    static bool set_s = false;
    if (!set_s) {
      cudaFuncSetAttribute(refresh_tcs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tcs::SMEM);
      set_s = true;
    }
    bool aligned = true;
    for (int q = 0; q < d.n; ++q) aligned &= (reinterpret_cast<uintptr_t>(d.p[q]) & 15) == 0;
    if (aligned) {
      int64_t g = (I + tcs::TM - 1) / tcs::TM;
      if (g > sm_count()) g = sm_count();
      refresh_tcs_kernel<<<(unsigned)g, 128, tcs::SMEM, s>>>(I, A, Bt, d, guard);
      return check_launch("ft_refresh(tcgen05 streaming)");
    }
  }
  if (use_tc_refresh(R)) {
    static bool set = false;
    if (!set) {
      cudaFuncSetAttribute(refresh_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)tc::SMEM);
      set = true;
    }
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, refresh_tc_kernel, 128, tc::SMEM) !=
            cudaSuccess ||
        per_sm < 1)
      per_sm = 1;
    int64_t g = (I + tc::M - 1) / tc::M;
    const int64_t cap = (int64_t)sm_count() * per_sm;
    if (g > cap) g = cap;
    refresh_tc_kernel<<<(unsigned)g, 128, tc::SMEM, s>>>(I, J, R, A, Bt, d, guard);
    return check_launch("ft_refresh(tcgen05)");
  }
  const int64_t blocks = (I + WARPS * TILE - 1) / (WARPS * TILE);
  refresh_kernel<<<(unsigned)blocks, WARPS * 32, 0, s>>>(I, J, R, A, Bt, d, guard);
  return check_launch("ft_refresh");
}

}  // namespace
}  // namespace ft

extern "C" int ft_refresh(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt,
                          float *C, uint32_t *guard, void *stream) {
  using namespace ft;
  if (I < 0 || J < 1 || R < 1 || J > FT_MAX_RANK || R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ft_refresh: I=%lld J=%d R=%d outside kernel cover",
                (long long)I, J, R);
  if (I == 0) return FT_OK;
  if (!A || !Bt || !C) return fail(FT_ERR_ARG, "ft_refresh: null pointer");
  Dsts d{};
  d.p[0] = C;
  d.n = 1;
  return launch_refresh(I, J, R, A, Bt, d, guard, as_stream(stream));
}

extern "C" int ft_refresh_scatter(int64_t I, int32_t J, int32_t R, const float *A, const float *Bt,
                                  float *const *dsts, int32_t ndst, uint32_t *guard,
                                  void *stream) {
  using namespace ft;
  if (I < 0 || J < 1 || R < 1 || J > FT_MAX_RANK || R > FT_MAX_RANK)
    return fail(FT_ERR_UNSUPPORTED, "ft_refresh_scatter: I=%lld J=%d R=%d outside kernel cover",
                (long long)I, J, R);
  if (!dsts || ndst < 1 || ndst > FT_MAX_PEERS)
    return fail(FT_ERR_ARG, "ft_refresh_scatter: 1..%d destinations required", FT_MAX_PEERS);
  if (I == 0) return FT_OK;
  if (!A || !Bt) return fail(FT_ERR_ARG, "ft_refresh_scatter: null pointer");
  Dsts d{};
  for (int k = 0; k < ndst; ++k) {
    if (!dsts[k]) return fail(FT_ERR_ARG, "ft_refresh_scatter: null destination %d", k);
    d.p[k] = dsts[k];
  }
  d.n = ndst;
  return launch_refresh(I, J, R, A, Bt, d, guard, as_stream(stream));
}

// ---- stream-ordered peer barrier (multi-GPU fused refresh + all-gather) ---------------------
// Rank `rank` publishes `seq` into slot `rank` of every rank's flag array (CUDA-IPC mappings;
// NVLink stores on a multi-GPU node) after a system-scope fence that orders the preceding
// refresh kernel's peer stores, then waits until every slot of its own array holds >= seq.
// Queued on the compute stream, so the next sweep waits on the device for every rank's C_u
// block without a host synchronize + barrier.  A peer that never arrives ends in a trap after
// 20 s (an error, not a hang).
namespace ft {
namespace {
struct Flags {
  uint32_t *p[FT_MAX_PEERS];
};
__global__ void peer_barrier_kernel(uint32_t *local, Flags peers, int world, int rank,
                                    uint32_t seq) {
  if (threadIdx.x != 0) return;
  __threadfence_system();
  for (int q = 0; q < world; ++q)
    asm volatile("st.release.sys.global.u32 [%0], %1;\n" ::"l"(peers.p[q] + rank), "r"(seq)
                 : "memory");
  uint64_t t0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (int q = 0; q < world; ++q) {
    for (;;) {
      uint32_t v;
      asm volatile("ld.acquire.sys.global.u32 %0, [%1];\n" : "=r"(v) : "l"(local + q) : "memory");
      if ((int32_t)(v - seq) >= 0) break;
      uint64_t t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 20000000000ull) __trap();
      __nanosleep(64);
    }
  }
}
}  // namespace
}  // namespace ft

extern "C" int ft_peer_barrier(uint32_t *local_flags, uint32_t *const *peer_flags, int32_t world,
                               int32_t rank, uint32_t seq, void *stream) {
  using namespace ft;
  if (!local_flags || !peer_flags || world < 1 || world > FT_MAX_PEERS || rank < 0 ||
      rank >= world)
    return fail(FT_ERR_ARG, "ft_peer_barrier: bad arguments (world %d, rank %d)", world, rank);
  Flags f{};
  for (int q = 0; q < world; ++q) {
    if (!peer_flags[q]) return fail(FT_ERR_ARG, "ft_peer_barrier: null flags of rank %d", q);
    f.p[q] = peer_flags[q];
  }
  peer_barrier_kernel<<<1, 32, 0, as_stream(stream)>>>(local_flags, f, world, rank, seq);
  return check_launch("ft_peer_barrier");
}
