// K3c: the exact factor sweep with the J x R combine on the 5th-generation tensor cores
// (tcgen05, kind::tf32, A operand in TMEM) and ONE THREAD PER ROW for the serial chain.
//
// Reference semantics (factor_sweep, _ckern.pyx:132-199 / _pykern.py:69-137): for every leaf of
// row i of A_u in the serial order of the tree rooted at u+1,
//     cross = C_{u+1}[i_{u+1}] * ... * C_{u-1}[i_{u-1}]   (left to right),   v = Bt_u^T cross,
//     s = A_u[i] . v,   e = x - s,   A_u[i] <- A_u[i] - lr (reg A_u[i] - e v).
// The row-owner schedule of sweep.cu (one owner per row of the tree rooted at u, updates in the
// reference's order, every other operand frozen) is kept; what changes is who does what:
//   * a CTA owns 128 SLOTS; slot s walks its own stream of rows (rows q, q + 128 G, ... of the
//     tree, q = block + G s) one leaf per batch.  Slot s is TMEM lane s and consumer thread s:
//     the thread keeps its row in registers (32 fp32 + the Fast2Sum residue) and runs the chain
//     without a single shuffle;
//   * the per-leaf operands come from the SLOT LAYOUT (ft_tree_slot_fill): the tree's leaf
//     coordinates and values re-ordered [CTA][batch][slot], so every batch's metadata is one
//     coalesced 128-B line per warp and array (a per-thread walk of its own row would touch 32
//     lines per load instruction: tools/gather_probe.cu, 5x slower);
//   * gathers: cp.async, 8 lanes per 128-B C row (coalesced), into a GS-deep shared-memory ring,
//     swizzled so that thread s reads its own slot's rows conflict-free;
//   * thread s forms its cross row, splits it 3xTF32 (truncation hi + fp32 lo) and writes both
//     halves into TMEM with tcgen05.st (the A operand never touches shared memory again);
//   * one elected thread of the MMA warp issues D = A_lo Bt_hi + A_hi Bt_lo + A_hi Bt_hi
//     (M = 128 slots, N = 32 = J padded, K = R in steps of 8; Bt_u^T hi / lo in shared memory,
//     K-major, 128-B swizzle) and commits to an mbarrier; thread s reads v (its TMEM lane) with
//     tcgen05.ld and runs the step.  Two TMEM stages: the MMA of batch b overlaps the chain of
//     batch b-1 and the gathers of batches up to b+GS-1 are in flight.
// Requirements (checked by the dispatcher): 3 <= N <= 4, J <= 32, R <= 32 with R % 4 == 0, the
// slot layout present.
#include <stdlib.h>
#include <string.h>

#include <cub/cub.cuh>

#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int SLOTS = 128;
constexpr int CWARPS = 4;                    // consumer warps: warp w <-> TMEM lanes 32w..32w+31
constexpr int THREADS = (CWARPS + 1) * 32;   // + the MMA warp
constexpr int TCOLS = 96;                    // TMEM columns per stage: A_hi | A_lo | D
constexpr uint32_t ROW_START = 0x80000000u;  // slot_lc flag: first leaf of the slot's next row
constexpr int32_t PAD = -1;                  // slot_lc of a padding entry (slot stream ended)

__device__ __forceinline__ uint32_t su32(const void *p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t hi_bits(float x) { return __float_as_uint(x) & 0xffffe000u; }
__device__ __forceinline__ uint64_t sw128(uint32_t addr) {
  uint64_t d = 0;
  d |= (uint64_t)((addr & 0x3FFFF) >> 4);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}
__device__ __forceinline__ void mbar_init(uint64_t *b, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive(uint64_t *b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *b, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra WAIT_%=;\n}\n" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
}
__device__ __forceinline__ void cp16(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void tmem_st8(uint32_t taddr, const uint32_t (&r)[8]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7])
      : "memory");
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t d[32];
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
  asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(d[j]);
}
// D (tmem) [+]= A (tmem) * B (smem descriptor), kind::tf32
__device__ __forceinline__ void mma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc,
                                       uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ float2 f2fma(float2 a, float2 b, float2 c) {
  unsigned long long d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)),
        "l"(*reinterpret_cast<unsigned long long *>(&c)));
  return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 f2add(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 f2sub(float2 a, float2 b) {
  return f2add(a, make_float2(-b.x, -b.y));
}

struct TcParams {
  const int32_t *slot_lc;
  const int32_t *slot_pc;
  const float *slot_x;
  const int32_t *batch_ptr;
  const int32_t *row_coord;
  int64_t nrows;
  const float *Cpre[2];
  const float *Cleaf;
  float *A;
  const float *Bt;
  int J, R;
  float lr, reg;
};

template <int NPRE, int GS>
struct TcPlan {
  static constexpr int LEVELS = NPRE + 1;                 // gathered C rows per leaf
  static constexpr int STAGE = SLOTS * LEVELS * 128;      // bytes per gather stage
  static constexpr int B_BYTES = 32 * 128;                // Bt^T tile (N = 32 rows of 128 B)
  static constexpr int MS = 2 * GS;                       // metadata ring stages
  static constexpr int MWORDS = (NPRE + 2) * SLOTS;       // lc|flags, pc[NPRE], x per stage
  static constexpr int META = MS * MWORDS * 4;
  static constexpr size_t SMEM = 1024 + 2 * B_BYTES + (size_t)GS * STAGE + META + 64;
};

template <int NPRE, int GS, bool COMP>
__global__ void __launch_bounds__(THREADS, 1) factor_rows_tc_kernel(const TcParams p) {
  using P = TcPlan<NPRE, GS>;
  extern __shared__ __align__(1024) uint8_t smraw[];
  uint8_t *base = reinterpret_cast<uint8_t *>(
      (reinterpret_cast<uintptr_t>(smraw) + 1023) & ~(uintptr_t)1023);
  uint8_t *b_hi = base, *b_lo = base + P::B_BYTES;
  uint8_t *ring = base + 2 * P::B_BYTES;
  int32_t *meta = reinterpret_cast<int32_t *>(ring + (size_t)GS * P::STAGE);
  uint64_t *bar = reinterpret_cast<uint64_t *>(reinterpret_cast<uint8_t *>(meta) + P::META);
  uint64_t *a_ready = bar, *v_ready = bar + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(bar + 4);
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int J = p.J, R = p.R;

  // Bt_u^T (N = j rows, K = r) -> hi / lo, K-major, 128-B swizzle, zero padded to 32 x 32
  for (int e = tid; e < 32 * 8; e += THREADS) {
    const int j = e >> 3, c = e & 7;
    float v[4];
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const int r = 4 * c + t;
      v[t] = (j < J && r < R) ? __ldg(p.Bt + (int64_t)r * J + j) : 0.f;
    }
    const uint32_t off = j * 128 + ((c ^ (j & 7)) << 4);
    uint4 h, l;
    h.x = hi_bits(v[0]), h.y = hi_bits(v[1]), h.z = hi_bits(v[2]), h.w = hi_bits(v[3]);
    l.x = __float_as_uint(v[0] - __uint_as_float(h.x));
    l.y = __float_as_uint(v[1] - __uint_as_float(h.y));
    l.z = __float_as_uint(v[2] - __uint_as_float(h.z));
    l.w = __float_as_uint(v[3] - __uint_as_float(h.w));
    *reinterpret_cast<uint4 *>(b_hi + off) = h;
    *reinterpret_cast<uint4 *>(b_lo + off) = l;
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    mbar_init(a_ready, CWARPS);
    mbar_init(a_ready + 1, CWARPS);
    mbar_init(v_ready, 1);
    mbar_init(v_ready + 1, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B tiles -> tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t b0 = __ldg(p.batch_ptr + blockIdx.x);
  const int nb = __ldg(p.batch_ptr + blockIdx.x + 1) - (int)b0;

  if (w == CWARPS) {  // ---- MMA warp ----
    // kind::tf32, D fp32, A / B tf32 K-major, N = 32, M = 128
    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((32u >> 3) << 17) | ((128u >> 4) << 24);
    const int ksteps = (R + 7) >> 3;
    const uint32_t bh = su32(b_hi), bl = su32(b_lo);
    for (int b = 0; b < nb; ++b) {
      const int st = b & 1;
      mbar_wait(a_ready + st, (b >> 1) & 1);
      tc_fence_after();
      if (lane == 0) {
        const uint32_t ah = tmem + TCOLS * st, al = ah + 32, d = ah + 64;
        for (int k = 0; k < ksteps; ++k) {
          mma_ts(d, al + 8 * k, sw128(bh + 32 * k), idesc, k > 0);
          mma_ts(d, ah + 8 * k, sw128(bl + 32 * k), idesc, 1);
          mma_ts(d, ah + 8 * k, sw128(bh + 32 * k), idesc, 1);
        }
        asm volatile(
            "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                su32(v_ready + st))
            : "memory");
      }
      __syncwarp();
    }
  } else {  // ---- consumer warps: slot s = TMEM lane s = this thread ----
    const int s = tid;
    const uint32_t tlane = tmem + ((uint32_t)(32 * w) << 16);
    const int64_t gslots = (int64_t)gridDim.x * SLOTS;
    const float lr = p.lr, cdec = -p.lr * p.reg;
    const int gc = lane & 7, gs = lane >> 3;
    const bool gok = gc < (R >> 2);

    // Metadata of batch g (lc | flags, pc[NPRE], x of this lane's slot) -> meta ring stage
    // g % MS by 4-B cp.async, requested 2 GS - 1 batches ahead so that it has landed (its group
    // retired) before the gathers of batch g are issued: no load latency on the issue path.
    auto request_meta = [&](int g) {
      if (g < nb) {
        const int64_t bb = b0 + g;
        const uint32_t m0 = su32(meta + (g % P::MS) * P::MWORDS + s);
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(m0),
                     "l"(p.slot_lc + bb * SLOTS + s));
#pragma unroll
        for (int d = 0; d < NPRE; ++d)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(m0 + 4 * SLOTS * (1 + d)),
                       "l"(p.slot_pc + (bb * NPRE + d) * SLOTS + s));
        asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(m0 + 4 * SLOTS * (1 + NPRE)),
                     "l"(p.slot_x + bb * SLOTS + s));
      }
    };
    auto meta_lc = [&](int g) { return meta[(g % P::MS) * P::MWORDS + s]; };
    auto meta_x = [&](int g) { return meta[(g % P::MS) * P::MWORDS + (1 + NPRE) * SLOTS + s]; };
    // gathers of batch g into ring stage g % GS (cooperative: 8 lanes per 128-B row)
    auto issue = [&](int g) {
      if (g < nb) {
        const int lcf = meta_lc(g);
        int coord[NPRE + 1];
#pragma unroll
        for (int d = 0; d < NPRE; ++d)
          coord[d] = lcf == PAD ? -1 : meta[(g % P::MS) * P::MWORDS + (1 + d) * SLOTS + s];
        coord[NPRE] = lcf == PAD ? -1 : (int)((uint32_t)lcf & ~ROW_START);
        const uint32_t st0 = su32(ring + (size_t)(g % GS) * P::STAGE);
#pragma unroll
        for (int lv = 0; lv <= NPRE; ++lv) {
          const float *C = lv < NPRE ? p.Cpre[lv] : p.Cleaf;
#pragma unroll
          for (int it = 0; it < 8; ++it) {
            const int t = 4 * it + gs;  // slot (within the warp) this lane copies for
            const int cs = __shfl_sync(FULL, coord[lv], t);
            const int srow = 32 * w + t;
            if (gok && cs >= 0)
              cp16(st0 + (uint32_t)((lv * SLOTS + srow) * 128 + ((gc ^ (srow & 7)) << 4)),
                   C + (int64_t)cs * R + 4 * gc);
          }
        }
      }
    };

    float a[32], lo[32], na[32];
    int64_t row = (int64_t)blockIdx.x + (int64_t)gridDim.x * s;  // this slot's first row
    bool have = false;                                          // a holds a row
    int64_t cur_i = -1;
    // row coordinates run two rows ahead of the chain, the A row one row ahead, so a row
    // switch never waits on a dependent global load
    int ci1 = row < p.nrows ? __ldg(p.row_coord + row) : -1;      // coordinate of `row`
    int ci2 = row + gslots < p.nrows ? __ldg(p.row_coord + row + gslots) : -1;  // ... next
    auto load_row = [&](float (&dst)[32], int ci) {
      if (ci >= 0) {
        const float *ar = p.A + (int64_t)ci * J;
        if (J == 32) {
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            const float4 q = *reinterpret_cast<const float4 *>(ar + 4 * c);
            dst[4 * c] = q.x, dst[4 * c + 1] = q.y, dst[4 * c + 2] = q.z, dst[4 * c + 3] = q.w;
          }
        } else {
#pragma unroll
          for (int j = 0; j < 32; ++j) dst[j] = j < J ? ar[j] : 0.f;
        }
      }
    };
    auto store_row = [&]() {
      float *ar = p.A + cur_i * J;
      if (J == 32) {
#pragma unroll
        for (int c = 0; c < 8; ++c)
          *reinterpret_cast<float4 *>(ar + 4 * c) =
              make_float4(a[4 * c], a[4 * c + 1], a[4 * c + 2], a[4 * c + 3]);
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j < J) ar[j] = a[j];
      }
    };
#pragma unroll
    for (int j = 0; j < 32; ++j) a[j] = 0.f, lo[j] = 0.f, na[j] = 0.f;
    load_row(na, ci1);  // the first row's values, installed at its first leaf

    // the chain of batch b (its v is in TMEM stage b & 1)
    auto chain = [&](int b, int2 m) {
      const int st = b & 1;
      mbar_wait(v_ready + st, (b >> 1) & 1);
      tc_fence_after();
      float v[32];
      tmem_ld32(tlane + TCOLS * st + 64, v);
      if (m.x == PAD) return;
      if ((uint32_t)m.x & ROW_START) {
        if (have) {
          store_row();
          row += gslots;
          ci1 = ci2;
          ci2 = row + gslots < p.nrows ? __ldg(p.row_coord + row + gslots) : -1;
        }
        have = true;
        cur_i = ci1;
#pragma unroll
        for (int j = 0; j < 32; ++j) a[j] = na[j], lo[j] = 0.f;
        load_row(na, ci2);  // prefetch the slot's next row
      }
      const float x = __int_as_float(m.y);
      float2 s2a = make_float2(0.f, 0.f), s2b = make_float2(0.f, 0.f);
#pragma unroll
      for (int j = 0; j < 32; j += 4) {
        s2a = f2fma(make_float2(a[j], a[j + 1]), make_float2(v[j], v[j + 1]), s2a);
        s2b = f2fma(make_float2(a[j + 2], a[j + 3]), make_float2(v[j + 2], v[j + 3]), s2b);
      }
      const float dot = (s2a.x + s2a.y) + (s2b.x + s2b.y);
      const float e = x - dot;
      const float2 l2 = make_float2(lr * e, lr * e), c2 = make_float2(cdec, cdec);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 aj = make_float2(a[j], a[j + 1]), vj = make_float2(v[j], v[j + 1]);
        if (COMP) {
          const float2 d = f2fma(l2, vj, f2fma(c2, aj, make_float2(lo[j], lo[j + 1])));
          const float2 t = f2add(aj, d);
          const float2 r = f2sub(d, f2sub(t, aj));
          a[j] = t.x, a[j + 1] = t.y, lo[j] = r.x, lo[j + 1] = r.y;
        } else {
          const float2 t = f2fma(l2, vj, f2fma(c2, aj, aj));
          a[j] = t.x, a[j + 1] = t.y;
        }
      }
    };

    // prologue: metadata of batches 0 .. 2 GS - 2 (landed), gathers of batches 0 .. GS - 2
#pragma unroll 1
    for (int g = 0; g < 2 * GS - 1; ++g) request_meta(g);
    cp_commit();
    cp_wait<0>();
#pragma unroll 1
    for (int g = 0; g < GS - 1; ++g) {
      issue(g);
      cp_commit();
    }
    int2 mprev = make_int2(PAD, 0);  // (lc | flags, x) of the batch whose chain runs next
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      // one group per batch (empty past the end keeps the count uniform): the metadata of
      // batch b + 2 GS - 1 and the gathers of batch b + GS - 1, whose metadata retired with
      // the group of batch b - GS
      request_meta(b + 2 * GS - 1);
      issue(b + GS - 1);
      cp_commit();
      cp_wait<GS - 1>();  // this lane's copies of batch b have landed
      __syncwarp();       // ... and every lane's
      {  // cross of slot s -> 3xTF32 halves -> TMEM A stage (b & 1)
        const int2 mb = make_int2(meta_lc(b), meta_x(b));
        const int m0 = mb.x;
        const uint8_t *st0 = ring + (size_t)(b % GS) * P::STAGE;
        const uint32_t ah = tlane + TCOLS * (b & 1), al = ah + 32;
#pragma unroll
        for (int h = 0; h < 4; ++h) {  // 8 columns per TMEM store
          uint32_t hv[8], lv8[8];
#pragma unroll
          for (int q = 0; q < 2; ++q) {
            const int c = 2 * h + q;
            float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
            if (m0 != PAD && 4 * c < R) {
              x = *reinterpret_cast<const float4 *>(st0 + s * 128 + ((c ^ (s & 7)) << 4));
#pragma unroll
              for (int lv = 1; lv <= NPRE; ++lv) {
                const float4 y = *reinterpret_cast<const float4 *>(
                    st0 + (lv * SLOTS + s) * 128 + ((c ^ (s & 7)) << 4));
                x.x *= y.x, x.y *= y.y, x.z *= y.z, x.w *= y.w;
              }
            }
            const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              const uint32_t hb = hi_bits(xs[t]);
              hv[4 * q + t] = hb;
              lv8[4 * q + t] = __float_as_uint(xs[t] - __uint_as_float(hb));
            }
          }
          tmem_st8(ah + 8 * h, hv);
          tmem_st8(al + 8 * h, lv8);
        }
        asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
        tc_fence_before();
        __syncwarp();  // every lane's stores (and its reads of the ring stage) are done
        if (lane == 0) mbar_arrive(a_ready + (b & 1));
        if (b > 0) chain(b - 1, mprev);
        mprev = mb;
      }
    }
    if (nb > 0) chain(nb - 1, mprev);
    if (have) store_row();
    cp_wait<0>();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(tmem));
}

// ---- K1d: the slot layout ------------------------------------------------------------------
// Slot q = c + G s (CTA c, slot s) owns rows q, q + 128 G, q + 256 G, ... of the tree; its
// stream is their leaves in order.  slot_plan: per-CTA batch counts (the longest stream of its
// slots); slot_fill: entry [batch][s] of CTA c = the slot's stream position `batch`.
__global__ void slot_count_kernel(const int32_t *__restrict__ row_leaf_ptr, int64_t rows, int G,
                                  int32_t *__restrict__ nbatch) {
  const int c = blockIdx.x, s = threadIdx.x;
  const int64_t gsl = (int64_t)G * SLOTS;
  int64_t tot = 0;
  for (int64_t r = c + (int64_t)G * s; r < rows; r += gsl)
    tot += __ldg(row_leaf_ptr + r + 1) - __ldg(row_leaf_ptr + r);
  using BR = cub::BlockReduce<int64_t, SLOTS>;
  __shared__ typename BR::TempStorage ts;
  const int64_t mx = BR(ts).Reduce(tot, cub::Max());
  if (s == 0) nbatch[c] = (int32_t)mx;
}

__global__ void slot_scan_kernel(const int32_t *__restrict__ nbatch, int G, int32_t *batch_ptr) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int32_t acc = 0;
    for (int c = 0; c < G; ++c) {
      batch_ptr[c] = acc;
      acc += nbatch[c];
    }
    batch_ptr[G] = acc;
  }
}

__global__ void slot_fill_kernel(const int32_t *__restrict__ row_leaf_ptr, int64_t rows, int G,
                                 int npre, const int32_t *__restrict__ batch_ptr,
                                 const int32_t *__restrict__ leaf_coord,
                                 const int32_t *__restrict__ leaf_pc,
                                 const float *__restrict__ vals, int32_t *__restrict__ slot_lc,
                                 int32_t *__restrict__ slot_pc, float *__restrict__ slot_x) {
  const int c = blockIdx.x, s = threadIdx.x;
  const int64_t gsl = (int64_t)G * SLOTS;
  const int64_t b0 = batch_ptr[c];
  const int nb = batch_ptr[c + 1] - (int)b0;
  int64_t r = c + (int64_t)G * s;
  int64_t L = 0, Le = 0;
  bool start = false;
  if (r < rows) L = row_leaf_ptr[r], Le = row_leaf_ptr[r + 1], start = true;
  for (int b = 0; b < nb; ++b) {
    while (r < rows && L >= Le) {  // next non-empty row of the stream
      r += gsl;
      if (r < rows) L = row_leaf_ptr[r], Le = row_leaf_ptr[r + 1], start = true;
    }
    const int64_t e = (b0 + b) * SLOTS + s;
    if (r < rows) {
      slot_lc[e] = (int32_t)((uint32_t)leaf_coord[L] | (start ? ROW_START : 0u));
      for (int d = 0; d < npre; ++d) slot_pc[((b0 + b) * npre + d) * SLOTS + s] = leaf_pc[L * npre + d];
      slot_x[e] = vals[L];
      start = false;
      ++L;
    } else {
      slot_lc[e] = PAD;
      for (int d = 0; d < npre; ++d) slot_pc[((b0 + b) * npre + d) * SLOTS + s] = 0;
      slot_x[e] = 0.f;
    }
  }
}

bool tc_shape_ok(int N, int J, int R) {
  return N >= 3 && N <= 4 && J >= 1 && J <= 32 && R >= 4 && R <= 32 && R % 4 == 0;
}

// FT_FACTOR_TC=0 disables the tcgen05 factor sweep (the quadr / quadw kernels run instead)
bool tc_enabled() {
  static const bool on = [] {
    const char *e = getenv("FT_FACTOR_TC");
    return !(e && strcmp(e, "0") == 0);
  }();
  return on;
}

template <int NPRE, int GS>
int launch_tc_t(const TcParams &q, int G, bool comp, cudaStream_t s) {
  const size_t sm = TcPlan<NPRE, GS>::SMEM;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_tc_kernel<NPRE, GS, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(factor_rows_tc_kernel<NPRE, GS, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  if (comp)
    factor_rows_tc_kernel<NPRE, GS, true><<<G, THREADS, sm, s>>>(q);
  else
    factor_rows_tc_kernel<NPRE, GS, false><<<G, THREADS, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(tcgen05)");
}

}  // namespace

// rows the tcgen05 sweep needs to fill the GPU (one 128-slot CTA per SM); fewer long rows
// (Netflix mode 2) keep the warp-level kernels
int64_t tc_min_rows() { return (int64_t)sm_count() * SLOTS / 2; }

// Called by ft_factor_sweep_rows (sweep.cu) before its own dispatch: returns -1 when the
// tcgen05 sweep does not apply to this tree (no slot layout, shape, FT_FACTOR_TC=0).
int launch_factor_tc(const ft_tree_t *t, const ft_model_t *m, float lr, float reg,
                     cudaStream_t s) {
  if (!tc_enabled() || !t->slot_lc || t->slot_grid <= 0) return -1;
  const int N = t->order, u = t->root_mode;
  if (!tc_shape_ok(N, m->ranks[u], m->core_rank)) return -1;
  TcParams q{};
  q.slot_lc = t->slot_lc;
  q.slot_pc = t->slot_pc;
  q.slot_x = t->slot_x;
  q.batch_ptr = t->slot_batch_ptr;
  q.row_coord = t->row_coord;
  q.nrows = t->num_rows;
  for (int d = 1; d <= N - 2; ++d) q.Cpre[d - 1] = m->dots[(u + d) % N];
  q.Cleaf = m->dots[(u + N - 1) % N];
  q.A = m->factors[u];
  q.Bt = m->cores_t[u];
  q.J = m->ranks[u];
  q.R = m->core_rank;
  q.lr = lr;
  q.reg = reg;
  for (int d = 0; d < N; ++d)
    if (d != u && !m->dots[d]) return fail(FT_ERR_ARG, "dots[%d] is null", d);
  // the Fast2Sum residue when rows are long (tens of thousands of serial updates drift ~1e-4
  // in plain fp32; tests/test_netflix_parity_gpu.py)
  static const int force_comp = [] {  // FT_TC_COMP=0/1 forces the form (tests)
    const char *e = getenv("FT_TC_COMP");
    return e ? (strcmp(e, "0") == 0 ? 0 : 1) : -1;
  }();
  const bool comp = force_comp >= 0 ? force_comp == 1
                                    : t->num_rows > 0 && t->nnz / t->num_rows > 1024;
  if (N == 3) return launch_tc_t<1, 5>(q, t->slot_grid, comp, s);
  return launch_tc_t<2, 3>(q, t->slot_grid, comp, s);
}

}  // namespace ft

using namespace ft;

extern "C" int ft_tree_slot_plan(const ft_tree_t *tree, int32_t J, int32_t R, int32_t *grid_out,
                                 int32_t *batch_ptr, int64_t *len_out, void *stream) {
  if (!tree || !grid_out || !len_out) return fail(FT_ERR_ARG, "ft_tree_slot_plan: null argument");
  *grid_out = 0;
  *len_out = 0;
  const int64_t rows = tree->num_rows;
  if (!tree->row_leaf_ptr || !tree->leaf_pc || rows <= 0 || !tc_enabled() ||
      !tc_shape_ok(tree->order, J, R) || rows < tc_min_rows())
    return FT_OK;  // the tcgen05 sweep does not apply: no layout
  const int64_t G64 = (rows + SLOTS - 1) / SLOTS;
  const int G = (int)(G64 < sm_count() ? G64 : sm_count());
  if (!batch_ptr) {  // size query
    *grid_out = G;
    return FT_OK;
  }
  cudaStream_t s = as_stream(stream);
  int32_t *nbatch = nullptr;
  FT_CUDA(cudaMallocAsync(&nbatch, sizeof(int32_t) * G, s));
  slot_count_kernel<<<G, SLOTS, 0, s>>>(tree->row_leaf_ptr, rows, G, nbatch);
  if (int rc = check_launch("ft_tree_slot_plan(count)")) return rc;
  slot_scan_kernel<<<1, 32, 0, s>>>(nbatch, G, batch_ptr);
  if (int rc = check_launch("ft_tree_slot_plan(scan)")) return rc;
  int32_t total = 0;
  FT_CUDA(cudaMemcpyAsync(&total, batch_ptr + G, sizeof(int32_t), cudaMemcpyDeviceToHost, s));
  FT_CUDA(cudaFreeAsync(nbatch, s));
  FT_CUDA(cudaStreamSynchronize(s));
  *grid_out = G;
  *len_out = (int64_t)total * SLOTS;
  return FT_OK;
}

extern "C" int ft_tree_slot_fill(const ft_tree_t *tree, int32_t grid, const int32_t *batch_ptr,
                                 int32_t *slot_lc, int32_t *slot_pc, float *slot_x,
                                 void *stream) {
  if (!tree || !batch_ptr || !slot_lc || !slot_x || grid <= 0)
    return fail(FT_ERR_ARG, "ft_tree_slot_fill: null argument");
  const int npre = tree->order - 2;
  if (npre > 0 && (!slot_pc || !tree->leaf_pc))
    return fail(FT_ERR_ARG, "ft_tree_slot_fill: prefix index missing");
  slot_fill_kernel<<<grid, SLOTS, 0, as_stream(stream)>>>(
      tree->row_leaf_ptr, tree->num_rows, grid, npre, batch_ptr, tree->leaf_coord, tree->leaf_pc,
      tree->vals, slot_lc, slot_pc, slot_x);
  return check_launch("ft_tree_slot_fill");
}
