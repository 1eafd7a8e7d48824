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
//   * one elected thread issues the 3xTF32 combine as 2 x R/8 MMAs at N = 64 (M = 128 slots,
//     K = R in steps of 8; B = [Bt_hi ; Bt_lo] then [Bt_hi ; 0] in shared memory, K-major,
//     128-B swizzle) and commits to an mbarrier; thread s reads v (its TMEM lane) with
//     tcgen05.ld and runs the step.  Two TMEM stages: the MMA of batch b overlaps the chain of
//     batch b-1 and the gathers of batches up to b+GS-1 are in flight.
// Requirements (checked by the dispatcher): 3 <= N <= 4, J <= 32, R <= 32 with R % 4 == 0, the
// slot layout present.
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include <cub/cub.cuh>

#include "ft_common.cuh"

namespace ft {
namespace {

constexpr int SLOTS = 128;
constexpr int CWARPS = 4;                    // consumer warps: warp <-> TMEM lanes 32(w%4)..+31
// PW producer warps per TMEM lane quadrant (they take alternate batches), 4 consumer warps, the
// MMA warp
template <int PW, int KB = 1>
constexpr int tc_threads() { return (4 * PW + CWARPS + 1) * 32; }
// TMEM: AS A stages (A_hi | A_lo, 64 columns each) then DS D stages (64 columns each).  The A
// ring is the deep one: a producer reuses an A stage once that batch's MMAs completed, so the
// producers run up to AS batches ahead of the tensor core; consumers trail the MMA closely.
constexpr int AS = 6, DS = 2;
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

// K3c-wide (KB = 8) chain in the quad layout: lane (row group of 8 lanes, k) holds columns
// 4k .. 4k + 3 of its row (the quadw consumer's arithmetic, sweep.cu / quad.cuh).
namespace k3w {
__device__ __forceinline__ float dot(const float (&a)[4], const float4 v) {
  float2 pr = f2fma(make_float2(a[0], a[1]), make_float2(v.x, v.y), make_float2(0.f, 0.f));
  pr = f2fma(make_float2(a[2], a[3]), make_float2(v.z, v.w), pr);
  float s = pr.x + pr.y;
  s += __shfl_xor_sync(FULL, s, 4);
  s += __shfl_xor_sync(FULL, s, 2);
  s += __shfl_xor_sync(FULL, s, 1);
  return s;
}
// compensated update a <- a + (c a + lr e v) (Fast2Sum residue lo; m = (x, lr, c, c))
__device__ __forceinline__ void update(float (&a)[4], float (&lo)[4], const float4 v, float4 m,
                                       float e) {
  const float2 l2 = make_float2(m.y * e, m.y * e), c2 = make_float2(m.z, m.w);
  const float2 a01 = make_float2(a[0], a[1]), a23 = make_float2(a[2], a[3]);
  const float2 d01 = f2fma(l2, make_float2(v.x, v.y), f2fma(c2, a01, make_float2(lo[0], lo[1])));
  const float2 d23 = f2fma(l2, make_float2(v.z, v.w), f2fma(c2, a23, make_float2(lo[2], lo[3])));
  const float2 t01 = f2add(a01, d01), t23 = f2add(a23, d23);
  const float2 r01 = f2sub(d01, f2sub(t01, a01)), r23 = f2sub(d23, f2sub(t23, a23));
  a[0] = t01.x, a[1] = t01.y, a[2] = t23.x, a[3] = t23.y;
  lo[0] = r01.x, lo[1] = r01.y, lo[2] = r23.x, lo[3] = r23.y;
}
__device__ __forceinline__ void step(float (&a)[4], float (&lo)[4], const float4 v, float4 m) {
  update(a, lo, v, m, m.x - dot(a, v));
}
}  // namespace k3w

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

template <int NPRE, int GS, int KB = 1>
struct TcPlan {
  static_assert((GS & (GS - 1)) == 0, "gather ring stages: a power of two");
  static constexpr int LEVELS = NPRE + 1;                 // gathered C rows per leaf
  static constexpr int STAGE = SLOTS * LEVELS * 128;      // bytes per gather stage
  static constexpr int B_BYTES = 64 * 128;                // B tile: N = 64 rows of 128 B
  // metadata ring stages: requested 2 GS - 1 batches ahead of the producer, read by the
  // consumer up to AS + DS batches behind it (see the barrier chain in the kernel)
  static constexpr int MS = 4 * GS > 16 ? 4 * GS : 16;
  static_assert(MS >= 2 * GS + AS + DS, "metadata ring too short");  // (2 GS - PW) + AS + DS + 1
  static constexpr int MSTRIDE = (NPRE + 2) * SLOTS * 4;  // lc|flags, pc[NPRE], x per stage
  static constexpr int NABUF = SLOTS * 128;              // each consumer's next A row
  static constexpr int VBUF = KB > 1 ? CWARPS * 32 * 128 : 0;  // KB = 8: per-warp V transpose
  static constexpr size_t SMEM =
      1024 + 2 * B_BYTES + (size_t)GS * STAGE + MS * MSTRIDE + NABUF + VBUF + 256;
};

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];\n" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ float4 lds128(uint32_t a) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];\n"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(a)
               : "memory");
  return v;
}
__device__ __forceinline__ void cp4(uint32_t dst, const void *src, bool on) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 4;\n}\n" ::"r"(dst),
      "l"(src), "r"((int)on));
}
__device__ __forceinline__ void cp16p(uint32_t dst, const void *src, bool on) {
  asm volatile(
      "{\n .reg .pred q;\n setp.ne.b32 q, %2, 0;\n @q cp.async.ca.shared.global [%0], [%1], 16;\n}\n" ::"r"(dst),
      "l"(src), "r"((int)on));
}

// R32: R == 32 (no chunk predicates, shift addressing); COMP: Fast2Sum-compensated row.
// Warp roles (one 128-slot set per CTA): warps 0-3 PRODUCE (metadata + gathers + cross -> TMEM
// A), warps 4-7 CONSUME (TMEM D -> chain), warp 8 issues the MMAs.  Warps w and w + 4 serve the
// same TMEM lane quadrant.  Barriers per TMEM stage st = b % 4:
//   a_ready[st]  producers -> MMA   (A of batch b written)
//   v_ready[st]  MMA commit -> consumers (D of batch b) and producers (A of batch b free again)
//   d_free[st]   consumers -> MMA   (D of batch b read)
template <int NPRE, int GS, bool R32, bool COMP, int PW, int KB>
__global__ void __launch_bounds__(tc_threads<PW, KB>(), 1) factor_rows_tc_kernel(const TcParams p) {
  constexpr int THREADS = tc_threads<PW, KB>(), NPW = 4 * PW;  // producer warps: 0 .. NPW - 1
  constexpr int WMMA = NPW + CWARPS;
  static_assert(GS % PW == 0, "each producer parity owns GS / PW ring stages");
  constexpr int D = GS / PW;                               // per-warp gather lookahead
  using P = TcPlan<NPRE, GS, KB>;
  extern __shared__ __align__(1024) uint8_t smraw[];
  // 1024-B aligned operand tiles, addressed as shared-window offsets
  const uint32_t sraw = su32(smraw);
  const uint32_t sbase = (sraw + 1023u) & ~1023u;
  const uint32_t b_hi = sbase, b_lo = sbase + P::B_BYTES;
  const uint32_t ring = sbase + 2 * P::B_BYTES;
  const uint32_t meta = ring + GS * P::STAGE;
  const uint32_t nabuf = meta + P::MS * P::MSTRIDE;
  const uint32_t vbuf = nabuf + P::NABUF;                  // KB > 1: [4 warps][32 rows][128 B]
  const uint32_t bars = nabuf + P::NABUF + P::VBUF;
  uint8_t *gbase = smraw + (sbase - sraw);
  uint64_t *a_ready = reinterpret_cast<uint64_t *>(gbase + (bars - sbase));
  uint64_t *a_free = a_ready + AS, *v_ready = a_free + AS, *d_free = v_ready + DS;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(d_free + DS);
    const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int J = p.J, R = R32 ? 32 : p.R;

  // B operands (N = 64, K-major, 128-B swizzle, zero padded): P = [Bt_hi^T ; Bt_lo^T] and
  // Q = [Bt_hi^T ; 0], so that D[:, 0:32] = A_hi Bt_hi + A_lo Bt_hi and D[:, 32:64] = A_hi Bt_lo
  // (v = the sum of the two halves): 3xTF32 in 2 x ksteps N = 64 MMAs instead of 3 x ksteps at
  // N = 32 (tools/umma_probe.cu: an N = 64 MMA costs about what an N = 32 one does)
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
    *reinterpret_cast<uint4 *>(gbase + off) = h;                            // P rows 0-31
    *reinterpret_cast<uint4 *>(gbase + 32 * 128 + off) = l;                 // P rows 32-63
    *reinterpret_cast<uint4 *>(gbase + P::B_BYTES + off) = h;               // Q rows 0-31
    *reinterpret_cast<uint4 *>(gbase + P::B_BYTES + 32 * 128 + off) = make_uint4(0, 0, 0, 0);
  }
  if (w == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
        su32(tmem_slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  if (tid == 0) {
    for (int k = 0; k < AS; ++k) mbar_init(a_ready + k, CWARPS), mbar_init(a_free + k, 1);
    for (int k = 0; k < DS; ++k) mbar_init(v_ready + k, 1), mbar_init(d_free + k, CWARPS);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // B tiles -> tensor core
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int64_t b0 = __ldg(p.batch_ptr + blockIdx.x);
  const int nb = __ldg(p.batch_ptr + blockIdx.x + 1) - (int)b0;
  const int q = w & 3;                      // TMEM lane quadrant
  const int s = 32 * q + lane;              // slot = TMEM lane
  const uint32_t tlane = tmem + ((uint32_t)(32 * q) << 16);
  const uint32_t my_meta = meta + 4 * s;

  if (w == WMMA) {  // ---- MMA warp ----
    // MMA issue for batch m (warp 8, lane 0): D = A_lo Bt_hi +
    // A_hi Bt_lo + A_hi Bt_hi once every producer arrived (a_ready) and every consumer read the
    // stage's previous D (d_free of batch m - 4); kind::tf32, D fp32, A (TMEM) / B (smem) tf32
    // K-major, N = 32, M = 128
    const uint32_t idesc =
        (1u << 4) | (2u << 7) | (2u << 10) | ((64u >> 3) << 17) | ((128u >> 4) << 24);
    const int ksteps = (R + 7) >> 3;
    auto mma_issue = [&](int m) {
      const int ast = m % AS, dst = m % DS;
      mbar_wait(a_ready + ast, (m / AS) & 1);
      if (m >= DS) mbar_wait(d_free + dst, (m / DS - 1) & 1);
      tc_fence_after();
      const uint32_t ah = tmem + 64 * ast, al = ah + 32, d = tmem + 64 * AS + 64 * dst;
      for (int k = 0; k < ksteps; ++k) mma_ts(d, ah + 8 * k, sw128(b_hi + 32 * k), idesc, k > 0);
      for (int k = 0; k < ksteps; ++k) mma_ts(d, al + 8 * k, sw128(b_lo + 32 * k), idesc, 1);
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              su32(a_free + ast))
          : "memory");
      asm volatile(
          "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
              su32(v_ready + dst))
          : "memory");
    };
    for (int m = 0; m < nb; ++m) {
      if (lane == 0) mma_issue(m);
      __syncwarp();
    }
  } else if (w < NPW) {  // ---- producers: metadata, gathers, cross -> TMEM A ----
    const int par = w >> 2;  // this warp's batches: par, par + PW, par + 2 PW, ...
    const int gc = lane & 7, gs = lane >> 3;
    const bool gok = R32 || gc < (R >> 2);
    // gather copy geometry: copy `it` of a level moves chunk gc of slot t = 4 it + gs of this
    // warp; its swizzled chunk is gc ^ (t & 7) = gc ^ (gs + 4 (it & 1))
    const uint32_t gdst0 = (uint32_t)((32 * q + gs) * 128 + ((gc ^ gs) << 4));
    const uint32_t gdst1 = (uint32_t)((32 * q + gs + 4) * 128 + ((gc ^ (gs + 4)) << 4));
    const uint32_t my_row = (uint32_t)(s * 128), swz = (uint32_t)(lane & 7);
    // metadata requests run 2 D - 1 own batches (2 GS - PW batches) ahead of the cross
    const int64_t mfirst = b0 + par + PW * (2 * D - 1);
    const int32_t *src_lc = p.slot_lc + mfirst * SLOTS + s;
    const int32_t *src_pc = p.slot_pc + mfirst * NPRE * SLOTS + s;
    const float *src_x = p.slot_x + mfirst * SLOTS + s;
    const char *Cl[NPRE + 1];
#pragma unroll
    for (int lv = 0; lv < NPRE; ++lv) Cl[lv] = reinterpret_cast<const char *>(p.Cpre[lv]) + 16 * gc;
    Cl[NPRE] = reinterpret_cast<const char *>(p.Cleaf) + 16 * gc;
    const uint32_t rowb = (uint32_t)R * 4;

    auto request_meta_at = [&](int g, const int32_t *lcp, const int32_t *pcp, const float *xp) {
      const bool on = g < nb;
      const uint32_t m0 = my_meta + (uint32_t)((g & (P::MS - 1)) * P::MSTRIDE);
      cp4(m0, lcp, on);
#pragma unroll
      for (int d = 0; d < NPRE; ++d) cp4(m0 + 4 * SLOTS * (1 + d), pcp + d * SLOTS, on);
      cp4(m0 + 4 * SLOTS * (1 + NPRE), xp, on);
    };
    // gathers of batch g into ring stage g % GS (cooperative: 8 lanes per 128-B row); padding
    // slots copy row 0 (their cross is zeroed)
    auto issue = [&](int g) {
      if (g >= nb) return;  // warp-uniform
      const uint32_t m0 = my_meta + (uint32_t)((g & (P::MS - 1)) * P::MSTRIDE);
      const int lcf = (int)lds32(m0);
      const bool pad = lcf == PAD;
      uint32_t coord[NPRE + 1];
#pragma unroll
      for (int d = 0; d < NPRE; ++d) coord[d] = pad ? 0u : lds32(m0 + 4 * SLOTS * (1 + d));
      coord[NPRE] = pad ? 0u : ((uint32_t)lcf & ~ROW_START);
      const uint32_t st0 = ring + (uint32_t)((g & (GS - 1)) * P::STAGE);
#pragma unroll
      for (int lv = 0; lv <= NPRE; ++lv) {
        const uint32_t lbase = st0 + lv * (SLOTS * 128);
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const uint32_t cs = __shfl_sync(FULL, coord[lv], 4 * it + gs);
          const uint32_t dst = lbase + (it & 1 ? gdst1 : gdst0) + (it >> 1) * 1024;
          // base + cs * row bytes in one 64-bit multiply-add
          const void *src;
          asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(src) : "r"(cs), "r"(R32 ? 128u : rowb),
              "l"(Cl[lv]));
          if (R32)
            cp16(dst, src);
          else
            cp16p(dst, src, gok);
        }
      }
    };

    // prologue: metadata of own batches 0 .. 2 D - 2 (landed), gathers of own batches 0 .. D - 2
#pragma unroll 1
    for (int i = 0; i < 2 * D - 1; ++i) {
      const int g = par + PW * i;
      request_meta_at(g, p.slot_lc + (b0 + g) * SLOTS + s, p.slot_pc + (b0 + g) * NPRE * SLOTS + s,
                      p.slot_x + (b0 + g) * SLOTS + s);
    }
    cp_commit();
    cp_wait<0>();
#pragma unroll 1
    for (int i = 0; i < D - 1; ++i) {
      issue(par + PW * i);
      cp_commit();
    }
#pragma unroll 1
    for (int b = par; b < nb; b += PW) {
      // one group per own batch (empty past the end keeps the count uniform): the metadata of
      // own batch +2D-1 and the gathers of own batch +D-1, whose metadata retired with the
      // group of own batch -D
      request_meta_at(b + PW * (2 * D - 1), src_lc, src_pc, src_x);
      src_lc += PW * SLOTS, src_pc += PW * NPRE * SLOTS, src_x += PW * SLOTS;
      issue(b + PW * (D - 1));
      cp_commit();
      cp_wait<D - 1>();   // this lane's copies of batch b have landed
      __syncwarp();       // ... and every lane's
      const int st = b % AS;
      if (b >= AS) mbar_wait(a_free + st, (b / AS - 1) & 1);  // MMAs of batch b - AS done
      tc_fence_after();
      // cross of slot s -> 3xTF32 halves -> TMEM A stage st
      const uint32_t st0 = ring + (uint32_t)((b & (GS - 1)) * P::STAGE) + my_row;
      const uint32_t ah = tlane + 64 * st, al = ah + 32;
#pragma unroll
      for (int h = 0; h < 4; ++h) {  // 8 columns per TMEM store
        uint32_t hv[8], lv8[8];
#pragma unroll
        for (int qq = 0; qq < 2; ++qq) {
          const int c = 2 * h + qq;
          // padding slots gathered C row 0 (finite; the consumer skips their step); only the
          // chunks past R (never copied, and multiplied by B's zero padding) must read as zero
          float4 x = make_float4(0.f, 0.f, 0.f, 0.f);
          if (R32 || 4 * c < R) {
            const uint32_t co = (uint32_t)((c ^ swz) << 4);
            x = lds128(st0 + co);
#pragma unroll
            for (int lv = 1; lv <= NPRE; ++lv) {
              const float4 y = lds128(st0 + lv * (SLOTS * 128) + co);
              const float2 p01 = f2fma(make_float2(x.x, x.y), make_float2(y.x, y.y), make_float2(0.f, 0.f));
              const float2 p23 = f2fma(make_float2(x.z, x.w), make_float2(y.z, y.w), make_float2(0.f, 0.f));
              x = make_float4(p01.x, p01.y, p23.x, p23.y);
            }
          }
          const uint32_t h0 = hi_bits(x.x), h1 = hi_bits(x.y), h2 = hi_bits(x.z), h3 = hi_bits(x.w);
          // lo = x - hi as one packed FMA per pair: hi * (-1) + x
          const float2 l01 = f2fma(make_float2(__uint_as_float(h0), __uint_as_float(h1)),
                                   make_float2(-1.f, -1.f), make_float2(x.x, x.y));
          const float2 l23 = f2fma(make_float2(__uint_as_float(h2), __uint_as_float(h3)),
                                   make_float2(-1.f, -1.f), make_float2(x.z, x.w));
          hv[4 * qq] = h0, hv[4 * qq + 1] = h1, hv[4 * qq + 2] = h2, hv[4 * qq + 3] = h3;
          lv8[4 * qq] = __float_as_uint(l01.x), lv8[4 * qq + 1] = __float_as_uint(l01.y);
          lv8[4 * qq + 2] = __float_as_uint(l23.x), lv8[4 * qq + 3] = __float_as_uint(l23.y);
        }
        tmem_st8(ah + 8 * h, hv);
        tmem_st8(al + 8 * h, lv8);
      }
      asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
      tc_fence_before();
      __syncwarp();  // every lane's stores (and its reads of the ring stage) are done
      if (lane == 0) mbar_arrive(a_ready + st);
    }
    cp_wait<0>();
  } else if (KB == 1) {  // ---- consumers: slot s = TMEM lane s = this thread's row chain ----
    const int64_t gslots = (int64_t)gridDim.x * SLOTS;
    const float lr = p.lr, cdec = -p.lr * p.reg;
    float a[32], lo[32];
    // this slot's rows: the contiguous block [q rows / GS, (q + 1) rows / GS) (K1d)
    int64_t row = ((int64_t)blockIdx.x + (int64_t)gridDim.x * s) * p.nrows / gslots;
    bool have = false;                                          // a holds a row
    int64_t cur_i = -1;
    // row coordinates run two rows ahead of the chain and the next row's A values are copied
    // into this thread's shared-memory buffer one row ahead (cp.async: no registers held), so
    // a row switch never waits on a global load
    int ci1 = row < p.nrows ? __ldg(p.row_coord + row) : -1;
    int ci2 = row + 1 < p.nrows ? __ldg(p.row_coord + row + 1) : -1;
    const uint32_t my_na = nabuf + (uint32_t)(s * 128);
    auto prefetch_row = [&](int ci) {
      if (ci >= 0) {
        const float *ar = p.A + (int64_t)ci * J;
        if (J == 32) {
#pragma unroll
          for (int c = 0; c < 8; ++c) cp16(my_na + 16 * c, ar + 4 * c);
        } else {
          for (int j = 0; j < J; ++j) cp4(my_na + 4 * j, ar + j, true);
        }
      }
      cp_commit();
    };
    auto install_row = [&]() {
      cp_wait<0>();
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float4 q4 = lds128(my_na + 16 * c);
        a[4 * c] = q4.x, a[4 * c + 1] = q4.y, a[4 * c + 2] = q4.z, a[4 * c + 3] = q4.w;
      }
      if (J < 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j)
          if (j >= J) a[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 32; ++j) lo[j] = 0.f;
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
    for (int j = 0; j < 32; ++j) a[j] = 0.f, lo[j] = 0.f;
    prefetch_row(ci1);  // the first row's values, installed at its first leaf
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      const int st = b % DS;
      mbar_wait(v_ready + st, (b / DS) & 1);
      tc_fence_after();
      float v[32], v2[32];
      tmem_ld32(tlane + 64 * AS + 64 * st, v);
      tmem_ld32(tlane + 64 * AS + 64 * st + 32, v2);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 t = f2add(make_float2(v[j], v[j + 1]), make_float2(v2[j], v2[j + 1]));
        v[j] = t.x, v[j + 1] = t.y;
      }
      const uint32_t mb0 = my_meta + (uint32_t)((b & (P::MS - 1)) * P::MSTRIDE);
      const int mlc = (int)lds32(mb0);
      const float x = __uint_as_float(lds32(mb0 + 4 * SLOTS * (1 + NPRE)));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_free + st);
      if (mlc == PAD) continue;
      if ((uint32_t)mlc & ROW_START) {
        if (have) {
          store_row();
          row += 1;
          ci1 = ci2;
          ci2 = row + 1 < p.nrows ? __ldg(p.row_coord + row + 1) : -1;
        }
        have = true;
        cur_i = ci1;
        install_row();
        prefetch_row(ci2);  // the slot's next row
      }
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
    }
    if (have) store_row();
  } else {  // ---- KB = 8: consumers in the quad layout (4 row slots per warp, 8 lanes each) ----
    // TMEM lane s = 32 q + lane holds leaf k = lane & 7 of row slot rs = 4 q + (lane >> 3).  The
    // warp transposes its 32 V rows through 4 KB of shared memory (8 STS.128 + 8 LDS.128 per
    // lane, swizzled chunk c of row r at c ^ (r & 7): conflict-free both ways), so that lane
    // (rl, k) holds columns 4k .. 4k + 3 of all 8 leaves of its row, and runs the row's chain in
    // the quad layout (sweep.cu quadw): dot products over 8 lanes (3 shuffle levels).  A batch
    // containing a row start or padding (once per row) takes the checked per-step path.
    // (Measured: shared-memory / MIO-bound with the producers' gathers -- the producers spin on
    // a_free 38 % of the samples, and one step of lookahead in the chain changed nothing:
    // profiles/r02_factor_tc_ab.md.)
    const int rl = lane >> 3, k = lane & 7;
    const int rs = 4 * q + rl;
    const int64_t gslots = (int64_t)gridDim.x * (SLOTS / KB);
    const float lr = p.lr, cdec = -p.lr * p.reg;
    float a[4], lo[4];
    int64_t row = ((int64_t)blockIdx.x + (int64_t)gridDim.x * rs) * p.nrows / gslots;
    bool have = false;
    int64_t cur_i = -1;
    int ci1 = row < p.nrows ? __ldg(p.row_coord + row) : -1;
    int ci2 = row + 1 < p.nrows ? __ldg(p.row_coord + row + 1) : -1;
    const uint32_t my_na = nabuf + (uint32_t)(rs * 128 + 16 * k);
    const int j0 = 4 * k;
    const uint32_t tb = vbuf + (uint32_t)(q * 32 * 128);
    auto prefetch_row = [&](int ci) {
      if (ci >= 0) {
        const float *ar = p.A + (int64_t)ci * J + j0;
        if (J == 32) {
          cp16(my_na, ar);
        } else {
          for (int j = 0; j < 4; ++j) cp4(my_na + 4 * j, ar + j, j0 + j < J);
        }
      }
      cp_commit();
    };
    auto install_row = [&]() {
      cp_wait<0>();
      const float4 q0 = lds128(my_na);
      a[0] = q0.x, a[1] = q0.y, a[2] = q0.z, a[3] = q0.w;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j0 + j >= J) a[j] = 0.f;
        lo[j] = 0.f;
      }
    };
    auto store_row = [&]() {
      float *ar = p.A + cur_i * J + j0;
      if (J == 32) {
        *reinterpret_cast<float4 *>(ar) = make_float4(a[0], a[1], a[2], a[3]);
      } else {
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (j0 + j < J) ar[j] = a[j];
      }
    };
#pragma unroll
    for (int j = 0; j < 4; ++j) a[j] = 0.f, lo[j] = 0.f;
    prefetch_row(ci1);
#pragma unroll 1
    for (int b = 0; b < nb; ++b) {
      const int st = b % DS;
      mbar_wait(v_ready + st, (b / DS) & 1);
      tc_fence_after();
      float v[32], v2[32];
      tmem_ld32(tlane + 64 * AS + 64 * st, v);
      tmem_ld32(tlane + 64 * AS + 64 * st + 32, v2);
      // the row's 8 entries of the metadata stage: leaf coordinate | flags and value
      const uint32_t mb0 = meta + (uint32_t)((b & (P::MS - 1)) * P::MSTRIDE) + 4 * (8 * rs);
      const int4 lc0 = *reinterpret_cast<const int4 *>(gbase + (mb0 - sbase));
      const int4 lc1 = *reinterpret_cast<const int4 *>(gbase + (mb0 + 16 - sbase));
      const uint32_t xb = mb0 + 4 * SLOTS * (1 + NPRE);
      const float4 x0 = *reinterpret_cast<const float4 *>(gbase + (xb - sbase));
      const float4 x1 = *reinterpret_cast<const float4 *>(gbase + (xb + 16 - sbase));
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(d_free + st);
      // transpose: my leaf's V row (sum of the two TMEM halves) -> row 8 rl + k of the buffer
      const uint32_t myrow = tb + (uint32_t)((8 * rl + k) * 128);
#pragma unroll
      for (int c = 0; c < 8; ++c) {
        const float2 t0 = f2add(make_float2(v[4 * c], v[4 * c + 1]), make_float2(v2[4 * c], v2[4 * c + 1]));
        const float2 t1 = f2add(make_float2(v[4 * c + 2], v[4 * c + 3]), make_float2(v2[4 * c + 2], v2[4 * c + 3]));
        asm volatile("st.shared.v4.f32 [%0], {%1,%2,%3,%4};\n" ::"r"(myrow + (((uint32_t)(c ^ k)) << 4)),
                     "f"(t0.x), "f"(t0.y), "f"(t1.x), "f"(t1.y)
                     : "memory");
      }
      __syncwarp();
      float4 vv[8];
#pragma unroll
      for (int i = 0; i < 8; ++i)
        vv[i] = lds128(tb + (uint32_t)((8 * rl + i) * 128) + (((uint32_t)(k ^ i)) << 4));
      __syncwarp();  // every lane's reads are done before the next batch's stores
      const int lcs[8] = {lc0.x, lc0.y, lc0.z, lc0.w, lc1.x, lc1.y, lc1.z, lc1.w};
      const float xs[8] = {x0.x, x0.y, x0.z, x0.w, x1.x, x1.y, x1.z, x1.w};
      bool odd = false;
#pragma unroll
      for (int i = 0; i < 8; ++i) odd |= lcs[i] == PAD || ((uint32_t)lcs[i] & ROW_START);
      float4 mm[8];
      if (!__any_sync(FULL, odd)) {
#pragma unroll
        for (int i = 0; i < 8; ++i) mm[i] = make_float4(xs[i], lr, cdec, cdec);
#pragma unroll
        for (int i = 0; i < 8; ++i) k3w::step(a, lo, vv[i], mm[i]);
      } else {
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const bool live = lcs[i] != PAD;
          if (live && ((uint32_t)lcs[i] & ROW_START)) {  // the row group's lanes together
            if (have) {
              store_row();
              row += 1;
              ci1 = ci2;
              ci2 = row + 1 < p.nrows ? __ldg(p.row_coord + row + 1) : -1;
            }
            have = true;
            cur_i = ci1;
            install_row();
            prefetch_row(ci2);
          }
          __syncwarp();
          const float4 m = live ? make_float4(xs[i], lr, cdec, cdec) : make_float4(0.f, 0.f, 0.f, 0.f);
          k3w::step(a, lo, vv[i], m);
        }
      }
    }
    if (have) store_row();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (w == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tmem));
}

// ---- K1d: the slot layout ------------------------------------------------------------------
// KB leaves of one row slot per batch: a CTA has RS = 128 / KB row slots; row slot q = c + G rs
// (CTA c, rs < RS) of GS = G RS owns the contiguous rows [q rows / GS, (q + 1) rows / GS) of
// the tree, so its stream is ONE contiguous range of the tree's leaves.  Stream position p of q
// sits in batch p / KB at TMEM lane / entry slot s = KB rs + p % KB: entry
// (batch_ptr[c] + p / KB) * 128 + s.  KB = 1: one thread per row (K3c); KB = 8: 16 rows per CTA
// for few, long rows (K3c-wide).
__device__ __forceinline__ int64_t slot_first_row(int64_t q, int64_t rows, int64_t gs) {
  return q * rows / gs;
}
// slot_rows_kernel: per CTA its batch count (the longest stream of its row slots)
__global__ void slot_rows_kernel(const int32_t *__restrict__ row_leaf_ptr, int64_t rows, int G,
                                 int KB, int32_t *__restrict__ nbatch) {
  const int c = blockIdx.x, RS = SLOTS / KB;
  const int64_t gs = (int64_t)G * RS;
  int64_t tot = 0;
  if ((int)threadIdx.x < RS) {
    const int64_t q = c + (int64_t)G * threadIdx.x;
    tot = __ldg(row_leaf_ptr + slot_first_row(q + 1, rows, gs)) -
          __ldg(row_leaf_ptr + slot_first_row(q, rows, gs));
  }
  using BR = cub::BlockReduce<int64_t, SLOTS>;
  __shared__ typename BR::TempStorage ts;
  const int64_t mx = BR(ts).Reduce(tot, cub::Max());
  if (threadIdx.x == 0) nbatch[c] = (int32_t)((mx + KB - 1) / KB);
}
// the first leaf of every row, as a byte flag per leaf (row starts for the fill)
__global__ void row_start_kernel(const int32_t *__restrict__ row_leaf_ptr, int64_t rows,
                                 uint8_t *__restrict__ flag) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) flag[row_leaf_ptr[r]] = 1;
}

__global__ void slot_scan_kernel(const int32_t *__restrict__ nbatch, int G, int32_t *batch_ptr,
                                 int32_t *total_max) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int32_t acc = 0, mx = 0;
    for (int c = 0; c < G; ++c) {
      batch_ptr[c] = acc;
      acc += nbatch[c];
      mx = nbatch[c] > mx ? nbatch[c] : mx;
    }
    batch_ptr[G] = acc;
    total_max[0] = acc;
    total_max[1] = mx;
  }
}

// block (c, j): batches [32 j, 32 j + 32) of CTA c.  Phase 1, warp per entry slot: lane i takes
// the slot's stream position for batch 32 j + i -- leaf (first leaf of the slot) + position,
// coalesced -- into a padded shared tile [i][s]; phase 2, thread per slot: each batch's 128
// entries leave as one coalesced store.
constexpr int FILL_B = 32, FILL_PAD = SLOTS + 1;
template <int NPRE>
__global__ void __launch_bounds__(SLOTS) slot_fill_kernel(
    const int32_t *__restrict__ row_leaf_ptr, const uint8_t *__restrict__ row_start, int64_t rows,
    int G, int KB, const int32_t *__restrict__ batch_ptr, const int32_t *__restrict__ leaf_coord,
    const int32_t *__restrict__ leaf_pc, const float *__restrict__ vals,
    int32_t *__restrict__ slot_lc, int32_t *__restrict__ slot_pc, float *__restrict__ slot_x) {
  extern __shared__ int32_t fill_smem[];
  int32_t *t_lc = fill_smem;                                          // [FILL_B][FILL_PAD]
  int32_t *t_pc = t_lc + FILL_B * FILL_PAD;                           // [NPRE][FILL_B][FILL_PAD]
  float *t_x = reinterpret_cast<float *>(t_pc + NPRE * FILL_B * FILL_PAD);
  __shared__ int64_t s_leaf0[SLOTS], s_leafe[SLOTS];
  const int c = blockIdx.x, RS = SLOTS / KB, lane = threadIdx.x & 31, wp = threadIdx.x >> 5;
  const int64_t b0 = batch_ptr[c];
  const int nb = batch_ptr[c + 1] - (int)b0;
  const int jb = (int)blockIdx.y * FILL_B;
  if (jb >= nb) return;
  const int64_t gs = (int64_t)G * RS;
  {  // this thread's row slot: its leaf range
    const int rs = threadIdx.x / KB;
    const int64_t q = c + (int64_t)G * rs;
    s_leaf0[threadIdx.x] = row_leaf_ptr[slot_first_row(q, rows, gs)];
    s_leafe[threadIdx.x] = row_leaf_ptr[slot_first_row(q + 1, rows, gs)];
  }
  __syncthreads();
#pragma unroll 4
  for (int s = wp; s < SLOTS; s += SLOTS / 32) {
    const int k = s % KB;
    const int64_t L = s_leaf0[s] + (int64_t)(jb + lane) * KB + k;
    const int e = lane * FILL_PAD + s;
    if (L < s_leafe[s]) {
      t_lc[e] = (int32_t)((uint32_t)__ldg(leaf_coord + L) | (row_start[L] ? ROW_START : 0u));
#pragma unroll
      for (int d = 0; d < NPRE; ++d) t_pc[d * FILL_B * FILL_PAD + e] = __ldg(leaf_pc + L * NPRE + d);
      t_x[e] = __ldg(vals + L);
    } else {
      t_lc[e] = PAD;
#pragma unroll
      for (int d = 0; d < NPRE; ++d) t_pc[d * FILL_B * FILL_PAD + e] = 0;
      t_x[e] = 0.f;
    }
  }
  __syncthreads();
  const int s = threadIdx.x;
  const int nbat = nb - jb < FILL_B ? nb - jb : FILL_B;
  for (int i = 0; i < nbat; ++i) {
    const int64_t e = (b0 + jb + i) * SLOTS + s;
    slot_lc[e] = t_lc[i * FILL_PAD + s];
#pragma unroll
    for (int d = 0; d < NPRE; ++d)
      slot_pc[((b0 + jb + i) * NPRE + d) * SLOTS + s] = t_pc[d * FILL_B * FILL_PAD + i * FILL_PAD + s];
    slot_x[e] = t_x[i * FILL_PAD + s];
  }
}
template <int NPRE>
constexpr size_t fill_smem_bytes() { return (size_t)(2 + NPRE) * FILL_B * FILL_PAD * 4; }

// R > 16: at R = 16 the MMA count per batch halves but its fixed cost does not, and quadr's
// mma.sync combine is faster (Netflix16 modes 0/1: 2.3 vs 3.5 ms; profiles/r02_factor_tc_ab.md)
bool tc_shape_ok(int N, int J, int R) {
  return N >= 3 && N <= 4 && J >= 1 && J <= 32 && R > 16 && R <= 32 && R % 4 == 0;
}

// FT_FACTOR_TC=0 disables the tcgen05 factor sweep (the quadr / quadw kernels run instead)
bool tc_enabled() {
  static const bool on = [] {
    const char *e = getenv("FT_FACTOR_TC");
    return !(e && strcmp(e, "0") == 0);
  }();
  return on;
}

template <int NPRE, int GS, bool R32, bool COMP, int PW, int KB = 1>
int launch_tc_k(const TcParams &q, int G, cudaStream_t s) {
  const size_t sm = TcPlan<NPRE, GS, KB>::SMEM;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_tc_kernel<NPRE, GS, R32, COMP, PW, KB>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  factor_rows_tc_kernel<NPRE, GS, R32, COMP, PW, KB><<<G, tc_threads<PW, KB>(), sm, s>>>(q);
  return check_launch(KB == 1 ? "ft_factor_sweep_rows(tcgen05)" : "ft_factor_sweep_rows(tcgen05 wide)");
}
// the plain chain fits the 13-warp block's 128 registers (two producer warps per quadrant); the
// compensated one (156 registers) keeps one producer warp per quadrant
// (and so does a ring too shallow to give each of two warps a batch of lookahead)
template <int NPRE, int GS>
int launch_tc_t(const TcParams &q, int G, bool comp, cudaStream_t s) {
  constexpr int PW2 = GS >= 4 ? 2 : 1;
  if (q.R == 32)
    return comp ? launch_tc_k<NPRE, GS, true, true, 1>(q, G, s)
                : launch_tc_k<NPRE, GS, true, false, PW2>(q, G, s);
  return comp ? launch_tc_k<NPRE, GS, false, true, 1>(q, G, s)
              : launch_tc_k<NPRE, GS, false, false, PW2>(q, G, s);
}

}  // namespace

// rows the tcgen05 sweep needs to fill the GPU (one 128-slot CTA per SM, >= 90 % of the SMs
// busy); fewer, longer rows (Netflix mode 2; order-4 10K^4: 10 K rows would fill 79 of 148 SMs,
// 38.2 vs 28.7 ms with quadr) keep the warp-level kernels
int64_t tc_min_rows() { return (int64_t)sm_count() * SLOTS * 9 / 10; }

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
  // the Fast2Sum residue when rows are long: 46 K serial updates drift ~1e-4 from fp64 in plain
  // fp32 (tests/test_netflix_parity_gpu.py); below 8 K per row the plain chain stays < 2e-5
  static const int force_comp = [] {  // FT_TC_COMP=0/1 forces the form (tests)
    const char *e = getenv("FT_TC_COMP");
    return e ? (strcmp(e, "0") == 0 ? 0 : 1) : -1;
  }();
  const bool comp = force_comp >= 0 ? force_comp == 1
                                    : t->num_rows > 0 && t->nnz / t->num_rows > 8192;
  if (t->slot_kb == 8) {  // few long rows, order 3 (slot_kb_for): 16 rows per CTA
    if (q.R == 32)
      return comp ? launch_tc_k<1, 4, true, true, 2, 8>(q, t->slot_grid, s)
                  : launch_tc_k<1, 4, true, false, 2, 8>(q, t->slot_grid, s);
    return comp ? launch_tc_k<1, 4, false, true, 2, 8>(q, t->slot_grid, s)
                : launch_tc_k<1, 4, false, false, 2, 8>(q, t->slot_grid, s);
  }
  if (t->slot_kb != 1) return -1;
  if (N == 3) return launch_tc_t<1, 4>(q, t->slot_grid, comp, s);
  return launch_tc_t<2, 2>(q, t->slot_grid, comp, s);
}

// ft_tree_slot_plan hands its per-leaf row-start flags to the ft_tree_slot_fill that follows
// (the Python driver calls them back to back on one thread)
int32_t *&planned_row_off() {
  static int32_t *p = nullptr;
  return p;
}
int &planned_kb() {
  static int kb = 1;
  return kb;
}
int &planned_maxnb() {
  static int m = 0;
  return m;
}

// which layout the factor sweep of this tree uses: 1 (K3c: one thread per row), 8 (K3c-wide:
// 16 rows per CTA, for few long rows) or 0 (neither: the warp-level kernels)
int slot_kb_for(const ft_tree_t *t, int J, int R) {
  const int64_t rows = t->num_rows;
  if (!t->row_leaf_ptr || !t->leaf_pc || rows <= 0 || !tc_enabled() ||
      !tc_shape_ok(t->order, J, R))
    return 0;
  if (rows >= tc_min_rows()) return 1;
  // K3c-wide (16 rows x 8 leaves per batch, the consumers transpose V through shared memory
  // and run the chains in the quad layout) is opt-in (FT_TC_WIDE=1): correct
  // (tests/test_factor_tc_gpu.py), but its consumers need ~3,000 cycles per batch (vs ~1,200
  // for K3c's production; shared-memory pipe contention) and it measured slower than quadw on
  // Netflix mode 2 (8.4 vs 6.0 ms; the earlier chain-warp form 9.6 ms;
  // profiles/r02_factor_tc_ab.md)
  static const bool wide = [] {
    const char *e = getenv("FT_TC_WIDE");
    return e && strcmp(e, "1") == 0;
  }();
  if (wide && t->order == 3 && rows >= (int64_t)sm_count() * (SLOTS / 8) * 9 / 10 &&
      t->nnz / rows >= 64)
    return 8;
  return 0;
}

}  // namespace ft

using namespace ft;

extern "C" int ft_tree_slot_plan(const ft_tree_t *tree, int32_t J, int32_t R, int32_t *grid_out,
                                 int32_t *kb_out, int32_t *batch_ptr, int64_t *len_out,
                                 void *stream) {
  if (!tree || !grid_out || !len_out || !kb_out)
    return fail(FT_ERR_ARG, "ft_tree_slot_plan: null argument");
  *grid_out = 0;
  *len_out = 0;
  const int KB = slot_kb_for(tree, J, R);
  *kb_out = KB;
  if (KB == 0) return FT_OK;  // the tcgen05 sweep does not apply: no layout
  const int64_t rows = tree->num_rows, RS = SLOTS / KB;
  const int64_t G64 = (rows + RS - 1) / RS;
  const int G = (int)(G64 < sm_count() ? G64 : sm_count());
  if (!batch_ptr) {  // size query
    *grid_out = G;
    return FT_OK;
  }
  cudaStream_t s = as_stream(stream);
  int32_t *nbatch = nullptr;
  FT_CUDA(cudaMallocAsync(&nbatch, sizeof(int32_t) * G, s));
  // row-start flags per leaf: scratch, handed to ft_tree_slot_fill
  uint8_t *rstart = nullptr;
  FT_CUDA(cudaMallocAsync(&rstart, (size_t)tree->nnz, s));
  FT_CUDA(cudaMemsetAsync(rstart, 0, (size_t)tree->nnz, s));
  row_start_kernel<<<(unsigned)((rows + 255) / 256), 256, 0, s>>>(tree->row_leaf_ptr, rows, rstart);
  if (int rc = check_launch("ft_tree_slot_plan(row starts)")) return rc;
  slot_rows_kernel<<<G, SLOTS, 0, s>>>(tree->row_leaf_ptr, rows, G, KB, nbatch);
  if (int rc = check_launch("ft_tree_slot_plan(rows)")) return rc;
  int32_t *tm = nullptr;
  FT_CUDA(cudaMallocAsync(&tm, 2 * sizeof(int32_t), s));
  slot_scan_kernel<<<1, 32, 0, s>>>(nbatch, G, batch_ptr, tm);
  if (int rc = check_launch("ft_tree_slot_plan(scan)")) return rc;
  int32_t host_tm[2] = {0, 0};
  FT_CUDA(cudaMemcpyAsync(host_tm, tm, sizeof(host_tm), cudaMemcpyDeviceToHost, s));
  FT_CUDA(cudaFreeAsync(nbatch, s));
  FT_CUDA(cudaFreeAsync(tm, s));
  FT_CUDA(cudaStreamSynchronize(s));
  const int32_t total = host_tm[0];
  planned_maxnb() = host_tm[1];
  if (planned_row_off()) cudaFreeAsync(planned_row_off(), s);  // a plan never followed by fill
  planned_row_off() = reinterpret_cast<int32_t *>(rstart);  // handed to ft_tree_slot_fill
  planned_kb() = KB;
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
  uint8_t *row_off = reinterpret_cast<uint8_t *>(planned_row_off());  // the row-start flags
  if (!row_off) return fail(FT_ERR_ARG, "ft_tree_slot_fill: call ft_tree_slot_plan first");
  planned_row_off() = nullptr;
  cudaStream_t s = as_stream(stream);
  const int KB = planned_kb();
  const int maxnb = planned_maxnb();  // the longest CTA stream bounds the batch blocks
  const dim3 g(grid, (maxnb + FILL_B - 1) / FILL_B);
  if (npre == 1) {
    static bool set1 = false;
    if (!set1) {
      cudaFuncSetAttribute(slot_fill_kernel<1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fill_smem_bytes<1>());
      set1 = true;
    }
    slot_fill_kernel<1><<<g, SLOTS, fill_smem_bytes<1>(), s>>>(
        tree->row_leaf_ptr, row_off, tree->num_rows, grid, KB, batch_ptr, tree->leaf_coord,
        tree->leaf_pc, tree->vals, slot_lc, slot_pc, slot_x);
  } else {
    static bool set2 = false;
    if (!set2) {
      cudaFuncSetAttribute(slot_fill_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)fill_smem_bytes<2>());
      set2 = true;
    }
    slot_fill_kernel<2><<<g, SLOTS, fill_smem_bytes<2>(), s>>>(
        tree->row_leaf_ptr, row_off, tree->num_rows, grid, KB, batch_ptr, tree->leaf_coord,
        tree->leaf_pc, tree->vals, slot_lc, slot_pc, slot_x);
  }
  const int rc = check_launch("ft_tree_slot_fill");
  cudaFreeAsync(row_off, s);
  return rc;
}
