// K3b "quad": the exact factor sweep with FOUR rows per warp over the leaf-major index.
// Included by sweep.cu inside namespace ft::<anon> (uses SweepParams, to_tf32, mma_tf32,
// ffma2, smem_u32, cp_async_wait_all).
//
// Same schedule and arithmetic contract as the other K3b kernels (sweep.cu header; reference
// factor_sweep, _ckern.pyx:132-199): every row of A_u is owned by one 8-lane quarter of a warp,
// which replays the row's updates in the reference's serial order
//     s = a . v,  e = x - s,  a <- a - lr (reg a - e v),   v = Bt_u^T (C_{u+1}[pc] * C_{u-1}[lc]).
// What is different (ncu on the two-rows-per-warp `dual` kernel: 40 warp instructions per leaf,
// of which ~26 % went to gather address arithmetic and the fiber-window ballot -> fiber_coord
// dependent loads, ~36 % to the 16-lane serial chain):
//   * operands come from the leaf-major index (ft_tree_leaf_index): leaf_pc[L] is the leaf's
//     prefix coordinate, row_leaf_ptr the row's leaf range, so a batch's per-leaf data are three
//     coalesced streaming loads, issued one batch ahead (next row's header one row ahead);
//   * a quarter owns a row (lane l holds columns 4l..4l+3), so one chain step advances FOUR rows
//     and its dot product reduces over 8 lanes (3 shuffle levels); the step's broadcast operands
//     (x, lr, -lr reg) come from one shared-memory float4, the decay and update run as FFMA2;
//   * gathers: lane (slot-in-4, float4 column) -> one shuffle + one wide IMAD + one LDGSTS per
//     16 B, no per-slot predicates (slots past a quarter's batch copy C row 0 and run as no-op
//     steps with lr = 0);
//   * V = cross * Bt_u on tensor cores (mma.sync m16n8k8, 3xTF32, two m16 tiles per 32-slot
//     batch) with the k index paired (MMA k-slot t <-> r = 2t, t+4 <-> r = 2t+1 within a k-tile)
//     so every A fragment pair is one LDS.64; the Bt_u fragments use the same pairing.
// Requirements (checked by the dispatcher): order 3, 16 < J <= 32, R <= 32 with R % 4 == 0,
// leaf-major index present.
namespace quad {
constexpr int QB = 8;                       // leaves per quarter batch
constexpr int XS = 40;                      // staging row stride (floats): 160-B rows; LDS.64
                                            // fragment loads / STS.64 V stores conflict-free
constexpr int TILE = 32 * XS;               // 32 slots
constexpr int MQ = 9;                       // meta float4 per quarter (8 + 1: disjoint banks)
constexpr int WARP_FLOATS = 2 * TILE + 4 * MQ * 4;
constexpr int WPB = 8;
constexpr int KT = 4, NT = 4;               // RP = JP = 32
constexpr int BFRAG_U4 = KT * NT * 32;
constexpr size_t bytes() { return (size_t)BFRAG_U4 * 16 + (size_t)WPB * WARP_FLOATS * 4; }
}  // namespace quad

__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  unsigned long long d;
  asm("mul.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}

__device__ __forceinline__ void cp_async16_s(uint32_t dst, const float *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

__global__ void __launch_bounds__(quad::WPB * 32, 2) factor_rows_quad_kernel(const SweepParams p) {
  using namespace quad;
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q = lane >> 3, l = lane & 7;    // quarter (row stream), lane in quarter
  const int gq = lane >> 2, tq = lane & 3;  // mma fragment coordinates
  uint4 *bfrag = reinterpret_cast<uint4 *>(smem4);
  float *X = reinterpret_cast<float *>(bfrag + BFRAG_U4) + w * quad::WARP_FLOATS;
  float *Y = X + TILE;
  float4 *meta = reinterpret_cast<float4 *>(Y + TILE);
  float *V = X;  // V = cross * Bt_u overwrites X once the fragments are read
  for (int k = lane; k < 2 * TILE; k += 32) X[k] = 0.f;  // Y's zero columns r >= R stay zero
  for (int f = threadIdx.x; f < BFRAG_U4; f += blockDim.x) {
    const int ll = f & 31, nt = (f >> 5) % NT, kt = (f >> 5) / NT;
    const int g = ll >> 2, t = ll & 3, j = 8 * nt + g;
    uint32_t hv[2], lv[2];
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int r = 8 * kt + 2 * t + hh;  // paired k order (see header)
      const float bv = (r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f;
      hv[hh] = to_tf32(bv);
      lv[hh] = to_tf32(bv - __uint_as_float(hv[hh]));
    }
    bfrag[f] = make_uint4(hv[0], hv[1], lv[0], lv[1]);
  }
  __syncthreads();

  const int64_t nstream = (int64_t)gridDim.x * quad::WPB * 4;
  int64_t row = ((int64_t)blockIdx.x * quad::WPB + w) * 4 + q;
  const int J = p.J;
  const bool j32 = J == 32;
  // current row (ci < 0: none) and the next row of this quarter's stream, one row ahead
  int ci = -1, cL0 = 0, cLe = 0, ni = -1, nLb = 0, nLe = 0;
  if (row < p.nrows) {
    ci = __ldg(p.row_coord + row);
    cL0 = __ldg(p.row_leaf_ptr + row);
    cLe = __ldg(p.row_leaf_ptr + row + 1);
  }
  if (row + nstream < p.nrows) {
    ni = __ldg(p.row_coord + row + nstream);
    nLb = __ldg(p.row_leaf_ptr + row + nstream);
    nLe = __ldg(p.row_leaf_ptr + row + nstream + 1);
  }
  float a[4] = {0.f, 0.f, 0.f, 0.f};
  auto load_row = [&](int i) {
    const float *ar = p.A + (int64_t)i * J;
    if (j32) {
      const float4 v = *reinterpret_cast<const float4 *>(ar + 4 * l);
      a[0] = v.x, a[1] = v.y, a[2] = v.z, a[3] = v.w;
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t) a[t] = 4 * l + t < J ? ar[4 * l + t] : 0.f;
    }
  };
  auto store_row = [&](int i) {
    float *ar = p.A + (int64_t)i * J;
    if (j32) {
      *reinterpret_cast<float4 *>(ar + 4 * l) = make_float4(a[0], a[1], a[2], a[3]);
    } else {
#pragma unroll
      for (int t = 0; t < 4; ++t)
        if (4 * l + t < J) ar[4 * l + t] = a[t];
    }
  };
  if (ci >= 0) load_row(ci);
  // leaf data of the batch about to run (prefetched one batch ahead; lanes past it: 0)
  int plc = 0, ppc = 0;
  float px = 0.f;
  if (ci >= 0 && cL0 + l < cLe) {
    plc = __ldcs(p.leaf_coord + cL0 + l);
    ppc = __ldcs(p.leaf_pc + cL0 + l);
    px = __ldcs(p.vals + cL0 + l);
  }
  const float lr = p.lr;
  // gather lanes: slot-in-4 and float4 column
  const int gc = lane & 7, gs = lane >> 3;
  const bool gok = gc < (p.R >> 2);
  const uint32_t xs0 = smem_u32(X + gs * XS + 4 * gc), ys0 = smem_u32(Y + gs * XS + 4 * gc);
  const float *cpre = p.Cpre[0] + 4 * gc, *cleaf = p.Cleaf + 4 * gc;
  const int64_t Rs = p.R;

  for (;;) {
    // ---- a quarter whose row is exhausted writes it back and moves to its next row ----
    if (ci >= 0 && cL0 >= cLe) {
      store_row(ci);
      row += nstream;
      ci = ni, cL0 = nLb, cLe = nLe;
      if (ci >= 0) {
        load_row(ci);  // consumed by the chain, after this batch's gathers and MMA
        const int64_t r2 = row + nstream;
        if (r2 < p.nrows) {
          ni = __ldg(p.row_coord + r2);
          nLb = __ldg(p.row_leaf_ptr + r2);
          nLe = __ldg(p.row_leaf_ptr + r2 + 1);
        } else {
          ni = -1;
        }
      }
    }
    if (!__any_sync(FULL, ci >= 0)) break;
    const int nb = ci >= 0 ? min(QB, cLe - cL0) : 0;
    const int lc = plc, pc = ppc;
    const float lrk = l < nb ? lr : 0.f;
    const float ck = -lrk * p.reg;
    meta[q * MQ + l] = make_float4(l < nb ? px : 0.f, lrk, ck, ck);
    {  // prefetch the next batch of this quarter (same row, or the next row's first leaves)
      const bool same = cL0 + nb < cLe;
      const int pos = same ? cL0 + nb : nLb, end = same ? cLe : nLe;
      const bool ok = ci >= 0 && (same || ni >= 0) && pos + l < end;
      plc = ok ? __ldcs(p.leaf_coord + pos + l) : 0;
      ppc = ok ? __ldcs(p.leaf_pc + pos + l) : 0;
      px = ok ? __ldcs(p.vals + pos + l) : 0.f;
    }
    // ---- gathers: slot s = 4 it + gs holds the leaf of lane s (quarter s / 8) ----
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int s = 4 * it + gs;
      const int pcs = __shfl_sync(FULL, pc, s), lcs = __shfl_sync(FULL, lc, s);
      if (gok) {
        cp_async16_s(xs0 + it * 4 * XS * 4, cpre + pcs * Rs);
        cp_async16_s(ys0 + it * 4 * XS * 4, cleaf + lcs * Rs);
      }
    }
    cp_async_wait_all();
    __syncwarp();
    // ---- V = (X * Y) * Bt_u: two m16 tiles (slots 0-15, 16-31), 3xTF32 ----
    float acc[2][NT][4];
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt)
#pragma unroll
        for (int t = 0; t < 4; ++t) acc[mt][nt][t] = 0.f;
#pragma unroll
    for (int kt = 0; kt < KT; ++kt) {
      uint32_t ah[2][4], al[2][4];
#pragma unroll
      for (int mt = 0; mt < 2; ++mt) {
        const int o0 = (16 * mt + gq) * XS + 8 * kt + 2 * tq, o1 = o0 + 8 * XS;
        const float2 x0 = *reinterpret_cast<const float2 *>(X + o0);
        const float2 x1 = *reinterpret_cast<const float2 *>(X + o1);
        const float2 y0 = *reinterpret_cast<const float2 *>(Y + o0);
        const float2 y1 = *reinterpret_cast<const float2 *>(Y + o1);
        const float2 c0 = fmul2(x0, y0), c1 = fmul2(x1, y1);
        // fragment order a0 = (gq, k=tq), a1 = (gq+8, tq), a2 = (gq, tq+4), a3 = (gq+8, tq+4)
        const float cv[4] = {c0.x, c1.x, c0.y, c1.y};
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          ah[mt][t] = to_tf32(cv[t]);
          al[mt][t] = to_tf32(cv[t] - __uint_as_float(ah[mt][t]));
        }
      }
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const uint4 bb = bfrag[(kt * NT + nt) * 32 + lane];
#pragma unroll
        for (int mt = 0; mt < 2; ++mt) {
          mma_tf32(acc[mt][nt], al[mt][0], al[mt][1], al[mt][2], al[mt][3], bb.x, bb.y);
          mma_tf32(acc[mt][nt], ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bb.z, bb.w);
          mma_tf32(acc[mt][nt], ah[mt][0], ah[mt][1], ah[mt][2], ah[mt][3], bb.x, bb.y);
        }
      }
    }
    __syncwarp();  // every lane's fragments are read before V overwrites X
#pragma unroll
    for (int mt = 0; mt < 2; ++mt)
#pragma unroll
      for (int nt = 0; nt < NT; ++nt) {
        const int o = (16 * mt + gq) * XS + 8 * nt + 2 * tq;
        *reinterpret_cast<float2 *>(V + o) = make_float2(acc[mt][nt][0], acc[mt][nt][1]);
        *reinterpret_cast<float2 *>(V + o + 8 * XS) = make_float2(acc[mt][nt][2], acc[mt][nt][3]);
      }
    __syncwarp();
    // ---- four serial chains (one per quarter): lane l holds columns 4l .. 4l+3 ----
    const int nbmax = __reduce_max_sync(FULL, (unsigned)nb);
    const float *Vq = V + 8 * q * XS + 4 * l;
    const float4 *mq = meta + q * MQ;
#pragma unroll
    for (int k = 0; k < QB; ++k) {
      if (k >= nbmax) break;
      const float4 v = *reinterpret_cast<const float4 *>(Vq + k * XS);
      float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(v.x, v.y));
      pr = ffma2(make_float2(a[2], a[3]), make_float2(v.z, v.w), pr);
      float s = pr.x + pr.y;
      s += __shfl_xor_sync(FULL, s, 4);
      s += __shfl_xor_sync(FULL, s, 2);
      s += __shfl_xor_sync(FULL, s, 1);
      const float4 m = mq[k];  // (x, lr, -lr reg, -lr reg); lr = 0 on padding steps
      const float e = m.x - s;
      const float lre = m.y * e;
      // a <- a + (-lr reg) a  (the decay, never through a rounded 1 - lr reg), then a += lr e v
      const float2 a01 = ffma2(make_float2(m.z, m.w), make_float2(a[0], a[1]), make_float2(a[0], a[1]));
      const float2 a23 = ffma2(make_float2(m.z, m.w), make_float2(a[2], a[3]), make_float2(a[2], a[3]));
      a[0] = __fmaf_rn(lre, v.x, a01.x);
      a[1] = __fmaf_rn(lre, v.y, a01.y);
      a[2] = __fmaf_rn(lre, v.z, a23.x);
      a[3] = __fmaf_rn(lre, v.w, a23.y);
    }
    __syncwarp();  // V / meta reads done before the next batch's gathers and meta stores
    cL0 += nb;
  }
}

int launch_quad(const SweepParams &q, cudaStream_t s) {
  const size_t sm = quad::bytes();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_quad_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sm);
    set = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_rows_quad_kernel,
                                                    quad::WPB * 32, sm) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = (q.nrows + 4 * quad::WPB - 1) / (4 * quad::WPB);
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  factor_rows_quad_kernel<<<(int)g, quad::WPB * 32, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(quad)");
}

bool quad_ok(const SweepParams &p) {
  return p.N == 3 && p.leaf_pc && p.row_leaf_ptr && p.J > 16 && p.J <= 32 && p.R <= 32 &&
         (p.R & 3) == 0;
}
