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
//   * the combine runs TRANSPOSED on tensor cores, V^T (J x 32 slots) = Bt_u^T (J x R) *
//     cross^T (R x 32), mma.sync m16n8k8 3xTF32: the constant Bt_u^T is the A operand (its hi /
//     lo fragments precomputed per block in shared memory) and the per-leaf cross rows are the
//     B operand, whose two registers per lane are exactly one LDS.64 pair of X, one of Y and
//     one FMUL2 when the k index is paired (MMA k-slot t <-> r = 2t, t+4 <-> r = 2t+1 within a
//     k-tile).  (With cross as the A operand the four-register fragment straddles two such
//     pairs and ptxas re-packs it with four MOVs per HMMA.)
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
constexpr int QVS = 36;                     // V tile row stride: conflict-free scalar stores
constexpr int KT = 4, MT = 2, NT = 4;       // k = r (32), m = j (32), n = slot (32)
constexpr int BFRAG_U4 = 2 * KT * MT * 32;  // Bt_u^T A fragments: hi and lo quads
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

template <int N>
__device__ __forceinline__ void cp_async_wait_group() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}
__device__ __forceinline__ void cp_async16_s(uint32_t dst, const float *src) {
  // .ca: the leaf-level C rows of a sweep are often a small matrix (Netflix C_2: 280 KB) that
  // stays L1-resident -- measured .cg (L2 only): core sweep modes 0/1 3.2 -> 4.2-4.6 ms
  asm volatile("cp.async.ca.shared.global [%0], [%1], 16;\n" ::"r"(dst), "l"(src));
}

// Bt_u^T as the A operand of the transposed combine: for (mt, kt, lane g t) the quad
// a0 = Bt[r][j], a1 = Bt[r][j+8], a2 = Bt[r+1][j], a3 = Bt[r+1][j+8], r = 8kt + 2t, j = 16mt + g
// (paired k order), as a hi quad and a lo quad (3xTF32 split).
// RL > 0 (quadr DIRECT): the k order r = RL t + 2 kt (+1), so that lane t's B values over all
// k-tiles are the RL consecutive columns RL t .. RL t + RL - 1 of its slots' rows (RL = 8 for
// R <= 32, 4 for the two-k-tile SMALL form) -- one or two LDG.128 per operand and slot.
template <int RL = 0>
__device__ __forceinline__ void quad_afrag_init(const SweepParams &p, uint4 *afr) {
  using namespace quad;
  for (int f = threadIdx.x; f < KT * MT * 32; f += blockDim.x) {
    const int ll = f & 31, kt = (f >> 5) % KT, mt = (f >> 5) / KT;
    const int g = ll >> 2, t = ll & 3;
    uint32_t hv[4], lv[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int r = (RL ? RL * t + 2 * kt : 8 * kt + 2 * t) + (e >> 1), j = 16 * mt + g + 8 * (e & 1);
      if (RL && 2 * kt >= RL) {  // k-tiles past the SMALL form's two: unused
        hv[e] = lv[e] = 0u;
        continue;
      }
      const float bv = (r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f;
      hv[e] = to_tf32(bv);
      lv[e] = to_tf32(bv - __uint_as_float(hv[e]));
    }
    afr[f] = make_uint4(hv[0], hv[1], hv[2], hv[3]);
    afr[KT * MT * 32 + f] = make_uint4(lv[0], lv[1], lv[2], lv[3]);
  }
}

// ... one lane's (kt, mt) quads straight into registers (quadw DB: no shared-memory copy)
__device__ __forceinline__ void quad_afrag_lane(const SweepParams &p, int kt, int mt, int ll,
                                                uint4 &ah, uint4 &al) {
  const int g = ll >> 2, t = ll & 3;
  uint32_t hv[4], lv[4];
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const int r = 8 * kt + 2 * t + (e >> 1), j = 16 * mt + g + 8 * (e & 1);
    const float bv = (r < p.R && j < p.J) ? __ldg(p.Bt + r * p.J + j) : 0.f;
    hv[e] = to_tf32(bv);
    lv[e] = to_tf32(bv - __uint_as_float(hv[e]));
  }
  ah = make_uint4(hv[0], hv[1], hv[2], hv[3]);
  al = make_uint4(lv[0], lv[1], lv[2], lv[3]);
}

// One k-tile of the transposed combine for n-tiles [nt0, nt0 + NN): acc[mt][nt] += Bt^T * cross^T,
// with the Bt^T fragments of this k-tile in registers.
template <int NN>
__device__ __forceinline__ void quad_mma_kt_r(const float *X, const float *Y, const uint4 (&ah)[2],
                                              const uint4 (&al)[2], int kt, int nt0, int lane,
                                              float (&acc)[2][4][4], int mts = 2) {
  using namespace quad;
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int nn = 0; nn < NN; ++nn) {
    const int nt = nt0 + nn;
    const int o = (8 * nt + gq) * XS + 8 * kt + 2 * tq;
    const float2 c = fmul2(*reinterpret_cast<const float2 *>(X + o),
                           *reinterpret_cast<const float2 *>(Y + o));
    const uint32_t bh0 = __float_as_uint(c.x), bh1 = __float_as_uint(c.y);  // the MMA truncates
    const uint32_t bl0 = __float_as_uint(c.x - __uint_as_float(to_tf32(c.x)));
    const uint32_t bl1 = __float_as_uint(c.y - __uint_as_float(to_tf32(c.y)));
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      if (mt >= mts) break;  // J <= 16: the second m-tile is all padding
      mma_tf32(acc[mt][nt], al[mt].x, al[mt].y, al[mt].z, al[mt].w, bh0, bh1);
      mma_tf32(acc[mt][nt], ah[mt].x, ah[mt].y, ah[mt].z, ah[mt].w, bl0, bl1);
      mma_tf32(acc[mt][nt], ah[mt].x, ah[mt].y, ah[mt].z, ah[mt].w, bh0, bh1);
    }
  }
}

// ... with the fragments read from the per-block shared-memory copy
template <int NN>
__device__ __forceinline__ void quad_mma_kt(const float *X, const float *Y, const uint4 *afr,
                                            int kt, int nt0, int lane, float (&acc)[2][4][4],
                                            int mts = 2) {
  using namespace quad;
  uint4 ah[MT], al[MT];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    ah[mt] = afr[(mt * KT + kt) * 32 + lane];
    al[mt] = afr[KT * MT * 32 + (mt * KT + kt) * 32 + lane];
  }
  quad_mma_kt_r<NN>(X, Y, ah, al, kt, nt0, lane, acc, mts);
}

// acc (V^T fragments) -> V[slot][j] (row stride QVS)
__device__ __forceinline__ void quad_store_v(float *V, const float (&acc)[2][4][4], int lane) {
  using namespace quad;
  const int gq = lane >> 2, tq = lane & 3;
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int nt = 0; nt < NT; ++nt) {
      float *v = V + (8 * nt + 2 * tq) * QVS + 16 * mt + gq;
      v[0] = acc[mt][nt][0];
      v[QVS] = acc[mt][nt][1];
      v[8] = acc[mt][nt][2];
      v[QVS + 8] = acc[mt][nt][3];
    }
}



__device__ __forceinline__ void quad_zero(float (&acc)[2][4][4]) {
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt)
#pragma unroll
      for (int u = 0; u < 4; ++u) acc[mt][nt][u] = 0.f;
}

// one serial step of a quarter's row: s = a . v (8 lanes x 4 columns), e = x - s,
// a <- a + (-lr reg) a  (the decay, never through a rounded 1 - lr reg), then a += lr e v
__device__ __forceinline__ void quad_chain_step_v(float (&a)[4], const float4 v, float4 m);
__device__ __forceinline__ void quad_chain_step(float (&a)[4], const float *vrow, float4 m) {
  quad_chain_step_v(a, *reinterpret_cast<const float4 *>(vrow), m);
}
__device__ __forceinline__ void quad_chain_step_v(float (&a)[4], const float4 v, float4 m) {
  float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(v.x, v.y));
  pr = ffma2(make_float2(a[2], a[3]), make_float2(v.z, v.w), pr);
  float s = pr.x + pr.y;
  s += __shfl_xor_sync(FULL, s, 4);
  s += __shfl_xor_sync(FULL, s, 2);
  s += __shfl_xor_sync(FULL, s, 1);
  const float e = m.x - s;  // m = (x, lr, -lr reg, -lr reg); lr = 0 on padding steps
  const float lre = m.y * e;
  const float2 a01 = ffma2(make_float2(m.z, m.w), make_float2(a[0], a[1]), make_float2(a[0], a[1]));
  const float2 a23 = ffma2(make_float2(m.z, m.w), make_float2(a[2], a[3]), make_float2(a[2], a[3]));
  a[0] = __fmaf_rn(lre, v.x, a01.x);
  a[1] = __fmaf_rn(lre, v.y, a01.y);
  a[2] = __fmaf_rn(lre, v.z, a23.x);
  a[3] = __fmaf_rn(lre, v.w, a23.y);
}

__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  unsigned long long d;
  asm("add.rn.f32x2 %0, %1, %2;"
      : "=l"(d)
      : "l"(*reinterpret_cast<unsigned long long *>(&a)),
        "l"(*reinterpret_cast<unsigned long long *>(&b)));
  return *reinterpret_cast<float2 *>(&d);
}
__device__ __forceinline__ float2 fsub2(float2 a, float2 b) {
  return fadd2(a, make_float2(-b.x, -b.y));
}

// The same step with a COMPENSATED row: a (the fp32 row the dot products use) plus lo, the
// rounding residue of every row update so far (Fast2Sum: the increment d is ~1e-4 of |a|).
// The increment d = (-lr reg) a + lr e v + lo folds the residue back in, so a stays the
// correctly rounded value of the exact fp32-increment sum.  Rows with tens of thousands of
// serial updates (Netflix mode 2: 45 K) otherwise drift ~1e-4 from the fp64 reference
// (tests/test_netflix_parity_gpu.py); the residue costs two packed adds per column pair, off
// the serial dependency except one FADD.
// a . v over a quarter (8 lanes x 4 columns): lane partial, 3-level butterfly
__device__ __forceinline__ float quad_dot(const float (&a)[4], const float4 v) {
  float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(v.x, v.y));
  pr = ffma2(make_float2(a[2], a[3]), make_float2(v.z, v.w), pr);
  float s = pr.x + pr.y;
  s += __shfl_xor_sync(FULL, s, 4);
  s += __shfl_xor_sync(FULL, s, 2);
  s += __shfl_xor_sync(FULL, s, 1);
  return s;
}
// the compensated row update of quad_chain_step_vc for a given error e
__device__ __forceinline__ void quad_update_c(float (&a)[4], float (&lo)[4], const float4 v,
                                              float4 m, float e) {
  const float2 l2 = make_float2(m.y * e, m.y * e), c2 = make_float2(m.z, m.w);
  const float2 a01 = make_float2(a[0], a[1]), a23 = make_float2(a[2], a[3]);
  const float2 d01 = ffma2(l2, make_float2(v.x, v.y), ffma2(c2, a01, make_float2(lo[0], lo[1])));
  const float2 d23 = ffma2(l2, make_float2(v.z, v.w), ffma2(c2, a23, make_float2(lo[2], lo[3])));
  const float2 t01 = fadd2(a01, d01), t23 = fadd2(a23, d23);
  const float2 r01 = fsub2(d01, fsub2(t01, a01)), r23 = fsub2(d23, fsub2(t23, a23));
  a[0] = t01.x, a[1] = t01.y, a[2] = t23.x, a[3] = t23.y;
  lo[0] = r01.x, lo[1] = r01.y, lo[2] = r23.x, lo[3] = r23.y;
}

// One quarter batch (QB consecutive updates of one row) with ONE STEP OF LOOKAHEAD.  With
// a_{k+1} = a_k + c_k a_k + lr_k e_k v_k (c_k = -lr_k reg; padding steps lr = c = 0),
//     a_k . v_k = (1 + c_{k-1}) (a_{k-1} . v_k) + lr_{k-1} e_{k-1} (v_{k-1} . v_k),
// so the butterfly for step k+1's dot p_{k+1} = a_k . v_{k+1} starts as soon as a_k exists, i.e.
// while e_k is still being formed, and e_k = x_k - (1 + c_{k-1}) p_k - lr_{k-1} g_k e_{k-1} is
// two FMAs after e_{k-1} (g_k = v_{k-1} . v_k: independent of the row, reduced up front).  The
// serial path per step drops from dot + butterfly + update to about half of it (the butterfly
// of one step overlaps the FMAs and update of the previous one).  Exact algebra, the reference's
// order of updates; the batch's first step takes the direct dot (no state crosses batches).
__device__ __forceinline__ void quad_batch_lookahead(float (&a)[4], float (&lo)[4],
                                                     const float4 (&vv)[quad::QB],
                                                     const float4 (&mm)[quad::QB]) {
  using quad::QB;
  float g[QB];  // g[k] = v_{k-1} . v_k (k >= 1)
#pragma unroll
  for (int k = 1; k < QB; ++k) {
    float2 pr = fmul2(make_float2(vv[k - 1].x, vv[k - 1].y), make_float2(vv[k].x, vv[k].y));
    pr = ffma2(make_float2(vv[k - 1].z, vv[k - 1].w), make_float2(vv[k].z, vv[k].w), pr);
    g[k] = pr.x + pr.y;
  }
#pragma unroll
  for (int msk = 4; msk >= 1; msk >>= 1)
#pragma unroll
    for (int k = 1; k < QB; ++k) g[k] += __shfl_xor_sync(FULL, g[k], msk);
  float p = quad_dot(a, vv[0]);
  float e_prev = 0.f, lg = 0.f, cprev = 0.f;
#pragma unroll
  for (int k = 0; k < QB; ++k) {
    const float pn = k + 1 < QB ? quad_dot(a, vv[k + 1]) : 0.f;  // a = a_k (before the update)
    const float ap = __fmaf_rn(cprev, p, p);
    const float e = __fmaf_rn(-lg, e_prev, mm[k].x - ap);
    quad_update_c(a, lo, vv[k], mm[k], e);
    if (k + 1 < QB) lg = mm[k].y * g[k + 1];
    cprev = mm[k].z, e_prev = e, p = pn;
  }
}

__device__ __forceinline__ void quad_chain_step_vc(float (&a)[4], float (&lo)[4], const float4 v,
                                                   float4 m) {
  float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(v.x, v.y));
  pr = ffma2(make_float2(a[2], a[3]), make_float2(v.z, v.w), pr);
  float s = pr.x + pr.y;
  s += __shfl_xor_sync(FULL, s, 4);
  s += __shfl_xor_sync(FULL, s, 2);
  s += __shfl_xor_sync(FULL, s, 1);
  const float e = m.x - s;  // m = (x, lr, -lr reg, -lr reg); lr = 0 on padding steps
  const float2 l2 = make_float2(m.y * e, m.y * e), c2 = make_float2(m.z, m.w);
  const float2 a01 = make_float2(a[0], a[1]), a23 = make_float2(a[2], a[3]);
  const float2 d01 = ffma2(l2, make_float2(v.x, v.y), ffma2(c2, a01, make_float2(lo[0], lo[1])));
  const float2 d23 = ffma2(l2, make_float2(v.z, v.w), ffma2(c2, a23, make_float2(lo[2], lo[3])));
  const float2 t01 = fadd2(a01, d01), t23 = fadd2(a23, d23);
  const float2 r01 = fsub2(d01, fsub2(t01, a01)), r23 = fsub2(d23, fsub2(t23, a23));
  a[0] = t01.x, a[1] = t01.y, a[2] = t23.x, a[3] = t23.y;
  lo[0] = r01.x, lo[1] = r01.y, lo[2] = r23.x, lo[3] = r23.y;
}


// Order-N gathers into a warp's 32-slot X / Y tiles (row stride XSD floats): X <- prod over the
// NPRE prefix levels of C_pre[d][pc_d] (gather, wait, multiply in place, level by level -- the
// reference's left-to-right chain), Y <- C_leaf[lc].  pc[d] / lc: lane s holds slot s's
// coordinates (0 for padding slots).  Returns with both tiles complete (cp.async waited).
template <int NPRE, int XSD>
__device__ __forceinline__ void quad_gather(const SweepParams &p, float *X, float *Y,
                                            const int (&pc)[NPRE], int lc, int lane) {
  const int gc = lane & 7, gs = lane >> 3;
  const bool gok = gc < (p.R >> 2);
  const int64_t Rs = p.R;
  const uint32_t xs0 = smem_u32(X + gs * XSD + 4 * gc), ys0 = smem_u32(Y + gs * XSD + 4 * gc);
  auto issue = [&](uint32_t dst0, const float *C, int coord) {
#pragma unroll
    for (int it = 0; it < 8; ++it) {
      const int cs = __shfl_sync(FULL, coord, 4 * it + gs);
      if (gok) cp_async16_s(dst0 + it * 4 * XSD * 4, C + 4 * gc + cs * Rs);
    }
  };
  auto fold = [&]() {  // lane = slot: X[s] *= Y[s]
    float4 *xr = reinterpret_cast<float4 *>(X + lane * XSD);
    const float4 *yr = reinterpret_cast<const float4 *>(Y + lane * XSD);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
      const float4 x = xr[c], y = yr[c];
      const float2 a = fmul2(make_float2(x.x, x.y), make_float2(y.x, y.y));
      const float2 b = fmul2(make_float2(x.z, x.w), make_float2(y.z, y.w));
      xr[c] = make_float4(a.x, a.y, b.x, b.y);
    }
  };
  issue(xs0, p.Cpre[0], pc[0]);
  if (NPRE == 1) {
    issue(ys0, p.Cleaf, lc);
    cp_async_wait_all();
    __syncwarp();
    return;
  }
#pragma unroll
  for (int d = 1; d < NPRE; ++d) {
    issue(ys0, p.Cpre[d], pc[d]);
    cp_async_wait_all();
    __syncwarp();
    fold();
    __syncwarp();
  }
  issue(ys0, p.Cleaf, lc);
  cp_async_wait_all();
  __syncwarp();
}

// ---- K3b "quadr": quad with the combine's output consumed straight from the MMA registers --
// quad stages V through shared memory to turn the Vᵀ fragments into lanes-over-columns rows
// (32 STS + 8 LDS.128 per batch on an L1 / shared-memory pipe that ncu shows at 84-88 %).
// quadr instead places each row's leaves on the MMA's n-slots so that the fragment layout IS the
// chain layout: row rho (0..3) of a warp lives in the 8 lanes 4 gq + rho (gq = 0..7), each
// holding columns j = gq, gq+8, gq+16, gq+24; leaf k of its batch is slot 8 (k/2) + 2 rho + (k&1),
// whose Vᵀ column lands exactly in those lanes' accumulators (d0/d2 for even k, d1/d3 for odd).
// The dot product reduces over lane bits 2-4 (xor 4, 8, 16).  Same arithmetic, order and
// gathers as quad; row streams rho are numbered block-fastest.
#ifndef QUADR_FULL8
#define QUADR_FULL8 1  // always run 8 chain steps (padding steps are no-ops): no break, loads hoist
#endif
// quadr DIRECT: the transposed combine fed straight from global memory.  Lane (g, t) loads,
// for each n-tile nt (slot 8 nt + g: row (g >> 1) & 3, leaf 2 nt + (g & 1)), the RL columns
// RL t .. RL t + RL - 1 of the slot's prefix row(s) and leaf row (LDG.128 through L1; the
// C matrices are read-only during the sweep), forms cross = X * Y in registers (the prefix
// chain left to right, as quad_gather) and runs the 3xTF32 MMAs with the RL-permuted k order
// (quad_afrag_init<RL>) -- no cp.async write, no LDS per fragment.  Padding slots load nothing
// (cross = 0: their V is 0 and their chain steps are no-ops).
template <bool SMALL, int NPRE>
__device__ __forceinline__ void quadr_direct_combine(const SweepParams &p, const int (&pc)[NPRE],
                                                     int lc, int nb, int lane, const uint4 *afr,
                                                     float (&acc)[2][4][4]) {
  using namespace quad;
  constexpr int RL = SMALL ? 4 : 8, NC = RL / 4, nkt = SMALL ? 2 : 4, mts = SMALL ? 1 : 2;
  const int gq = lane >> 2, tq = lane & 3;
  const int r2 = (gq >> 1) & 3;
  const int rnb = __shfl_sync(FULL, nb, r2);  // chain layout: lane rho holds row rho's nb
  const int64_t Rs = p.R;
#pragma unroll
  for (int nt = 0; nt < NT; ++nt) {
    const int sl = 8 * nt + gq;
    // slot-layout lane sl holds slot sl's coordinates
    const int cy = __shfl_sync(FULL, lc, sl);
    int cx[NPRE];
#pragma unroll
    for (int d = 0; d < NPRE; ++d) cx[d] = __shfl_sync(FULL, pc[d], sl);
    const bool ok = 2 * nt + (gq & 1) < rnb;
    float c[RL];
#pragma unroll
    for (int h = 0; h < NC; ++h) {
      const int r0 = RL * tq + 4 * h;
      float4 xv = make_float4(0.f, 0.f, 0.f, 0.f), yv = xv;
      if (ok && r0 < p.R) {
        float4 lv[NPRE];
#pragma unroll
        for (int d = 0; d < NPRE; ++d)
          lv[d] = __ldg(reinterpret_cast<const float4 *>(p.Cpre[d] + cx[d] * Rs + r0));
        yv = __ldg(reinterpret_cast<const float4 *>(p.Cleaf + cy * Rs + r0));
        xv = lv[0];
#pragma unroll
        for (int d = 1; d < NPRE; ++d) {
          const float2 a = fmul2(make_float2(xv.x, xv.y), make_float2(lv[d].x, lv[d].y));
          const float2 b = fmul2(make_float2(xv.z, xv.w), make_float2(lv[d].z, lv[d].w));
          xv = make_float4(a.x, a.y, b.x, b.y);
        }
      }
      const float2 a = fmul2(make_float2(xv.x, xv.y), make_float2(yv.x, yv.y));
      const float2 b = fmul2(make_float2(xv.z, xv.w), make_float2(yv.z, yv.w));
      c[4 * h] = a.x, c[4 * h + 1] = a.y, c[4 * h + 2] = b.x, c[4 * h + 3] = b.y;
    }
#pragma unroll
    for (int kt = 0; kt < nkt; ++kt) {
      const float c0 = c[2 * kt], c1 = c[2 * kt + 1];
      const uint32_t bh0 = __float_as_uint(c0), bh1 = __float_as_uint(c1);
      const uint32_t bl0 = __float_as_uint(c0 - __uint_as_float(to_tf32(c0)));
      const uint32_t bl1 = __float_as_uint(c1 - __uint_as_float(to_tf32(c1)));
#pragma unroll
      for (int mt = 0; mt < mts; ++mt) {
        const uint4 ah = afr[(mt * KT + kt) * 32 + lane];
        const uint4 al = afr[KT * MT * 32 + (mt * KT + kt) * 32 + lane];
        mma_tf32(acc[mt][nt], al.x, al.y, al.z, al.w, bh0, bh1);
        mma_tf32(acc[mt][nt], ah.x, ah.y, ah.z, ah.w, bl0, bl1);
        mma_tf32(acc[mt][nt], ah.x, ah.y, ah.z, ah.w, bh0, bh1);
      }
    }
  }
}

constexpr int QR_META = 4 * quad::MQ;  // float4 step operands per warp (4 rows x MQ)
template <bool SMALL, int NPRE, int WPBT>
__global__ void __launch_bounds__(WPBT * 32, 2) factor_rows_quadr_kernel(const SweepParams p) {
  using namespace quad;
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int rho = lane & 3, gq = lane >> 2;      // chain layout: row, column group
  const int srho = (lane >> 1) & 3;              // slot layout: lane s holds slot s = leaf
  const int sk = 2 * (lane >> 3) + (lane & 1);   //   sk of row srho
  uint4 *afr = reinterpret_cast<uint4 *>(smem4);
  // shared memory: the Bt^T fragments and each warp's step operands only -- the direct combine
  // stages nothing, so the rest of the SM's 256 KB serves the gathered C rows as L1
  float4 *meta = reinterpret_cast<float4 *>(afr + BFRAG_U4) + w * QR_META;
  quad_afrag_init<SMALL ? 4 : 8>(p, afr);
  __syncthreads();

  const int64_t nstream = (int64_t)gridDim.x * WPBT * 4;
  int64_t row = (int64_t)(4 * w + rho) * gridDim.x + blockIdx.x;
  const int J = p.J;
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
  float a[4] = {0.f, 0.f, 0.f, 0.f};  // columns gq, gq+8, gq+16, gq+24
  auto load_row = [&](int i) {
    const float *ar = p.A + (int64_t)i * J;
#pragma unroll
    for (int m = 0; m < 4; ++m) a[m] = gq + 8 * m < J ? ar[gq + 8 * m] : 0.f;
  };
  auto store_row = [&](int i) {
    float *ar = p.A + (int64_t)i * J;
#pragma unroll
    for (int m = 0; m < 4; ++m)
      if (gq + 8 * m < J) ar[gq + 8 * m] = a[m];
  };
  if (ci >= 0) load_row(ci);
  // leaf data of slot `lane` for the batch about to run (prefetched one batch ahead)
  int plc = 0, ppc[NPRE];
  float px = 0.f;
#pragma unroll
  for (int d = 0; d < NPRE; ++d) ppc[d] = 0;
  {
    const int sci = __shfl_sync(FULL, ci, srho), s0 = __shfl_sync(FULL, cL0, srho),
              se = __shfl_sync(FULL, cLe, srho);
    if (sci >= 0 && s0 + sk < se) {
      plc = __ldcs(p.leaf_coord + s0 + sk);
#pragma unroll
      for (int d = 0; d < NPRE; ++d) ppc[d] = __ldcs(p.leaf_pc + (int64_t)(s0 + sk) * NPRE + d);
      px = __ldcs(p.vals + s0 + sk);
    }
  }
  const float lr = p.lr;

  for (;;) {
    if (ci >= 0 && cL0 >= cLe) {
      store_row(ci);
      row += nstream;
      ci = ni, cL0 = nLb, cLe = nLe;
      if (ci >= 0) {
        load_row(ci);
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
    // the slot-layout view of this lane's row (srho)
    const int snb = __shfl_sync(FULL, nb, srho);
    const int lc = plc;
    int pc[NPRE];
#pragma unroll
    for (int d = 0; d < NPRE; ++d) pc[d] = ppc[d];
    {
      const float lrk = sk < snb ? lr : 0.f;
      const float ck = -lrk * p.reg;
      meta[srho * MQ + sk] = make_float4(sk < snb ? px : 0.f, lrk, ck, ck);
    }
    {  // prefetch the next batch of row srho (same row, or the next row's first leaves)
      const bool same = cL0 + nb < cLe;
      const int pos_r = same ? cL0 + nb : nLb, end_r = same ? cLe : nLe;
      const bool ok_r = ci >= 0 && (same || ni >= 0);
      const int pos = __shfl_sync(FULL, pos_r, srho), end = __shfl_sync(FULL, end_r, srho);
      const bool ok = __shfl_sync(FULL, (int)ok_r, srho) && pos + sk < end;
      plc = ok ? __ldcs(p.leaf_coord + pos + sk) : 0;
#pragma unroll
      for (int d = 0; d < NPRE; ++d)
        ppc[d] = ok ? __ldcs(p.leaf_pc + (int64_t)(pos + sk) * NPRE + d) : 0;
      px = ok ? __ldcs(p.vals + pos + sk) : 0.f;
    }
    float acc[2][4][4];
    quad_zero(acc);
    quadr_direct_combine<SMALL, NPRE>(p, pc, lc, nb, lane, afr, acc);
    __syncwarp();  // meta visible (its stores precede the gathers' waits)
    // ---- four serial chains on the accumulator registers ----
    const int nbmax = QUADR_FULL8 ? QB : __reduce_max_sync(FULL, (unsigned)nb);
    const float4 *mq = meta + rho * MQ;
#pragma unroll
    for (int k = 0; k < QB; ++k) {
      if (k >= nbmax) break;
      const int nt = k >> 1, o = k & 1;
      const float v0 = acc[0][nt][o], v1 = acc[0][nt][2 + o];
      const float v2 = SMALL ? 0.f : acc[1][nt][o], v3 = SMALL ? 0.f : acc[1][nt][2 + o];
      float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(v0, v1));
      pr = ffma2(make_float2(a[2], a[3]), make_float2(v2, v3), pr);
      float sv = pr.x + pr.y;
      sv += __shfl_xor_sync(FULL, sv, 4);
      sv += __shfl_xor_sync(FULL, sv, 8);
      sv += __shfl_xor_sync(FULL, sv, 16);
      const float4 m = mq[k];  // (x, lr, -lr reg, -lr reg); lr = 0 on padding steps
      const float e = m.x - sv;
      const float lre = m.y * e;
      const float2 a01 = ffma2(make_float2(m.z, m.w), make_float2(a[0], a[1]), make_float2(a[0], a[1]));
      const float2 a23 = ffma2(make_float2(m.z, m.w), make_float2(a[2], a[3]), make_float2(a[2], a[3]));
      a[0] = __fmaf_rn(lre, v0, a01.x);
      a[1] = __fmaf_rn(lre, v1, a01.y);
      a[2] = __fmaf_rn(lre, v2, a23.x);
      a[3] = __fmaf_rn(lre, v3, a23.y);
    }
    __syncwarp();  // meta / tiles read before the next batch's stores and gathers
    cL0 += nb;
  }
}

template <bool SMALL, int NPRE, int WPBT>
int launch_quadr_t(const SweepParams &q, cudaStream_t s) {
  const size_t sm = (size_t)quad::BFRAG_U4 * 16 + (size_t)WPBT * QR_META * 16;
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(factor_rows_quadr_kernel<SMALL, NPRE, WPBT>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    // two blocks x ~13 KB: the smallest carveout, the rest L1 for the gathered rows
    cudaFuncSetAttribute(factor_rows_quadr_kernel<SMALL, NPRE, WPBT>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 15);
    set = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_rows_quadr_kernel<SMALL, NPRE, WPBT>,
                                                    WPBT * 32, sm) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = (q.nrows + 4 * WPBT - 1) / (4 * WPBT);
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  factor_rows_quadr_kernel<SMALL, NPRE, WPBT><<<(int)g, WPBT * 32, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(quadr)");
}

// 8 warps per block (128 registers, a 16-B spill) at order 3; at order 4 (two prefix rows per
// slot) 6 warps at 162-168 registers, no spill (order-4 10K^4: 33.0 -> 28.7 ms per mode)
int launch_quadr(const SweepParams &q, cudaStream_t s) {
  const bool small = q.J <= 16 && q.R <= 16;
  if (small)
    return q.N == 4 ? launch_quadr_t<true, 2, quad::WPB>(q, s) : launch_quadr_t<true, 1, quad::WPB>(q, s);
  return q.N == 4 ? launch_quadr_t<false, 2, 6>(q, s) : launch_quadr_t<false, 1, quad::WPB>(q, s);
}

// Row-stream cursor and per-batch records shared by the quadw producers.
namespace quadp {
constexpr int WPB = 4;
constexpr int WARP_FLOATS = 5 * quad::TILE + 4 * quad::MQ * 4;  // X[2], Y[2], V, meta
constexpr size_t bytes() { return (size_t)quad::BFRAG_U4 * 16 + (size_t)WPB * WARP_FLOATS * 4; }

struct Cursor {   // a quarter's position in its row stream (replicated in its 8 lanes)
  int64_t row;    // current row (stream index)
  int i, L0, Le;  // current row coordinate (-1: none) and remaining leaf range
  int ni, nLb, nLe;  // the stream's next row, loaded one row ahead (ni < 0: none)
};
struct Rec {      // one quarter batch
  int nb, i, L0;
  bool newrow;    // first batch of row i
};

__device__ __forceinline__ void load_row_info(const SweepParams &p, int64_t r, int &i, int &lb,
                                              int &le) {
  if (r < p.nrows) {
    i = __ldg(p.row_coord + r);
    lb = __ldg(p.row_leaf_ptr + r);
    le = __ldg(p.row_leaf_ptr + r + 1);
  } else {
    i = -1, lb = le = 0;
  }
}

__device__ __forceinline__ Rec next_batch(const SweepParams &p, Cursor &c, int64_t nstream) {
  Rec r;
  r.newrow = false;
  if (c.L0 >= c.Le) {
    if (c.ni < 0) {
      r.nb = 0, r.i = -1, r.L0 = 0;
      c.i = -1;
      return r;
    }
    c.row += nstream;
    c.i = c.ni, c.L0 = c.nLb, c.Le = c.nLe;
    r.newrow = true;
    load_row_info(p, c.row + nstream, c.ni, c.nLb, c.nLe);
  }
  r.i = c.i, r.L0 = c.L0, r.nb = min(quad::QB, c.Le - c.L0);
  c.L0 += r.nb;
  return r;
}

template <int NPRE>
struct Leaf {
  int lc, pc[NPRE];
  float x;
};
template <int NPRE>
__device__ __forceinline__ Leaf<NPRE> load_leaf(const SweepParams &p, const Rec &r, int l) {
  Leaf<NPRE> d;
  d.lc = 0, d.x = 0.f;
#pragma unroll
  for (int k = 0; k < NPRE; ++k) d.pc[k] = 0;
  if (l < r.nb) {
    d.lc = __ldcs(p.leaf_coord + r.L0 + l);
#pragma unroll
    for (int k = 0; k < NPRE; ++k) d.pc[k] = __ldcs(p.leaf_pc + (int64_t)(r.L0 + l) * NPRE + k);
    d.x = __ldcs(p.vals + r.L0 + l);
  }
  return d;
}
}  // namespace quadp

// ---- K3b "quadw": the quad layout warp-specialised for FEW LONG ROWS ----------------------
// A warp GROUP owns four rows (one per 8-lane quarter of its consumer warp).  NP PRODUCER warps
// take batches round robin: each walks the rows' batch records, gathers its batch into its own
// X/Y tiles, runs the transposed 3xTF32 combine and publishes V, the batch's (x, lr, -lr reg)
// and, when a quarter starts a row, that row's A values (loaded a batch ahead) into an NS-stage
// shared-memory ring (mbarrier full / empty).  The CONSUMER warp only runs the four serial
// chains, so the chain -- the only serial work -- never waits on a gather or an MMA.
// Netflix mode 2: 2,182 rows of ~45 K updates -> 546 groups, ~3.7 per SM.
//
// GRAM (the segment form of the row recurrence): a quarter batch is 8
// consecutive updates of ONE row (batches never span rows), and with alpha = 1 - lr reg
//     a_k = alpha^k a_0 + sum_{i<k} lr alpha^(k-1-i) e_i v_i,
//     e_k = x_k - alpha^k (a_0 . v_k) - sum_{i<k} T_ik e_i,   T_ik = lr alpha^(k-1-i) (v_i . v_k),
//     a_8 = alpha^8 a_0 + sum_i lr alpha^(7-i) e_i v_i
// (exact algebra; padding steps have lr = 0).  The producers add the batch's four 8 x 8 Gram
// blocks V_q V_q^T (mma.sync 3xTF32, the diagonal blocks of two m-tiles) and store T; the
// consumer reduces the eight dots a_0 . v_k in ONE 3-level butterfly (instead of one per step),
// solves the 8 x 8 unit-triangular system in registers (28 FMAs, no communication) and updates
// a once per batch (compensated).  The serial dependency per batch drops from 8 x (dot +
// 3 shuffles + update) to one butterfly + 7 FMAs: what bounds the sweep when few rows share an
// SM (the row-sharded multi-GPU epoch) -- tools/time_shards.py.
namespace quadw {
// DB: the double-buffered per-step form (order 3): two X / Y tile pairs per producer, a 2-stage
// ring, the Bt^T fragments built straight into registers (no shared-memory copy)
template <int NP, bool DB = false>
struct Cfg {
  static constexpr int NS = DB ? 2 : NP <= 2 ? 4 : 2 * NP;  // ring stages (producer k writes k, k + NP, ..)
  static constexpr int VREG = 32 * quad::QVS + 32;  // V tile
  // stage: V [32][QVS] | meta float4 [4][MQ] | info int4 [4] | A rows [4][32] |
  //        GRAM: per quarter T [28] + x [8] + pad [4]
  static constexpr int META = VREG, INFO = META + 4 * quad::MQ * 4, AROW = INFO + 16,
                       TCOEF = AROW + 4 * 32, TQ = 40;
  static constexpr int STAGE_FLOATS = TCOEF + 4 * TQ;
  // ring + X, Y per producer (two pairs when DB)
  static constexpr int XY_FLOATS = (DB ? 4 : 2) * quad::TILE;
  static constexpr int GROUP_FLOATS = NS * STAGE_FLOATS + NP * XY_FLOATS;
  static constexpr int BAR_BYTES = 2 * NS * 8 + 16;
  static constexpr int FRAG_BYTES = DB ? 0 : quad::BFRAG_U4 * 16;
  static constexpr int THREADS = (NP + 1) * 32;
  static constexpr size_t bytes() {
    return (size_t)FRAG_BYTES + BAR_BYTES + (size_t)GROUP_FLOATS * 4;
  }
};
// position of T_ik (i < k) in a quarter's packed 28-float block: rows i = 0..6, columns k > i
__host__ __device__ constexpr int tpos(int i, int k) { return 7 * i - i * (i - 1) / 2 + (k - i - 1); }
}  // namespace quadw

// The batch's four diagonal Gram blocks G_q = V_q V_q^T (8 x 8, q = quarter) from the stage's V
// tile by mma.sync 3xTF32, scaled into the consumer's T coefficients (packed, quadw::tpos):
// m-tile h = quarters 2h, 2h + 1 (16 slots) times n-tile = one quarter's 8 slots, so the
// diagonal blocks are rows 0-7 of (h, 2h) and rows 8-15 of (h, 2h + 1); k order paired as in the
// combine (k-slot t <-> j = 2t, t + 4 <-> 2t + 1): every fragment register pair is one LDS.64.
// Lane (g, t) ends with G_q[g][2t], G_q[g][2t + 1]; tc0 / tc1 = lr alpha^(k-1-i) for those two
// entries (lane constants), nb[q] the quarters' live batch lengths (T = 0 for padding rows i).
template <bool SMALL>
__device__ __forceinline__ void quadw_gram(const float *V, float *T, const int (&nb)[4], float tc0,
                                           float tc1, int lane) {
  using namespace quad;
  const int gq = lane >> 2, tq = lane & 3;
  float ga[2][2][4];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int nn = 0; nn < 2; ++nn)
#pragma unroll
      for (int u = 0; u < 4; ++u) ga[h][nn][u] = 0.f;
#pragma unroll
  for (int ks = 0; ks < 4; ++ks) {
    if (SMALL && ks >= 2) break;  // J <= 16: columns 16.. are zero
    float2 bq[4];
#pragma unroll
    for (int n = 0; n < 4; ++n)
      bq[n] = *reinterpret_cast<const float2 *>(V + (8 * n + gq) * QVS + 8 * ks + 2 * tq);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const float2 r0v = *reinterpret_cast<const float2 *>(V + (16 * h + gq) * QVS + 8 * ks + 2 * tq);
      const float2 r1v = *reinterpret_cast<const float2 *>(V + (16 * h + gq + 8) * QVS + 8 * ks + 2 * tq);
      const uint32_t ah0 = __float_as_uint(r0v.x), ah1 = __float_as_uint(r1v.x),
                     ah2 = __float_as_uint(r0v.y), ah3 = __float_as_uint(r1v.y);  // MMA truncates
      const uint32_t al0 = __float_as_uint(r0v.x - __uint_as_float(to_tf32(r0v.x)));
      const uint32_t al1 = __float_as_uint(r1v.x - __uint_as_float(to_tf32(r1v.x)));
      const uint32_t al2 = __float_as_uint(r0v.y - __uint_as_float(to_tf32(r0v.y)));
      const uint32_t al3 = __float_as_uint(r1v.y - __uint_as_float(to_tf32(r1v.y)));
#pragma unroll
      for (int nn = 0; nn < 2; ++nn) {
        const float2 bv = bq[2 * h + nn];
        const uint32_t bh0 = __float_as_uint(bv.x), bh1 = __float_as_uint(bv.y);
        const uint32_t bl0 = __float_as_uint(bv.x - __uint_as_float(to_tf32(bv.x)));
        const uint32_t bl1 = __float_as_uint(bv.y - __uint_as_float(to_tf32(bv.y)));
        mma_tf32(ga[h][nn], al0, al1, al2, al3, bh0, bh1);
        mma_tf32(ga[h][nn], ah0, ah1, ah2, ah3, bl0, bl1);
        mma_tf32(ga[h][nn], ah0, ah1, ah2, ah3, bh0, bh1);
      }
    }
  }
#pragma unroll
  for (int qq = 0; qq < 4; ++qq) {
    const float g0 = (qq & 1) ? ga[qq >> 1][1][2] : ga[qq >> 1][0][0];
    const float g1 = (qq & 1) ? ga[qq >> 1][1][3] : ga[qq >> 1][0][1];
    const bool live = gq < nb[qq];
    if (gq < 2 * tq) T[40 * qq + quadw::tpos(gq, 2 * tq)] = live ? tc0 * g0 : 0.f;
    if (gq < 2 * tq + 1) T[40 * qq + quadw::tpos(gq, 2 * tq + 1)] = live ? tc1 * g1 : 0.f;
  }
}

template <bool SMALL, int NP, bool GRAM, int NPRE, bool DB = false>
__global__ void __launch_bounds__(quadw::Cfg<NP, DB>::THREADS, NP <= 2 ? 4 : 1)
    factor_rows_quadw_kernel(const SweepParams p) {
  using namespace quad;
  using Leaf = quadp::Leaf<NPRE>;
  using quadp::Rec;
  using C = quadw::Cfg<NP, DB>;
  static_assert(!DB || (NPRE == 1 && !GRAM), "DB: the order-3 per-step form");
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;  // w 0: consumer, 1..NP: producers
  const int q = lane >> 3, l = lane & 7;
  uint4 *afr = reinterpret_cast<uint4 *>(smem4);
  uint64_t *bars = reinterpret_cast<uint64_t *>(reinterpret_cast<char *>(smem4) + C::FRAG_BYTES);
  uint64_t *full = bars, *empty = bars + C::NS;
  float *ring = reinterpret_cast<float *>(reinterpret_cast<char *>(bars) + C::BAR_BYTES);
  if (w > 0) {
    float *tiles = ring + C::NS * C::STAGE_FLOATS + (w - 1) * C::XY_FLOATS;
    for (int k = lane; k < C::XY_FLOATS; k += 32) tiles[k] = 0.f;
  }
  if (threadIdx.x == 0)
    for (int st = 0; st < C::NS; ++st) {
      mbar_init(full + st, 32);
      mbar_init(empty + st, 32);
    }
  if (!DB) quad_afrag_init(p, afr);
  __syncthreads();
  // m-tiles (j) / k-tiles (r) in use: compile-time (SMALL: J <= 16 and R <= 16), so the
  // unrolled combine keeps no runtime guards; other shapes compute their zero padding
  constexpr int mts = SMALL ? 1 : 2, nkt = SMALL ? 2 : 4;
  const int J = p.J;
  const bool j32 = J == 32;
  auto stage_v = [&](int st) { return ring + st * C::STAGE_FLOATS; };
  auto stage_meta = [&](int st) { return reinterpret_cast<float4 *>(ring + st * C::STAGE_FLOATS + C::META); };
  auto stage_info = [&](int st) { return reinterpret_cast<int4 *>(ring + st * C::STAGE_FLOATS + C::INFO); };
  auto stage_a = [&](int st) { return ring + st * C::STAGE_FLOATS + C::AROW; };
  auto stage_t = [&](int st) { return ring + st * C::STAGE_FLOATS + C::TCOEF; };
  const float cdec = -p.lr * p.reg;  // alpha - 1
  // GRAM: this lane's two T entries per quarter, i = g, k = 2t and 2t + 1 (the C-fragment
  // positions of the diagonal Gram blocks), and their lane-constant lr alpha^(k-1-i)
  float tc0 = 0.f, tc1 = 0.f;
  if (GRAM) {
    const int gq = lane >> 2, tq = lane & 3;
    float d = 0.f;  // alpha^n - 1, accumulated without cancellation
    for (int n = 0; n < 8; ++n) {
      if (n == 2 * tq - gq - 1) tc0 = p.lr * (1.f + d);
      if (n == 2 * tq - gq) tc1 = p.lr * (1.f + d);
      d = __fmaf_rn(cdec, 1.f + d, d);
    }
  }
  // rows per group (runtime): 4 quarters normally, 2 or 1 when the rows leave SMs idle (the
  // quarters past rpg stream nothing and run padding)
  const int rpg = p.quadw_rpg > 0 ? p.quadw_rpg : 4;

  if (w > 0) {
    // ===================================== producers =====================================
    const int k = w - 1;  // this producer runs batches t = k, k + NP, ...
    float *X = ring + C::NS * C::STAGE_FLOATS + k * C::XY_FLOATS, *Y = X + TILE;
    const int64_t nstream = (int64_t)gridDim.x * rpg;
    quadp::Cursor cur;
    cur.row = (int64_t)q * gridDim.x + blockIdx.x - nstream;
    cur.i = -1, cur.L0 = cur.Le = 0;
    if (q < rpg) {
      quadp::load_row_info(p, cur.row + nstream, cur.ni, cur.nLb, cur.nLe);
    } else {  // no rows in this quarter
      cur.ni = -1, cur.nLb = cur.nLe = 0;
    }
    const int gc = lane & 7, gs = lane >> 3;
    const bool gok = gc < (p.R >> 2);
    const float *cpre = p.Cpre[0] + 4 * gc, *cleaf = p.Cleaf + 4 * gc;
    const int64_t Rs = p.R;
    const uint32_t xs = smem_u32(X + gs * XS + 4 * gc), ys = smem_u32(Y + gs * XS + 4 * gc);
    // order 3: C_pre[0][pc] -> X and C_leaf[lc] -> Y in one async round, waited below; order 4:
    // X <- C_pre[0][pc0], Y <- C_pre[1][pc1] now, then X *= Y and Y <- C_leaf[lc] at the wait
    // (the reference's left-to-right prefix chain, as quad_gather)
    auto issue = [&](uint32_t dst0, const float *C, int coord) {
#pragma unroll
      for (int it = 0; it < 8; ++it) {
        const int cs = __shfl_sync(FULL, coord, 4 * it + gs);
        if (gok) cp_async16_s(dst0 + it * 4 * XS * 4, C + 4 * gc + cs * Rs);
      }
    };
    auto gather = [&](const Leaf &d) {
      if (NPRE == 1) {
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int s = 4 * it + gs;
          const int pcs = __shfl_sync(FULL, d.pc[0], s), lcs = __shfl_sync(FULL, d.lc, s);
          if (gok) {
            cp_async16_s(xs + it * 4 * XS * 4, cpre + pcs * Rs);
            cp_async16_s(ys + it * 4 * XS * 4, cleaf + lcs * Rs);
          }
        }
      } else {
        issue(xs, p.Cpre[0], d.pc[0]);
        issue(ys, p.Cpre[1], d.pc[NPRE > 1 ? 1 : 0]);
      }
      cp_async_commit();
    };
    auto gather_finish = [&](const Leaf &d) {  // order 4: fold the prefix, then the leaf level
      cp_async_wait_all();
      __syncwarp();
      if (NPRE > 1) {
        float4 *xr = reinterpret_cast<float4 *>(X + lane * XS);
        const float4 *yr = reinterpret_cast<const float4 *>(Y + lane * XS);
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const float4 x = xr[c], y = yr[c];
          const float2 a2 = fmul2(make_float2(x.x, x.y), make_float2(y.x, y.y));
          const float2 b2 = fmul2(make_float2(x.z, x.w), make_float2(y.z, y.w));
          xr[c] = make_float4(a2.x, a2.y, b2.x, b2.y);
        }
        __syncwarp();
        issue(ys, p.Cleaf, d.lc);
        cp_async_commit();
        cp_async_wait_all();
        __syncwarp();
      }
    };
    auto load_arow = [&](const Rec &r) {  // A values of a row about to start (quarter lanes)
      float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
      if (r.newrow && r.nb > 0) {
        const float *ar = p.A + (int64_t)r.i * J;
        if (j32) {
          v = *reinterpret_cast<const float4 *>(ar + 4 * l);
        } else {
          v.x = 4 * l < J ? ar[4 * l] : 0.f;
          v.y = 4 * l + 1 < J ? ar[4 * l + 1] : 0.f;
          v.z = 4 * l + 2 < J ? ar[4 * l + 2] : 0.f;
          v.w = 4 * l + 3 < J ? ar[4 * l + 3] : 0.f;
        }
      }
      return v;
    };
    // the record of my next batch: skip the other producers' batches (row-start flags carry
    // over a skipped batch only if it started a row and mine continues it -- then mine is not
    // the row's first batch, which is what the consumer needs)
    auto next_mine = [&](bool first) {
      if (!first)
        for (int s = 0; s < NP - 1; ++s) (void)quadp::next_batch(p, cur, nstream);
      return quadp::next_batch(p, cur, nstream);
    };
    // the Bt^T fragments live in registers for the whole sweep (64 per lane): the shared-memory
    // pipe is the producers' scarce resource
    uint4 AH[KT][MT], AL[KT][MT];
#pragma unroll
    for (int kt = 0; kt < KT; ++kt)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        if (DB) {
          quad_afrag_lane(p, kt, mt, lane, AH[kt][mt], AL[kt][mt]);
        } else {
          AH[kt][mt] = afr[(mt * KT + kt) * 32 + lane];
          AL[kt][mt] = afr[KT * MT * 32 + (mt * KT + kt) * 32 + lane];
        }
      }
    for (int s = 0; s < k; ++s) (void)quadp::next_batch(p, cur, nstream);
    float acc[2][4][4];
    // publish batch t (V, step operands, row start / stop record) into ring stage t % NS
    auto publish = [&](int t, bool stop, const Rec &r0, const Leaf &d0, const float4 &av0) {
      const int st = t % C::NS;
      if (t >= C::NS) mbar_wait(empty + st, ((t / C::NS) - 1) & 1);
      int4 *info = stage_info(st);
      if (!stop) {
        quad_store_v(stage_v(st), acc, lane);
        const float lrk = l < r0.nb ? p.lr : 0.f;
        const float ck = -lrk * p.reg;
        if (!GRAM) stage_meta(st)[q * MQ + l] = make_float4(l < r0.nb ? d0.x : 0.f, lrk, ck, ck);
        if (r0.newrow) *reinterpret_cast<float4 *>(stage_a(st) + 32 * q + 4 * l) = av0;
        if (l == 0) info[q] = make_int4(r0.nb, r0.newrow ? 1 : 0, r0.i, 0);
        if (GRAM) {
          stage_t(st)[C::TQ * q + 28 + l] = l < r0.nb ? d0.x : 0.f;  // the batch's x, packed
          __syncwarp();
          int nbq[4];
#pragma unroll
          for (int qq = 0; qq < 4; ++qq) nbq[qq] = __shfl_sync(FULL, r0.nb, 8 * qq);
          quadw_gram<SMALL>(stage_v(st), stage_t(st), nbq, tc0, tc1, lane);
        }
      } else if (l == 0) {
        info[q] = make_int4(0, 0, -1, 1);  // stop
      }
      __syncwarp();
      mbar_arrive(full + st);
    };
    if (DB) {
      // double-buffered: the gathers of my next batch go into the other X / Y pair at the top
      // of the iteration and fly under this batch's combine and publication (two cp.async
      // groups in flight); leaf records two batches ahead
      const uint32_t tile2 = (uint32_t)(2 * TILE * 4);  // bytes between the two X / Y pairs
      auto gather_into = [&](int b, const Leaf &d) {
        const uint32_t off = b ? tile2 : 0u;
#pragma unroll
        for (int it = 0; it < 8; ++it) {
          const int s = 4 * it + gs;
          const int pcs = __shfl_sync(FULL, d.pc[0], s), lcs = __shfl_sync(FULL, d.lc, s);
          if (gok) {
            cp_async16_s(xs + off + it * 4 * XS * 4, cpre + pcs * Rs);
            cp_async16_s(ys + off + it * 4 * XS * 4, cleaf + lcs * Rs);
          }
        }
        cp_async_commit();
      };
      Rec r0 = next_mine(true);
      Leaf d0 = quadp::load_leaf<NPRE>(p, r0, l);
      float4 av0 = load_arow(r0);
      bool stop0 = !__any_sync(FULL, r0.nb > 0);
      if (!stop0) gather_into(0, d0);
      Rec r1 = next_mine(false);
      Leaf d1 = quadp::load_leaf<NPRE>(p, r1, l);
      float4 av1 = load_arow(r1);
      int buf = 0;
      for (int t = k;; t += NP) {
        const bool stop1 = !__any_sync(FULL, r1.nb > 0);
        if (!stop0 && !stop1) gather_into(buf ^ 1, d1);
        const Rec r2 = next_mine(false);
        const Leaf d2 = quadp::load_leaf<NPRE>(p, r2, l);
        const float4 av2 = load_arow(r2);
        if (!stop0) {
          if (!stop1) cp_async_wait_group<1>();
          else cp_async_wait_all();
          __syncwarp();
          const float *Xb = X + (buf ? 2 * TILE : 0), *Yb = Y + (buf ? 2 * TILE : 0);
          quad_zero(acc);
#pragma unroll
          for (int kt = 0; kt < KT; ++kt)
            if (kt < nkt) quad_mma_kt_r<NT>(Xb, Yb, AH[kt], AL[kt], kt, 0, lane, acc, mts);
        }
        publish(t, stop0, r0, d0, av0);  // ends in __syncwarp: X / Y [buf] are free again
        if (stop0) break;
        r0 = r1, d0 = d1, av0 = av1, stop0 = stop1;
        r1 = r2, d1 = d2, av1 = av2;
        buf ^= 1;
      }
    } else {
      Rec r0 = next_mine(true);
      Leaf d0 = quadp::load_leaf<NPRE>(p, r0, l);
      float4 av0 = load_arow(r0);
      for (int t = k;; t += NP) {
        const bool stop = !__any_sync(FULL, r0.nb > 0);
        if (!stop) gather(d0);
        const Rec r1 = next_mine(false);  // my next batch: indices and A values fly meanwhile
        const Leaf d1 = quadp::load_leaf<NPRE>(p, r1, l);
        const float4 av1 = load_arow(r1);
        if (!stop) {
          gather_finish(d0);
          quad_zero(acc);
#pragma unroll
          for (int kt = 0; kt < KT; ++kt)
            if (kt < nkt) quad_mma_kt_r<NT>(X, Y, AH[kt], AL[kt], kt, 0, lane, acc, mts);
        }
        publish(t, stop, r0, d0, av0);
        if (stop) break;
        r0 = r1, d0 = d1, av0 = av1;
      }
    }
    cp_async_wait_all();
  } else {
    // ===================================== consumer =====================================
    float a[4] = {0.f, 0.f, 0.f, 0.f}, lo[4] = {0.f, 0.f, 0.f, 0.f};
    int ai = -1;
    auto store_a = [&]() {
      float *ar = p.A + (int64_t)ai * J;
      const float o[4] = {a[0] + lo[0], a[1] + lo[1], a[2] + lo[2], a[3] + lo[3]};
      if (j32) {
        *reinterpret_cast<float4 *>(ar + 4 * l) = make_float4(o[0], o[1], o[2], o[3]);
      } else {
#pragma unroll
        for (int t = 0; t < 4; ++t)
          if (4 * l + t < J) ar[4 * l + t] = o[t];
      }
    };
    // GRAM: Dk[k] = alpha^k - 1 (k = 0..8) and the full batch's update weights lr alpha^(7-i)
    float Dk[9], wfull[8];
    Dk[0] = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) Dk[k + 1] = __fmaf_rn(cdec, 1.f + Dk[k], Dk[k]);
#pragma unroll
    for (int i = 0; i < 8; ++i) wfull[i] = p.lr * (1.f + Dk[7 - i]);
    if (!GRAM) {  // the per-step chain: short batches run all 8 steps (padding: lr = 0)
      for (int t = 0;; ++t) {
        const int st = t % C::NS;
        mbar_wait(full + st, (t / C::NS) & 1);
        const int4 info = stage_info(st)[q];
        if (info.w) break;  // stop (every quarter carries the flag)
        if (info.y) {       // this quarter starts row info.z
          if (ai >= 0) store_a();
          const float4 v = *reinterpret_cast<const float4 *>(stage_a(st) + 32 * q + 4 * l);
          a[0] = v.x, a[1] = v.y, a[2] = v.z, a[3] = v.w;
          lo[0] = lo[1] = lo[2] = lo[3] = 0.f;
          ai = info.z;
        }
        // the stage's 8 V rows and step operands up front: independent LDS.128, one latency
        const float *Vq = stage_v(st) + 8 * q * QVS + 4 * l;
        const float4 *mq = stage_meta(st) + q * MQ;
        float4 vv[QB], mm[QB];
#pragma unroll
        for (int kk = 0; kk < QB; ++kk) {
          vv[kk] = *reinterpret_cast<const float4 *>(Vq + kk * QVS);
          mm[kk] = mq[kk];
        }
        __syncwarp();
        mbar_arrive(empty + st);  // the stage is free once read
        if (DB) {  // one step of lookahead: the chain at about half the serial latency
          quad_batch_lookahead(a, lo, vv, mm);
        } else {
#pragma unroll
          for (int kk = 0; kk < QB; ++kk) quad_chain_step_vc(a, lo, vv[kk], mm[kk]);
        }
      }
    } else {
      // Gram form, software-pipelined: batch t + 1's stage is waited for, read into the other
      // register set and released while batch t is solved, so the loads and the mbarrier round
      // trip leave the serial path (butterfly -> solve -> update)
      struct Batch {
        int4 info;
        float4 arow;
        float4 vv[QB];
        float T[28], xk[QB];
      };
      auto load = [&](Batch &B, int t) {
        const int st = t % C::NS;
        mbar_wait(full + st, (t / C::NS) & 1);
        B.info = stage_info(st)[q];
        B.arow = *reinterpret_cast<const float4 *>(stage_a(st) + 32 * q + 4 * l);
        const float *Vq = stage_v(st) + 8 * q * QVS + 4 * l;
#pragma unroll
        for (int kk = 0; kk < QB; ++kk) B.vv[kk] = *reinterpret_cast<const float4 *>(Vq + kk * QVS);
        const float4 *tq4 = reinterpret_cast<const float4 *>(stage_t(st) + C::TQ * q);
#pragma unroll
        for (int u = 0; u < 7; ++u) {
          const float4 t4 = tq4[u];
          B.T[4 * u] = t4.x, B.T[4 * u + 1] = t4.y, B.T[4 * u + 2] = t4.z, B.T[4 * u + 3] = t4.w;
        }
        const float4 x0 = tq4[7], x1 = tq4[8];
        B.xk[0] = x0.x, B.xk[1] = x0.y, B.xk[2] = x0.z, B.xk[3] = x0.w;
        B.xk[4] = x1.x, B.xk[5] = x1.y, B.xk[6] = x1.z, B.xk[7] = x1.w;
        __syncwarp();
        mbar_arrive(empty + st);  // the stage is free once read
      };
      auto process = [&](const Batch &B) {
        if (B.info.y) {  // this quarter starts row info.z
          if (ai >= 0) store_a();
          a[0] = B.arow.x, a[1] = B.arow.y, a[2] = B.arow.z, a[3] = B.arow.w;
          lo[0] = lo[1] = lo[2] = lo[3] = 0.f;
          ai = B.info.z;
        }
        // the eight dots a_0 . v_k: lane partials, one butterfly over the quarter's 8 lanes
        float pk[QB];
#pragma unroll
        for (int kk = 0; kk < QB; ++kk) {
          float2 pr = fmul2(make_float2(a[0], a[1]), make_float2(B.vv[kk].x, B.vv[kk].y));
          pr = ffma2(make_float2(a[2], a[3]), make_float2(B.vv[kk].z, B.vv[kk].w), pr);
          pk[kk] = pr.x + pr.y;
        }
#pragma unroll
        for (int m = 4; m >= 1; m >>= 1)
#pragma unroll
          for (int kk = 0; kk < QB; ++kk) pk[kk] += __shfl_xor_sync(FULL, pk[kk], m);
        // r_k = x_k - alpha^k p_k, then the unit lower-triangular solve (right-looking)
        float r[QB];
#pragma unroll
        for (int kk = 0; kk < QB; ++kk) r[kk] = __fmaf_rn(-Dk[kk], pk[kk], B.xk[kk] - pk[kk]);
#pragma unroll
        for (int i = 0; i < QB - 1; ++i)
#pragma unroll
          for (int kk = i + 1; kk < QB; ++kk) r[kk] = __fmaf_rn(-B.T[quadw::tpos(i, kk)], r[i], r[kk]);
        // a_nb = alpha^nb a_0 + sum_i lr alpha^(nb-1-i) e_i v_i: full batches use the constant
        // weights; otherwise (a row's last batch, or a quarter without rows: nb = 0) the
        // weights are rescaled by alpha^-(8-nb) and the padding zeroed -- selects, no loops
        const int nb = B.info.x;
        float wsc[QB], dn = Dk[QB];
#pragma unroll
        for (int i = 0; i < QB; ++i) wsc[i] = wfull[i];
        if (!__all_sync(FULL, nb == QB)) {
          float dd = 0.f;
#pragma unroll
          for (int m = 0; m < QB; ++m)
            if (nb == m) dn = Dk[m], dd = Dk[QB - m];
          const float sc = __fdividef(1.f, 1.f + dd);
#pragma unroll
          for (int i = 0; i < QB; ++i) wsc[i] = i < nb ? wfull[i] * sc : 0.f;
        }
        // d = sum_i w_i e_i v_i in two independent chains
        float2 da01 = make_float2(0.f, 0.f), da23 = da01, db01 = da01, db23 = da01;
#pragma unroll
        for (int i = 0; i < QB; i += 2) {
          const float w0 = wsc[i] * r[i], w1 = wsc[i + 1] * r[i + 1];
          da01 = ffma2(make_float2(w0, w0), make_float2(B.vv[i].x, B.vv[i].y), da01);
          da23 = ffma2(make_float2(w0, w0), make_float2(B.vv[i].z, B.vv[i].w), da23);
          db01 = ffma2(make_float2(w1, w1), make_float2(B.vv[i + 1].x, B.vv[i + 1].y), db01);
          db23 = ffma2(make_float2(w1, w1), make_float2(B.vv[i + 1].z, B.vv[i + 1].w), db23);
        }
        const float2 d01 = fadd2(da01, db01), d23 = fadd2(da23, db23);
        // compensated a <- a + (dn a + d + lo)
        const float2 c2 = make_float2(dn, dn);
        const float2 a01 = make_float2(a[0], a[1]), a23 = make_float2(a[2], a[3]);
        const float2 e01 = fadd2(d01, ffma2(c2, a01, make_float2(lo[0], lo[1])));
        const float2 e23 = fadd2(d23, ffma2(c2, a23, make_float2(lo[2], lo[3])));
        const float2 t01 = fadd2(a01, e01), t23 = fadd2(a23, e23);
        const float2 s01 = fsub2(e01, fsub2(t01, a01)), s23 = fsub2(e23, fsub2(t23, a23));
        a[0] = t01.x, a[1] = t01.y, a[2] = t23.x, a[3] = t23.y;
        lo[0] = s01.x, lo[1] = s01.y, lo[2] = s23.x, lo[3] = s23.y;
      };
      Batch b0, b1;
      load(b0, 0);
      for (int t = 0;; t += 2) {
        if (b0.info.w) break;  // stop (every quarter carries the flag)
        load(b1, t + 1);
        process(b0);
        if (b1.info.w) break;
        load(b0, t + 2);
        process(b1);
      }
    }
    if (ai >= 0) store_a();
  }
}

template <bool SMALL, int NP, bool GRAM, int NPRE, bool DB = false>
int launch_quadw_t(const SweepParams &q0, int rpg, cudaStream_t s) {
  SweepParams q = q0;
  q.quadw_rpg = rpg;
  using C = quadw::Cfg<NP, DB>;
  auto kern = factor_rows_quadw_kernel<SMALL, NP, GRAM, NPRE, DB>;
  const size_t sm = C::bytes();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    set = true;
  }
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, C::THREADS, sm) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  int64_t g = (q.nrows + rpg - 1) / rpg;
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  kern<<<(int)g, C::THREADS, sm, s>>>(q);
  return check_launch("ft_factor_sweep_rows(quadw)");
}

// Few rows per SM (the row-sharded multi-GPU sweeps: groups <= SMs): the Gram form, six
// producers per group, 2 or 1 rows per group when 4 would leave SMs idle -- the serial chain is
// the bound there.  Many rows (one GPU: 3.7 groups per SM): the per-step chain and two producers
// -- there the producers' gathers / combine leave no room for the Gram blocks (measured: 5.9 vs
// 7.5-7.9 ms on Netflix mode 2, profiles/r02_quadw_gram.md).  FT_QUADW_GRAM=0 / 1 forces one
// form (A/B).
template <bool SMALL, int NPRE>
int launch_quadw_s(const SweepParams &q, cudaStream_t s) {
  static const int forced = [] {
    const char *e = getenv("FT_QUADW_GRAM");
    return e ? atoi(e) : -1;
  }();
  const int64_t sms = sm_count();
  int rpg = 4;
  while (rpg > 1 && (q.nrows + rpg / 2 - 1) / (rpg / 2) <= sms) rpg /= 2;
  const bool few = (q.nrows + 3) / 4 <= sms;
  static const bool db = [] {  // FT_QUADW_DB=0: the single-buffered per-step form (A/B)
    const char *e = getenv("FT_QUADW_DB");
    return !(e && e[0] == '0');
  }();
  if (forced == 0 || (forced < 0 && !few)) {
    if constexpr (NPRE == 1)
      if (db) return launch_quadw_t<SMALL, 2, false, NPRE, true>(q, 4, s);
    return launch_quadw_t<SMALL, 2, false, NPRE>(q, 4, s);
  }
  return launch_quadw_t<SMALL, 6, true, NPRE>(q, few ? rpg : 4, s);
}

int launch_quadw(const SweepParams &q, cudaStream_t s) {
  const bool small = q.J <= 16 && q.R <= 16;
  if (q.N == 4) return small ? launch_quadw_s<true, 2>(q, s) : launch_quadw_s<false, 2>(q, s);
  return small ? launch_quadw_s<true, 1>(q, s) : launch_quadw_s<false, 1>(q, s);
}

// the quad kernels run any J, R <= 32 (R % 4 == 0; padding columns are zero); J = R = 16 has
// its own instantiation (one m-tile, two k-tiles)
bool quad_ok(const SweepParams &p) {
  return p.N >= 3 && p.N <= 6 && p.leaf_pc && p.row_leaf_ptr && p.J <= 32 && p.R <= 32 &&
         (p.R & 3) == 0;
}

// ---- K4 "quad": the core-gradient row sweep over the leaf-major index ---------------------
// Reference core_sweep (_ckern.pyx:202-269) in its row form: with A_u, Bt_u
// frozen and C_u = A_u Bt_u^T coherent, s = A_u[i] . vec = C_u[i] . cross, and
//     acc = -sum_i g_i (x) A_u[i],   g_i = sum_{leaves of row i} e cross.
// Four rows per warp (quarters) as in the quad factor kernel, same gathers and index pipeline.
// Per 32-slot batch: lane k computes s_k = sum_r X[k][r] Y[k][r] C_u[i_q][r] for its own slot
// (conflict-free stride-36 rows, C_u row broadcast per quarter), then quarter lanes over r
// accumulate g_q += e_k cross_k over the quarter's 8 slots.  When a row ends its g (8 lanes x 4)
// is spread to lanes over r and the warp adds g (x) A_u[i] into per-lane accumulators
// (lane r: acc[j]); a fixed-order block reduction writes one R x J partial per block.
namespace cquad {
constexpr int XS = 36;
constexpr int TILE = 32 * XS;
constexpr int WARP_FLOATS = 2 * TILE + 4 * 32 + 32;  // X, Y, C_u rows [4][32], e [32]
constexpr int WPB = 8;
constexpr size_t bytes() { return (size_t)WPB * WARP_FLOATS * 4; }
// the DIRECT form stages nothing: its shared memory is only the block's fixed-order reduction
// (R x J floats per warp), so the rest of the SM's 256 KB stays L1 data cache -- where the small
// gathered C matrices (Netflix C_2: 280 KB) hit instead of going to L2
constexpr int DIRECT_WS = FT_MAX_RANK * FT_MAX_RANK;
constexpr size_t direct_bytes() { return (size_t)WPB * DIRECT_WS * 4; }
}  // namespace cquad

// SSE = true: the same walk scores the tree's leaves instead (K6b, evaluate over the training
// entries, train.py:91-98): per slot e = x - C_u[i] . cross, sum e^2 and |e| in fp64 per lane,
// fixed-order block reduction to p.partials as doubles [block][2] (no gradient work).
#ifndef CORE_FUSED
#define CORE_FUSED 1  // K4 quad: fused single pass in the quarter layout (0: lane-per-slot s-pass)
#endif
// DIRECT (gradient form): the R x J accumulator lives in the warp's shared-memory slice
// ([j][lane r], conflict-free) instead of 32 registers per lane, so three blocks fit an SM --
// more gathers in flight for a kernel that waits on them (the long-scoreboard stalls)
template <bool SSE, int NPRE, bool DIRECT = false>
__global__ void __launch_bounds__(cquad::WPB * 32, DIRECT ? 3 : 2) core_rows_quad_kernel(const SweepParams p) {
  using namespace cquad;
  extern __shared__ float4 smem4[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int q = lane >> 3, l = lane & 7;
  constexpr int WS = DIRECT ? DIRECT_WS : WARP_FLOATS;  // per-warp shared-memory floats
  float *X = reinterpret_cast<float *>(smem4) + w * WS;
  float *Y = X + TILE;
  float *cus = Y + TILE;  // [4][32] (staged form only)
  float *es = cus + 128;  // [32]
  constexpr bool SMACC = DIRECT && !SSE;
  float *accs = X;  // SMACC: [j][r] accumulator slice of this warp
  if (!DIRECT) {
    for (int k = lane; k < WARP_FLOATS; k += 32) X[k] = 0.f;
    __syncwarp();
  } else if (SMACC) {
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j) accs[j * 32 + lane] = 0.f;
    __syncwarp();
  }
  const int J = p.J, R = p.R;
  const int64_t nstream = (int64_t)gridDim.x * cquad::WPB * 4;
  int64_t row = (int64_t)(4 * w + q) * gridDim.x + blockIdx.x;  // block-fastest (see quad)
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
  float2 cu01 = make_float2(0.f, 0.f), cu23 = cu01;  // C_u[i_q][4l .. 4l+3] (fused pass)
  auto load_cu = [&](int i) {  // C_u[i, 0:R) -> cus[q][.] (zero beyond R)
    if (4 * l < R) {
      const float4 v = *reinterpret_cast<const float4 *>(p.Cu + (int64_t)i * R + 4 * l);
      if (CORE_FUSED) {
        cu01 = make_float2(v.x, v.y), cu23 = make_float2(v.z, v.w);
      } else {
        *reinterpret_cast<float4 *>(cus + 32 * q + 4 * l) = v;
      }
    }
  };
  if (ci >= 0) load_cu(ci);
  int plc = 0, ppc[NPRE];
  float px = 0.f;
#pragma unroll
  for (int d = 0; d < NPRE; ++d) ppc[d] = 0;
  if (ci >= 0 && cL0 + l < cLe) {
    plc = __ldcs(p.leaf_coord + cL0 + l);
#pragma unroll
    for (int d = 0; d < NPRE; ++d) ppc[d] = __ldcs(p.leaf_pc + (int64_t)(cL0 + l) * NPRE + d);
    px = __ldcs(p.vals + cL0 + l);
  }
  float acc[FT_MAX_RANK];  // lane r: acc[j] = sum_i g_i[r] A_u[i, j]
#pragma unroll
  for (int j = 0; j < FT_MAX_RANK; ++j) acc[j] = 0.f;
  float2 g01 = make_float2(0.f, 0.f), g23 = make_float2(0.f, 0.f);  // quarter lanes: g[4l..4l+3]
  double sse = 0.0, sae = 0.0;  // SSE mode
  const bool j32 = J == 32;

  for (;;) {
    // ---- rows that ended: acc += g (x) A_u[i] (warp-cooperative, one quarter at a time) ----
    const bool ending = ci >= 0 && cL0 >= cLe;
    unsigned em = SSE ? 0u : __ballot_sync(FULL, ending && l == 0);
    while (em) {
      const int qq = __ffs(em) - 1 >> 3;
      em &= em - 1;
      const int src = 8 * qq + (lane >> 2), comp = lane & 3;
      const float c0 = __shfl_sync(FULL, g01.x, src), c1 = __shfl_sync(FULL, g01.y, src);
      const float c2 = __shfl_sync(FULL, g23.x, src), c3 = __shfl_sync(FULL, g23.y, src);
      const float gr = comp == 0 ? c0 : comp == 1 ? c1 : comp == 2 ? c2 : c3;  // g_qq[lane]
      const float *ar = p.A + (int64_t)__shfl_sync(FULL, ci, 8 * qq) * J;
      if (SMACC) {
        float *ac = accs + lane;
        if (j32) {
#pragma unroll
          for (int j4 = 0; j4 < 8; ++j4) {
            const float4 a4 = __ldg(reinterpret_cast<const float4 *>(ar) + j4);
            ac[(4 * j4) * 32] = __fmaf_rn(gr, a4.x, ac[(4 * j4) * 32]);
            ac[(4 * j4 + 1) * 32] = __fmaf_rn(gr, a4.y, ac[(4 * j4 + 1) * 32]);
            ac[(4 * j4 + 2) * 32] = __fmaf_rn(gr, a4.z, ac[(4 * j4 + 2) * 32]);
            ac[(4 * j4 + 3) * 32] = __fmaf_rn(gr, a4.w, ac[(4 * j4 + 3) * 32]);
          }
        } else {
          for (int j = 0; j < J; ++j) ac[j * 32] = __fmaf_rn(gr, __ldg(ar + j), ac[j * 32]);
        }
      } else if (j32) {
#pragma unroll
        for (int j4 = 0; j4 < 8; ++j4) {
          const float4 a4 = __ldg(reinterpret_cast<const float4 *>(ar) + j4);
          acc[4 * j4] = __fmaf_rn(gr, a4.x, acc[4 * j4]);
          acc[4 * j4 + 1] = __fmaf_rn(gr, a4.y, acc[4 * j4 + 1]);
          acc[4 * j4 + 2] = __fmaf_rn(gr, a4.z, acc[4 * j4 + 2]);
          acc[4 * j4 + 3] = __fmaf_rn(gr, a4.w, acc[4 * j4 + 3]);
        }
      } else {
#pragma unroll
        for (int j = 0; j < FT_MAX_RANK; ++j)
          if (j < J) acc[j] = __fmaf_rn(gr, __ldg(ar + j), acc[j]);
      }
    }
    if (ending) {
      g01 = g23 = make_float2(0.f, 0.f);
      row += nstream;
      ci = ni, cL0 = nLb, cLe = nLe;
      if (ci >= 0) {
        load_cu(ci);
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
    const int nb = ci >= 0 ? min(quad::QB, cLe - cL0) : 0;
    const int lc = plc;
    int pc[NPRE];
#pragma unroll
    for (int d = 0; d < NPRE; ++d) pc[d] = ppc[d];
    const float x = px;
    {  // prefetch the next batch of this quarter
      const bool same = cL0 + nb < cLe;
      const int pos = same ? cL0 + nb : nLb, end = same ? cLe : nLe;
      const bool ok = ci >= 0 && (same || ni >= 0) && pos + l < end;
      plc = ok ? __ldcs(p.leaf_coord + pos + l) : 0;
#pragma unroll
      for (int d = 0; d < NPRE; ++d)
        ppc[d] = ok ? __ldcs(p.leaf_pc + (int64_t)(pos + l) * NPRE + d) : 0;
      px = ok ? __ldcs(p.vals + pos + l) : 0.f;
    }
    if (DIRECT) {
      // the fused pass with no staging: the K4 core has no MMA, so each lane loads the 16-B
      // chunks it consumes (columns 4l..4l+3 of its quarter's leaves) straight into registers --
      // no shared-memory write or read per leaf on an L1-bound kernel.  Four leaves in flight
      // per half-batch; padding leaves load nothing.  Arithmetic as in the staged pass.
      const bool lok = 4 * l < R;
      const int64_t Rs = R;
      constexpr int LH = NPRE <= 2 ? 4 : 2;  // leaves in flight per lane (register budget)
#pragma unroll
      for (int h = 0; h < 8 / LH; ++h) {
        float4 xv[LH], yv[LH];
#pragma unroll
        for (int kk = 0; kk < LH; ++kk) {
          const int k = LH * h + kk, sl = 8 * q + k;
          const int cy = __shfl_sync(FULL, lc, sl);
          int cx[NPRE];
#pragma unroll
          for (int d = 0; d < NPRE; ++d) cx[d] = __shfl_sync(FULL, pc[d], sl);
          const bool ok = lok && k < nb;
          xv[kk] = yv[kk] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (ok) {
            float4 lv[NPRE];
#pragma unroll
            for (int d = 0; d < NPRE; ++d)
              lv[d] = __ldg(reinterpret_cast<const float4 *>(p.Cpre[d] + cx[d] * Rs + 4 * l));
            yv[kk] = __ldg(reinterpret_cast<const float4 *>(p.Cleaf + cy * Rs + 4 * l));
            xv[kk] = lv[0];
#pragma unroll
            for (int d = 1; d < NPRE; ++d) {  // the prefix chain left to right (quad_gather's fold)
              const float2 a = fmul2(make_float2(xv[kk].x, xv[kk].y), make_float2(lv[d].x, lv[d].y));
              const float2 b = fmul2(make_float2(xv[kk].z, xv[kk].w), make_float2(lv[d].z, lv[d].w));
              xv[kk] = make_float4(a.x, a.y, b.x, b.y);
            }
          }
        }
#pragma unroll
        for (int kk = 0; kk < LH; ++kk) {
          const int k = LH * h + kk;
          const float2 c01 = fmul2(make_float2(xv[kk].x, xv[kk].y), make_float2(yv[kk].x, yv[kk].y));
          const float2 c23 = fmul2(make_float2(xv[kk].z, xv[kk].w), make_float2(yv[kk].z, yv[kk].w));
          const float2 sp = ffma2(c23, cu23, fmul2(c01, cu01));
          float sv = sp.x + sp.y;
          sv += __shfl_xor_sync(FULL, sv, 1);
          sv += __shfl_xor_sync(FULL, sv, 2);
          sv += __shfl_xor_sync(FULL, sv, 4);
          const float xk = __shfl_sync(FULL, x, 8 * q + k);
          const float e = k < nb ? xk - sv : 0.f;
          if (SSE) {
            if (l == 0) {
              sse += (double)e * (double)e;
              sae += fabs((double)e);
            }
          } else {
            const float2 e2 = make_float2(e, e);
            g01 = ffma2(e2, c01, g01);
            g23 = ffma2(e2, c23, g23);
          }
        }
      }
      cL0 += nb;
      continue;
    }
    quad_gather<NPRE, XS>(p, X, Y, pc, lc, lane);
    if (CORE_FUSED) {
      // one pass in the quarter layout (lane l: columns 4l..4l+3 of its quarter's rows): the
      // same X / Y loads feed s_k (partial dot with C_u[i], reduced over the quarter's 8 lanes)
      // and g += e_k cross_k -- half the shared-memory reads of the two-pass form
      const float *xq = X + 8 * q * XS + 4 * l, *yq = Y + 8 * q * XS + 4 * l;
#pragma unroll
      for (int k = 0; k < quad::QB; ++k) {
        const float4 xv = *reinterpret_cast<const float4 *>(xq + k * XS);
        const float4 yv = *reinterpret_cast<const float4 *>(yq + k * XS);
        const float2 c01 = fmul2(make_float2(xv.x, xv.y), make_float2(yv.x, yv.y));
        const float2 c23 = fmul2(make_float2(xv.z, xv.w), make_float2(yv.z, yv.w));
        const float2 sp = ffma2(c23, cu23, fmul2(c01, cu01));
        float sv = sp.x + sp.y;
        sv += __shfl_xor_sync(FULL, sv, 1);
        sv += __shfl_xor_sync(FULL, sv, 2);
        sv += __shfl_xor_sync(FULL, sv, 4);
        const float xk = __shfl_sync(FULL, x, 8 * q + k);
        const float e = k < nb ? xk - sv : 0.f;
        if (SSE) {
          if (l == 0) {
            sse += (double)e * (double)e;
            sae += fabs((double)e);
          }
        } else {
          const float2 e2 = make_float2(e, e);
          g01 = ffma2(e2, c01, g01);
          g23 = ffma2(e2, c23, g23);
        }
      }
      __syncwarp();
      cL0 += nb;
      continue;
    }
    // ---- lane = slot: s = C_u[i_q] . (X * Y), e = x - s ----
    {
      const float4 *xr = reinterpret_cast<const float4 *>(X + lane * XS);
      const float4 *yr = reinterpret_cast<const float4 *>(Y + lane * XS);
      const float4 *cr = reinterpret_cast<const float4 *>(cus + 32 * q);
      float2 s01 = make_float2(0.f, 0.f), s23 = make_float2(0.f, 0.f);
#pragma unroll
      for (int c4 = 0; c4 < 8; ++c4) {
        const float4 xv = xr[c4], yv = yr[c4], cv = cr[c4];
        s01 = ffma2(fmul2(make_float2(xv.x, xv.y), make_float2(yv.x, yv.y)),
                    make_float2(cv.x, cv.y), s01);
        s23 = ffma2(fmul2(make_float2(xv.z, xv.w), make_float2(yv.z, yv.w)),
                    make_float2(cv.z, cv.w), s23);
      }
      const float s = (s01.x + s01.y) + (s23.x + s23.y);
      const float e = l < nb ? x - s : 0.f;
      if (SSE) {
        sse += (double)e * (double)e;
        sae += fabs((double)e);
      } else {
        es[lane] = e;
      }
    }
    if (SSE) {
      __syncwarp();
      cL0 += nb;
      continue;
    }
    __syncwarp();
    // ---- quarter lanes over r: g_q += sum_k e_k cross_k ----
    {
      const int nbmax = __reduce_max_sync(FULL, (unsigned)nb);
      const float *xq = X + 8 * q * XS + 4 * l, *yq = Y + 8 * q * XS + 4 * l;
#pragma unroll
      for (int k = 0; k < quad::QB; ++k) {
        if (k >= nbmax) break;
        const float4 xv = *reinterpret_cast<const float4 *>(xq + k * XS);
        const float4 yv = *reinterpret_cast<const float4 *>(yq + k * XS);
        const float ek = es[8 * q + k];
        const float2 e2 = make_float2(ek, ek);
        g01 = ffma2(e2, fmul2(make_float2(xv.x, xv.y), make_float2(yv.x, yv.y)), g01);
        g23 = ffma2(e2, fmul2(make_float2(xv.z, xv.w), make_float2(yv.z, yv.w)), g23);
      }
    }
    __syncwarp();
    cL0 += nb;
  }
  // ---- fixed-order block reduction -> partials[block] (reuses the staging tiles) ----
  __syncthreads();
  if (SSE) {
    double *rd = reinterpret_cast<double *>(smem4);
    rd[2 * threadIdx.x] = sse;
    rd[2 * threadIdx.x + 1] = sae;
    __syncthreads();
    if (threadIdx.x == 0) {
      double a = 0.0, b = 0.0;
      for (int k = 0; k < (int)blockDim.x; ++k) {
        a += rd[2 * k];
        b += rd[2 * k + 1];
      }
      reinterpret_cast<double *>(p.partials)[2 * blockIdx.x] = a;
      reinterpret_cast<double *>(p.partials)[2 * blockIdx.x + 1] = b;
    }
    return;
  }
  const int RJ = R * J;
  float *red = reinterpret_cast<float *>(smem4);
  if (SMACC) {  // the warps' [j][r] slices are already in place
    __syncthreads();
    for (int k = threadIdx.x; k < RJ; k += blockDim.x) {
      const int r = k / J, j = k - r * J;
      float s = 0.f;
      for (int ww = 0; ww < cquad::WPB; ++ww) s += red[ww * WS + j * 32 + r];
      p.partials[(int64_t)blockIdx.x * RJ + k] = s;
    }
    return;
  }
  if (lane < R) {
#pragma unroll
    for (int j = 0; j < FT_MAX_RANK; ++j)
      if (j < J) red[w * WS + lane * J + j] = acc[j];
  }
  __syncthreads();
  for (int k = threadIdx.x; k < RJ; k += blockDim.x) {
    float s = 0.f;
    for (int ww = 0; ww < cquad::WPB; ++ww) s += red[ww * WS + k];
    p.partials[(int64_t)blockIdx.x * RJ + k] = s;
  }
}

bool core_quad_ok(const SweepParams &p) {
  return p.N >= 3 && p.N <= 6 && p.leaf_pc && p.row_leaf_ptr && p.J <= 32 && p.R <= 32 && (p.R & 3) == 0 &&
         p.R * p.J <= cquad::WARP_FLOATS;
}

// K4 direct (register gathers) while the gathered C matrices sit in L2, staged above
bool core_direct(const SweepParams &p) {
  // direct register loads keep 4 leaves in flight per lane, the staged pass 32 rows per warp:
  // direct wins while the gathered C matrices sit in L2 (Netflix32 61 MB: core 2.41 -> 2.20 ms
  // per mode; order-4 10K^4 19.9 -> 12.7 ms), staging wins once their misses go to HBM
  // (Yahoo32 mode 2, 208 MB: 8.1 vs 9.3 ms; modes 0 / 1, 80 MB: 6.5 vs 6.8 ms).
  // FT_CORE_DIRECT=0 / 1 forces either.
  static const int direct_env = [] {
    const char *e = getenv("FT_CORE_DIRECT");
    return e && e[0] ? (e[0] == '0' ? 0 : 1) : -1;
  }();
  return direct_env >= 0 ? direct_env == 1 : p.gather_bytes <= (64ll << 20);
}

template <bool SSE, int NPRE>
int core_quad_grid_t(const SweepParams &p) {
  const size_t sm = cquad::bytes();
  static bool set = false;
  if (!set) {
    cudaFuncSetAttribute(core_rows_quad_kernel<SSE, NPRE>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    cudaFuncSetAttribute(core_rows_quad_kernel<SSE, NPRE, true>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cquad::direct_bytes());
    // three blocks x 32 KB (accumulators / reduction): the smallest carveout that holds them,
    // the rest of the SM's 256 KB stays L1
    cudaFuncSetAttribute(core_rows_quad_kernel<SSE, NPRE, true>,
                         cudaFuncAttributePreferredSharedMemoryCarveout, 45);
    set = true;
  }
  int per_sm = 0;
  const bool direct = core_direct(p);
  cudaError_t oc = direct
      ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, core_rows_quad_kernel<SSE, NPRE, true>,
                                                      cquad::WPB * 32, cquad::direct_bytes())
      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, core_rows_quad_kernel<SSE, NPRE>,
                                                      cquad::WPB * 32, sm);
  if (oc != cudaSuccess || per_sm < 1) per_sm = 1;
  int64_t g = (p.nrows + 4 * cquad::WPB - 1) / (4 * cquad::WPB);
  const int64_t cap = (int64_t)sm_count() * per_sm;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

template <bool SSE = false>
int core_quad_grid(const SweepParams &p) {
  switch (p.N) {
    case 3: return core_quad_grid_t<SSE, 1>(p);
    case 4: return core_quad_grid_t<SSE, 2>(p);
    case 5: return core_quad_grid_t<SSE, 3>(p);
    default: return core_quad_grid_t<SSE, 4>(p);
  }
}

template <bool SSE>
int launch_core_quad_t(const SweepParams &p, int g, cudaStream_t s) {
  const bool direct = core_direct(p);
  const dim3 b(cquad::WPB * 32);
  const size_t sm = cquad::bytes(), smd = cquad::direct_bytes();
  switch (p.N) {
    case 3:
      if (direct) core_rows_quad_kernel<SSE, 1, true><<<g, b, smd, s>>>(p);
      else core_rows_quad_kernel<SSE, 1><<<g, b, sm, s>>>(p);
      break;
    case 4:
      if (direct) core_rows_quad_kernel<SSE, 2, true><<<g, b, smd, s>>>(p);
      else core_rows_quad_kernel<SSE, 2><<<g, b, sm, s>>>(p);
      break;
    case 5:
      if (direct) core_rows_quad_kernel<SSE, 3, true><<<g, b, smd, s>>>(p);
      else core_rows_quad_kernel<SSE, 3><<<g, b, sm, s>>>(p);
      break;
    default:
      if (direct) core_rows_quad_kernel<SSE, 4, true><<<g, b, smd, s>>>(p);
      else core_rows_quad_kernel<SSE, 4><<<g, b, sm, s>>>(p);
      break;
  }
  return check_launch(SSE ? "ft_sse_tree" : "ft_core_sweep_rows(quad)");
}

int launch_core_quad(const SweepParams &p, int g, cudaStream_t s) {
  return launch_core_quad_t<false>(p, g, s);
}

__global__ void sum_pairs_f64(const double *__restrict__ partials, int nblocks, double *out2) {
  if (threadIdx.x == 0) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < nblocks; ++k) {
      a += partials[2 * k];
      b += partials[2 * k + 1];
    }
    out2[0] = a;
    out2[1] = b;
  }
}
