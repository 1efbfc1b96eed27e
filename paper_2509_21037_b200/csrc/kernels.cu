// kernels.cu — the device hot path (sm_100a, FP64).
//
//   prep_panel_kernel /   one CTA per (subdomain, panel wider than 32) / one warp per narrower panel
//   prep_small_kernel     (NPAD = 8/16/32): scatters the panel's CSC values of L into the panel
//                         buffer (dense diagonal block, pruned below-diagonal rows in 64-row chunks,
//                         P:482-494) and replaces the diagonal block by its inverse (recursive
//                         doubling: 8x8 substitutions + DMMA products), so every tile's diagonal solve
//                         becomes a tensor-core product (W mode also forms W_p = L[R_p,p] inv(L_pp)).
//   trsm_smem_kernel      "X init + stepped supernodal TRSM" (SURVEY §8 rows a2+a3): one CTA per
//     <T, GS, YM, MINB>   (subdomain, RHS column tile of T columns).  X strip (rows of the panels of
//                         the tile's reach) in shared memory, or in place in the group strip (GS);
//                         zero + scatter of the permuted B~^T, then per panel
//                         Y = inv(L_pp) X_p and X[R_p] -= L[R_p,p] Y as FP64 DMMA (mma.sync m8n8k4)
//                         tiles.  A producer warp streams the L blocks with cp.async.bulk (TMA bulk
//                         copies) into a byte ring guarded by full/empty mbarriers and passes the step
//                         geometry in per-slot records; consumer warps synchronise per column-block
//                         group; solved rows go straight to the SYRK's group strip.  MINB = 2: the
//                         small-strip tile class at two CTAs per SM.
//   syrk_pair_kernel<G>   "block-sparse SYRK" (row a4): one CTA per G x G output tile (I >= J) of
//                         F' = X^T X, k restricted to rows both group strips hold.
//   apply_*               "explicit apply" (row a6): batched symmetric mat-vec on the lower F' with
//                         the stepped-order gather of lambda and a deterministic scatter-sum.
//   implicit_*            "implicit apply": forward + backward substitution per subdomain
//                         with the staged factor panels, no F.
#include <cuda_runtime.h>

// X init of the global-strip TRSM paths: zero only the rows of the tile's own reach (1) or every
// group-strip row (0)
#ifndef SC_CTA_ZERO_REACH
#define SC_CTA_ZERO_REACH 0  // 1 measured slower for 3D (one panel per thread: cfg3 TRSM 13.9 vs 12.8 ms)
#endif

#include <algorithm>
#include <cstdio>
#include <cstring>

#include "sc_internal.h"

namespace sc {

#define CUDA_TRY(expr)                                                       \
  do {                                                                       \
    cudaError_t e_ = (expr);                                                 \
    if (e_ != cudaSuccess) {                                                 \
      err = std::string(#expr) + ": " + cudaGetErrorString(e_);              \
      return e_ == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA;     \
    }                                                                        \
  } while (0)

// ------------------------------------------------------------------------------------------------
// FP64 tensor-core tile: D(8x8) += A(8x4) B(4x8).  Fragments (PTX ISA, mma.m8n8k4 .f64):
//   a = A[g][t], b = B[t][g], c = {C[g][2t], C[g][2t+1]} with g = lane>>2, t = lane&3.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}

// ---- stored elements of L / X / F': double, or float in the FP32 mode (FP64 arithmetic) ---------
__device__ __forceinline__ double ld_el(const void* p, int64_t i, bool f32) {
  return f32 ? (double)__ldg(static_cast<const float*>(p) + i) : __ldg(static_cast<const double*>(p) + i);
}
template <typename ST>
__device__ __forceinline__ double2 ld2(const ST* p) {
  if constexpr (sizeof(ST) == 8) {
    return *reinterpret_cast<const double2*>(p);
  } else {
    const float2 v = *reinterpret_cast<const float2*>(p);
    return make_double2(v.x, v.y);
  }
}
template <typename ST>
__device__ __forceinline__ void st2(ST* p, double2 v) {
  if constexpr (sizeof(ST) == 8) {
    *reinterpret_cast<double2*>(p) = v;
  } else {
    *reinterpret_cast<float2*>(p) = make_float2((float)v.x, (float)v.y);
  }
}

// ---- mbarrier + bulk async copy (TMA, non-tensor form) ------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// Sticky zero-pivot flags (reset at the start of every assemble / prepare): err[0] = the first
// failing (subdomain + 1, column) of the batch, err[1 + sub] = 1 + the first failing column of `sub`.
__device__ __forceinline__ void flag_zero_pivot(const DevPlan& P, int sub, int col) {
  atomicCAS(P.err, 0ull, ((unsigned long long)(sub + 1) << 32) | (unsigned long long)col);
  atomicCAS(P.err + 1 + sub, 0ull, (unsigned long long)col + 1ull);
}

// ------------------------------------------------------------------------------------------------
// prep: panel buffer = [inv(L_pp) | L[R_p, p] chunks]
// ------------------------------------------------------------------------------------------------
constexpr int kLdT = kMaxPanel + 4;  // smem triangle, column-major [col][row]

constexpr size_t kPrepSmem = 2 * sizeof(double) * kMaxPanel * kLdT;

// Scatter of the CSC values of a panel's columns: diagonal-block entries into the smem triangle D
// (column-major, stride LDD), pruned rows into the panel buffer.  U loads in flight per thread; the
// first batch is issued before the caller's zeroing work so its latency overlaps it.
#ifndef SC_PREP_U
#define SC_PREP_U 8
#endif
template <int U>
struct ScatterBatch {
  double v[U];
  int32_t d[U];
  bool f32 = false;
  __device__ __forceinline__ void load(const void* __restrict__ Lv, const int32_t* __restrict__ dest, int64_t q0,
                                       int64_t end, int nthr) {
#pragma unroll
    for (int u = 0; u < U; u++) {
      const int64_t q = q0 + (int64_t)u * nthr;
      d[u] = INT32_MIN;
      if (q < end) {
        v[u] = ld_el(Lv, q, f32);
        d[u] = __ldg(dest + q);
      }
    }
  }
  template <int LDD>
  __device__ __forceinline__ void store(double* __restrict__ PB, double* D) const {
#pragma unroll
    for (int u = 0; u < U; u++) {
      if (d[u] == INT32_MIN) continue;
      if (d[u] < 0) {
        const int idx = -1 - d[u];
        D[(idx >> 6) * LDD + (idx & 63)] = v[u];
      } else {
        PB[d[u]] = v[u];
      }
    }
  }
};
template <int LDD, int U>
__device__ __forceinline__ void scatter_rest(ScatterBatch<U>& sb, const void* __restrict__ Lv,
                                             const int32_t* __restrict__ dest, double* __restrict__ PB, double* D,
                                             const Panel& pn, int t, int nthr) {
  for (int64_t q0 = pn.csc_begin + t;;) {
    sb.template store<LDD>(PB, D);
    q0 += (int64_t)U * nthr;
    if (q0 >= pn.csc_end) break;
    sb.load(Lv, dest, q0, pn.csc_end, nthr);
  }
}

// Zero the entries of a panel's chunk region that the CSC scatter will not write: everything for
// a relaxed panel (structural zeros of merged supernodes), only the padding (rows past nR in the
// last chunk, columns past kw) for a single-supernode panel, whose pruned rows are all present in
// every column.  Work split over `nthr` threads starting at `t`.
__device__ __forceinline__ void zero_chunk_gaps(double* PB, const Panel& pn, int t, int nthr) {
  if (pn.nchunk == 0) return;
  const int kw4 = pn.kw4;
  double* c0 = PB + pn.buf_off + (int64_t)pn.ldD * kw4;
  if (pn.relaxed) {
    const int64_t len = ((int64_t)(pn.nchunk - 1) * kLdC + pn.ldLast) * kw4;
    double2* z = reinterpret_cast<double2*>(c0);
    for (int64_t q = t; q < len / 2; q += nthr) z[q] = make_double2(0.0, 0.0);
    return;
  }
  const int last_rows = pn.nR - (pn.nchunk - 1) * kChunk;
  for (int ch = 0; ch < pn.nchunk; ch++) {
    const int ld = (ch == pn.nchunk - 1) ? pn.ldLast : kLdC;
    const int rows = (ch == pn.nchunk - 1) ? last_rows : kChunk;
    double* blk = c0 + (int64_t)ch * kLdC * kw4;
    const int gap = ld - rows;  // < 8
    // rows [rows, ld) of columns [0, kw) (8 slots per column, no integer division) and all ld rows
    // of columns [kw, kw4)
    for (int q = t; q < 8 * pn.kw; q += nthr) {
      const int c = q >> 3, r = q & 7;
      if (r < gap) blk[(int64_t)c * ld + rows + r] = 0.0;
    }
    for (int c = pn.kw; c < kw4; c++)
      for (int r = t; r < ld; r += nthr) blk[(int64_t)c * ld + r] = 0.0;
  }
}


// W_p = L[R_p, p] inv(L_pp), in place on the panel's chunks (called after the scatter and the
// inversion, with the scatter's global writes visible to the calling threads): one 8-row block of
// one chunk per warp item; the whole row block is loaded before it is overwritten.  Winv: inverse
// in shared memory, column-major with stride LDW (zero above the diagonal, unit padding).
template <int LDW, int NPAD>
__device__ __forceinline__ void chunks_times_inverse(double* __restrict__ PB, const Panel& pn, const double* Winv,
                                                     int item0, int nitem_step, int lane) {
  if (pn.nchunk == 0) return;
  // RB row blocks per pass (their loads in flight together); k outer, column blocks inner (NPAD / 8
  // independent accumulator chains)
  constexpr int RB = NPAD == 64 ? 1 : 4;
  constexpr int KSN = NPAD / 4, NCB = NPAD / 8;
  const int g = lane >> 2, t4 = lane & 3;
  const int kw4 = pn.kw4;
  double* c0 = PB + pn.buf_off + (int64_t)pn.ldD * kw4;
  const int nitems = pn.nchunk * 8;
  for (int base = item0; base < nitems; base += RB * nitem_step) {
    double a[RB][KSN];
    double* blk[RB];
    int ld[RB], row[RB];
    bool ok[RB];
#pragma unroll
    for (int r = 0; r < RB; r++) {
      const int item = base + r * nitem_step;
      const int c = item >> 3, rb = item & 7;
      const int rows_c = item < nitems ? min(kChunk, pn.nR - c * kChunk) : 0;
      ld[r] = (c == pn.nchunk - 1) ? pn.ldLast : kLdC;
      blk[r] = c0 + (int64_t)c * kLdC * kw4;
      row[r] = rb * 8 + g;
      ok[r] = row[r] < rows_c;
#pragma unroll
      for (int ks = 0; ks < KSN; ks++) a[r][ks] = (ok[r] && 4 * ks < kw4) ? blk[r][(4 * ks + t4) * ld[r] + row[r]] : 0.0;
    }
    __syncwarp();  // every lane's loads of these rows precede any store into them
#pragma unroll
    for (int r = 0; r < RB; r++) {
      if (!__any_sync(0xffffffffu, ok[r])) continue;
      double acc[NCB][2];
#pragma unroll
      for (int cb = 0; cb < NCB; cb++) acc[cb][0] = acc[cb][1] = 0.0;
#pragma unroll
      for (int ks = 0; ks < KSN; ks++) {
        if (ks % 4 == 0 && 4 * ks >= kw4) break;
        if (4 * ks < kw4) {
#pragma unroll
          for (int cb = 0; cb <= ks / 2 && cb < NCB; cb++)  // inv lower triangular: k >= 8 cb
            dmma(acc[cb][0], acc[cb][1], a[r][ks], Winv[(cb * 8 + g) * LDW + 4 * ks + t4]);
        }
      }
      if (ok[r]) {
#pragma unroll
        for (int cb = 0; cb < NCB; cb++) {
          const int col = cb * 8 + 2 * t4;
          if (col < kw4) {  // kw4 is a multiple of 4, not of 8
            blk[r][col * ld[r] + row[r]] = acc[cb][0];
            blk[r][(col + 1) * ld[r] + row[r]] = acc[cb][1];
          }
        }
      }
    }
  }
}

template <bool WMODE>
__global__ void __launch_bounds__(kThreads) prep_panel_kernel(DevPlan P, int t0) {
  extern __shared__ __align__(16) unsigned char prep_smem[];
  double* D = reinterpret_cast<double*>(prep_smem);  // triangle, then temporaries
  double* W = D + kMaxPanel * kLdT;                  // inverse
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const I2 task = P.prep_tasks[t0 + blockIdx.x];
  const int sub = task.x;
  const Panel pn = P.panels[task.y];
  const int cls = P.sub_cls[sub];
  const int32_t* __restrict__ dest = P.dest + P.cls_csc_off[cls];
  const void* __restrict__ Lv = P.Lptr[sub];
  double* __restrict__ PB = P.PB + P.sub_PB_base[sub];
  const int kw = pn.kw, kw4 = pn.kw4;
  int npad = 8;  // triangle padded to npad = 8 * 2^k >= kw with a unit diagonal
  while (npad < kw) npad *= 2;
  {  // W needs no clearing: every block it is read at is written first (triangular loop bounds)
    double2* D2 = reinterpret_cast<double2*>(D);
    for (int q = tid; q < npad * kLdT / 2; q += kThreads) D2[q] = make_double2(0.0, 0.0);
  }
  ScatterBatch<4> sb;
  sb.f32 = P.fp32;
  sb.load(Lv, dest, pn.csc_begin + tid, pn.csc_end, kThreads);
  // Y mode: every chunk position the scatter does not write (padding, explicit zeros of merged
  // supernodes) is zero since the plan zero-filled the panel buffer and nothing else writes there;
  // W mode overwrites whole chunks with W_p, so their zeros are restored here
  if constexpr (WMODE) zero_chunk_gaps(PB, pn, tid, kThreads);
  __syncthreads();
  scatter_rest<kLdT>(sb, Lv, dest, PB, D, pn, tid, kThreads);
  // unit diagonal in the padding (its inverse stays the identity)
  for (int i = kw + tid; i < npad; i += kThreads) D[i * kLdT + i] = 1.0;
  __syncthreads();
  // inverse of the lower-triangular diagonal block by recursive doubling:
  //   inv([[A, 0], [C, B]]) = [[inv(A), 0], [-inv(B) C inv(A), inv(B)]]
  // level 0: 8x8 diagonal blocks by forward substitution (one warp each); levels 16..npad: the
  // off-diagonal blocks as two DMMA products per pair.  W holds the inverse; D's consumed diagonal
  // squares serve as the temporary C inv(A).
  if (warp * 8 < npad && lane < 8) {
    const int base = warp * 8, j = lane;
    // one division per lane: lane j holds 1 / d_jj, broadcast by shuffles
    const double djj = D[(base + j) * kLdT + base + j];
    if (base + j < kw && (!(djj > 0.0) || !isfinite(djj))) flag_zero_pivot(P, sub, pn.a + base + j);
    const double rj = 1.0 / djj;
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; k++) s -= (k >= j) ? D[(base + k) * kLdT + base + i] * x[k] : 0.0;
      const double ri = __shfl_sync(0xffu, rj, i);  // every lane of the mask shuffles
      x[i] = (i >= j) ? s * ri : 0.0;
    }
#pragma unroll
    for (int i = 0; i < 8; i++) W[(base + j) * kLdT + base + i] = x[i];
  }
  __syncthreads();
  const int g = lane >> 2, t4 = lane & 3;
  for (int b = 16; b <= npad; b *= 2) {
    const int h = b / 2, nbh = h / 8, npairs = npad / b;
    // T1 = C inv(A) -> D[A rows, A cols] (diagonal square of the pair's top block)
    for (int blk = warp; blk < npairs * nbh * nbh; blk += kThreads / 32) {
      const int pr = blk / (nbh * nbh), rem = blk - pr * nbh * nbh, bi = rem % nbh, bj = rem / nbh;
      const int base = pr * b;
      const double* Cm = D + base * kLdT + base + h;  // C: rows base+h.., cols base..
      const double* Ai = W + base * kLdT + base;
      double c0 = 0.0, c1 = 0.0;
      // inv(A) is lower triangular: only k >= 8 bj contributes
      for (int k = bj * 8; k < h; k += 4) dmma(c0, c1, Cm[(k + t4) * kLdT + bi * 8 + g], Ai[(bj * 8 + g) * kLdT + k + t4]);
      double* Tt = D + base * kLdT + base;
      Tt[(bj * 8 + 2 * t4) * kLdT + bi * 8 + g] = c0;
      Tt[(bj * 8 + 2 * t4 + 1) * kLdT + bi * 8 + g] = c1;
    }
    __syncthreads();
    // W[B rows, A cols] = -inv(B) T1
    for (int blk = warp; blk < npairs * nbh * nbh; blk += kThreads / 32) {
      const int pr = blk / (nbh * nbh), rem = blk - pr * nbh * nbh, bi = rem % nbh, bj = rem / nbh;
      const int base = pr * b;
      const double* Bi = W + (base + h) * kLdT + base + h;
      const double* Tt = D + base * kLdT + base;
      double c0 = 0.0, c1 = 0.0;
      // inv(B) is lower triangular: only k < 8 (bi + 1) contributes
      for (int k = 0; k < (bi + 1) * 8; k += 4) dmma(c0, c1, Bi[(k + t4) * kLdT + bi * 8 + g], Tt[(bj * 8 + g) * kLdT + k + t4]);
      double* Wo = W + base * kLdT + base + h;
      Wo[(bj * 8 + 2 * t4) * kLdT + bi * 8 + g] = -c0;
      Wo[(bj * 8 + 2 * t4 + 1) * kLdT + bi * 8 + g] = -c1;
    }
    __syncthreads();
  }
  // write inv(L_pp): ldD x kw4 column-major, zero outside [0,kw) x [0,kw)
  double* Dinv = PB + pn.buf_off;
  const int ldD = pn.ldD;
  // only the lower triangle: the upper triangle and the padding columns stay zero from plan creation
  // (the padding rows are never used)
  for (int j = warp; j < kw; j += kThreads / 32)  // warp per column, lanes over rows
    for (int i = j + lane; i < kw; i += 32) Dinv[j * ldD + i] = W[j * kLdT + i];
  // chunks: L[R_p, p] -> W_p = L[R_p, p] inv(L_pp) (the TRSM's update operand)
  if constexpr (WMODE) chunks_times_inverse<kLdT, kMaxPanel>(PB, pn, W, warp, kThreads / 32, lane);
}


// Panels of <= kSmallPanel columns: one warp per panel (no CTA barriers), same algorithm.  One
// instantiation per padded width NPAD = 8 / 16 / 32 (the planner buckets the tasks), so the
// shared memory per warp is sized to the panel and many more warps stay resident.
template <int NPAD>
struct SmallCfg {
  static constexpr int WARPS = NPAD <= 16 ? 8 : 4;  // warps (panels) per CTA
  static constexpr int LD = NPAD + 4;               // == 4 (mod 8): conflict-free fragment loads
  static constexpr size_t kWarpDoubles = 2 * (size_t)NPAD * LD;
  static constexpr size_t kSmem = sizeof(double) * kWarpDoubles * WARPS;
};

template <int NPAD, bool WMODE>
__global__ void __launch_bounds__(32 * SmallCfg<NPAD>::WARPS) prep_small_kernel(DevPlan P, int t_begin, int t_end) {
  using Cfg = SmallCfg<NPAD>;
  constexpr int LD = Cfg::LD;
  extern __shared__ __align__(16) unsigned char prep_smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int t = t_begin + blockIdx.x * Cfg::WARPS + warp;
  if (t >= t_end) return;
  double* D = reinterpret_cast<double*>(prep_smem) + (size_t)warp * Cfg::kWarpDoubles;
  double* W = D + NPAD * LD;
  const I2 task = P.prep_small_tasks[t];
  const int sub = task.x;
  const Panel pn = P.panels[task.y];
  const int32_t* __restrict__ dest = P.dest + P.cls_csc_off[P.sub_cls[sub]];
  const void* __restrict__ Lv = P.Lptr[sub];
  double* __restrict__ PB = P.PB + P.sub_PB_base[sub];
  const int kw = pn.kw, kw4 = pn.kw4;
  ScatterBatch<SC_PREP_U> sb;
  sb.f32 = P.fp32;
  sb.load(Lv, dest, pn.csc_begin + lane, pn.csc_end, 32);
  for (int q = lane; q < NPAD * LD / 2; q += 32) reinterpret_cast<double2*>(D)[q] = make_double2(0.0, 0.0);
  if constexpr (WMODE) zero_chunk_gaps(PB, pn, lane, 32);  // (Y mode: zero since plan creation)
  __syncwarp();
  scatter_rest<LD>(sb, Lv, dest, PB, D, pn, lane, 32);
  for (int i = kw + lane; i < NPAD; i += 32) D[i * LD + i] = 1.0;
  __syncwarp();
  {  // level 0: lane -> (8x8 block lane/8, column lane%8); all lanes run (blocks past NPAD read a
     // clamped block and store nothing) so the reciprocals can be shuffled with a full mask
    const int base = (lane >> 3) * 8, j = lane & 7;
    const int rb = base < NPAD ? base : 0;
    const double djj = D[(rb + j) * LD + rb + j];
    if (base < NPAD && base + j < kw && (!(djj > 0.0) || !isfinite(djj))) flag_zero_pivot(P, sub, pn.a + base + j);
    const double rj = 1.0 / djj;  // one division per lane, broadcast within the 8-lane group
    double x[8];
#pragma unroll
    for (int i = 0; i < 8; i++) {
      double s = (i == j) ? 1.0 : 0.0;
#pragma unroll
      for (int k = 0; k < i; k++) s -= (k >= j) ? D[(rb + k) * LD + rb + i] * x[k] : 0.0;
      const double ri = __shfl_sync(0xffffffffu, rj, (lane & ~7) + i);  // every lane shuffles
      x[i] = (i >= j) ? s * ri : 0.0;
    }
    if (base < NPAD) {
#pragma unroll
      for (int i = 0; i < 8; i++) W[(base + j) * LD + base + i] = x[i];
    }
  }
  __syncwarp();
  const int g = lane >> 2, t4 = lane & 3;
#pragma unroll
  for (int b = 16; b <= NPAD; b *= 2) {
    const int h = b / 2, nbh = h / 8, npairs = NPAD / b;
    for (int blk = 0; blk < npairs * nbh * nbh; blk++) {
      const int pr = blk / (nbh * nbh), rem = blk - pr * nbh * nbh, bi = rem % nbh, bj = rem / nbh;
      const int base = pr * b;
      const double* Cm = D + base * LD + base + h;
      const double* Ai = W + base * LD + base;
      double c0 = 0.0, c1 = 0.0;
      for (int k = bj * 8; k < h; k += 4) dmma(c0, c1, Cm[(k + t4) * LD + bi * 8 + g], Ai[(bj * 8 + g) * LD + k + t4]);
      double* Tt = D + base * LD + base;
      Tt[(bj * 8 + 2 * t4) * LD + bi * 8 + g] = c0;
      Tt[(bj * 8 + 2 * t4 + 1) * LD + bi * 8 + g] = c1;
    }
    __syncwarp();
    for (int blk = 0; blk < npairs * nbh * nbh; blk++) {
      const int pr = blk / (nbh * nbh), rem = blk - pr * nbh * nbh, bi = rem % nbh, bj = rem / nbh;
      const int base = pr * b;
      const double* Bi = W + (base + h) * LD + base + h;
      const double* Tt = D + base * LD + base;
      double c0 = 0.0, c1 = 0.0;
      for (int k = 0; k < (bi + 1) * 8; k += 4) dmma(c0, c1, Bi[(k + t4) * LD + bi * 8 + g], Tt[(bj * 8 + g) * LD + k + t4]);
      double* Wo = W + base * LD + base + h;
      Wo[(bj * 8 + 2 * t4) * LD + bi * 8 + g] = -c0;
      Wo[(bj * 8 + 2 * t4 + 1) * LD + bi * 8 + g] = -c1;
    }
    __syncwarp();
  }
  double* Dinv = PB + pn.buf_off;
  const int ldD = pn.ldD;
  // only the lower triangle (upper triangle and padding columns stay zero from plan creation): one
  // flat pass over the kw (kw + 1) / 2 packed entries, column j from the packed index
  for (int q = lane; q < kw * (kw + 1) / 2; q += 32) {
    int j = (int)((2.0f * kw + 1.0f - sqrtf((2.0f * kw + 1.0f) * (2.0f * kw + 1.0f) - 8.0f * q)) * 0.5f);
    int c0 = j * kw - j * (j - 1) / 2;  // packed start of column j
    if (q < c0) {
      j--;
      c0 = j * kw - j * (j - 1) / 2;
    } else if (q >= c0 + (kw - j)) {
      c0 += kw - j;
      j++;
    }
    const int i = j + (q - c0);
    Dinv[j * ldD + i] = W[j * LD + i];
  }
  if constexpr (WMODE) chunks_times_inverse<LD, NPAD>(PB, pn, W, 0, 1, lane);
}

// ------------------------------------------------------------------------------------------------
// TRSM with the X strip resident in shared memory (warp-specialised: 8 DMMA consumer warps + one
// TMA producer warp streaming the tile's L blocks through a byte ring with full/empty mbarriers)
// ------------------------------------------------------------------------------------------------
static_assert(kLdC == block_ld(kChunk), "chunk ld");

#ifndef SC_WN16
#define SC_WN16 1
#endif
#ifndef SC_NCW
#define SC_NCW 8
#endif
#ifndef SC_NCW2
#define SC_NCW2 4
#endif
#ifndef SC_KSPLIT
#define SC_KSPLIT 1   // chunk-product accumulator sets per output block, <= 2 blocks per warp
#endif                // (1 / 2 / 4 / 8 measured: fewer is faster, cfg2 TRSM 1.56 / 1.59 / 1.72 / - ms)
#ifndef SC_KSPLIT4
#define SC_KSPLIT4 1  // same for 4 output blocks per warp (T = 32): 1 vs 2 -> cfg4 TRSM 54.5 vs 59.4 ms
#endif
#ifndef SC_CHUNK_PIPE
#define SC_CHUNK_PIPE 0
#endif
#ifndef SC_GEMM1_SPLIT
#define SC_GEMM1_SPLIT 2
#endif
#ifndef SC_WN32
#define SC_WN32 1
#endif
template <int T, int MINB = 1>
struct TileCfg {
  static constexpr int LDX = strip_ld(T);       // strip / Y row stride in doubles
  static constexpr int NB = T / 8;              // 8-wide column blocks
  // 8 consumer warps (16 measured slower: 3.0 vs 2.6 ms cfg2, 17.2 vs 15.5 ms cfg3), one column
  // block each (keeps the register-resident Y fragments small); a 64 x T chunk product is
  // (8 / warp rows) row blocks per warp
  // consumer warps: 8, except 4 for the two-CTAs-per-SM class at T = 16 (cheaper group barriers and
  // no register cap spills: cfg2 TRSM -1.5 %)
  static constexpr int NCW = T == 64 ? 8 : (MINB >= 2 ? SC_NCW2 : (T == 8 ? 8 : SC_NCW));
  static constexpr int CT = NCW * 32;           // consumer threads
  static constexpr int WN = T >= 32 ? SC_WN32 : (T == 16 ? SC_WN16 : 1);  // column blocks per warp
  static constexpr int NWC = NB / WN;           // warps along the columns
  static constexpr int WM = 8 * NWC / NCW;      // row blocks per warp
  static_assert(WM >= 1 && (NCW / NWC) * WM == 8, "warp tiling must cover 64 rows");
  // Column swizzle of the unpadded strip (T >= 16): word (row, col) lives at row*T + (col ^ swz(row))
  // with swz = 0, 8, 4, 12 for row & 3 = 0..3.  DMMA B-fragment loads (rows k..k+3 x 8 columns)
  // and the 16-byte C-fragment stores (rows g, g+1 x 8 columns) are then bank-conflict free.
  // T == 8 keeps a padded stride of 12 (== 12 mod 16) instead.
  static __device__ __forceinline__ int idx(int row, int col) {
    if constexpr (T >= 16) {
      return row * LDX + (col ^ (((row & 1) << 3) | ((row & 2) << 1)));
    } else {
      return row * LDX + col;
    }
  }
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
template <int NT>
__device__ __forceinline__ void consumer_sync() {  // named barrier over the NT consumer threads
  asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
}

// Per-slot record written by the producer before it arms the slot's full barrier (the consumers
// read it after their wait): ring offset of the block and, for a step's first block (inv(L_pp)),
// the step's panel geometry, so the consumers never fetch descriptors from global memory.
struct SlotRec {
  int32_t off, kw, kw4, ldD, nchunk, nR, ldLast, strip_row, grow, pad[3];
};
static_assert(sizeof(SlotRec) == 48, "slot record");

// Producer (the whole warp): walks the tile's block stream [inv(L_pp), chunk 0, chunk 1, ...] per
// step.  Step / panel descriptors are fetched 32 steps at a time (lane l loads step s0 + l, so the
// dependent global loads overlap) and broadcast with shuffles; lane 0 issues each block with
// cp.async.bulk into the byte ring as soon as a slot and the bytes are free.  A chunk block travels
// with its 64 precomputed strip rows (128 B, same mbarrier).
__device__ __noinline__ void trsm_producer(const DevPlan& P, const Tile& tile, const double* PB, unsigned char* ring,
                                           uint64_t* full, uint64_t* empty, SlotRec* rec, uint16_t* srow, int lane,
                                           int ring_bytes) {
  int q_slot[kSlots], q_start[kSlots];  // FIFO of in-flight blocks (identical in every lane)
  int q_head = 0, inflight = 0, ring_head = 0, ring_tail = 0;
  int b = 0;
  for (int s0 = tile.step_begin; s0 < tile.step_end; s0 += 32) {
    Step stl{};
    Panel pnl{};
    if (s0 + lane < tile.step_end) {
      stl = P.steps[s0 + lane];
      pnl = P.panels[stl.panel];
    }
    const int cnt = min(32, tile.step_end - s0);
    for (int k = 0; k < cnt; k++) {
      const int64_t buf_off = __shfl_sync(0xffffffffu, pnl.buf_off, k);
      const int64_t srow_off = __shfl_sync(0xffffffffu, stl.srow_off, k);
      const int kw = __shfl_sync(0xffffffffu, pnl.kw, k), kw4 = __shfl_sync(0xffffffffu, pnl.kw4, k);
      const int ldD = __shfl_sync(0xffffffffu, pnl.ldD, k), nchunk = __shfl_sync(0xffffffffu, pnl.nchunk, k);
      const int nR = __shfl_sync(0xffffffffu, pnl.nR, k), ldLast = __shfl_sync(0xffffffffu, pnl.ldLast, k);
      const int strip_row = __shfl_sync(0xffffffffu, stl.strip_row, k), grow = __shfl_sync(0xffffffffu, stl.grow, k);
      for (int c = -1; c < nchunk; c++, b++) {
        const double* src;
        int bytes;
        if (c < 0) {
          src = PB + buf_off;
          bytes = ldD * kw4 * 8;
        } else {
          src = PB + buf_off + (int64_t)ldD * kw4 + (int64_t)c * kLdC * kw4;
          bytes = ((c == nchunk - 1) ? ldLast : kLdC) * kw4 * 8;
        }
        // wait until a slot and `bytes` contiguous ring bytes are free (pop oldest in-flight blocks)
        int start = 0;
        while (true) {
          bool ok = false;
          if (inflight == 0) {
            ring_head = ring_tail = 0;
            start = 0;
            ok = true;
          } else if (inflight < kSlots) {
            if (ring_tail > ring_head) {
              if (ring_bytes - ring_tail >= bytes) {
                start = ring_tail;
                ok = true;
              } else if (ring_head >= bytes) {
                start = 0;
                ok = true;
              }
            } else if (ring_tail < ring_head && ring_head - ring_tail >= bytes) {
              start = ring_tail;
              ok = true;
            }
          }
          if (ok) break;
          const int os = q_slot[q_head];
          mbar_wait(&empty[os], (uint32_t)((b - inflight) / kSlots) & 1u);
          q_head = (q_head + 1) % kSlots;
          inflight--;
          ring_head = inflight ? q_start[q_head] : ring_tail;
        }
        const int slot = b % kSlots;
        const int qi = (q_head + inflight) % kSlots;
        q_slot[qi] = slot;
        q_start[qi] = start;
        inflight++;
        ring_tail = start + bytes;
        if (lane == 0) {
          SlotRec& r = rec[slot];
          r.off = start;
          if (c < 0) {
            r.kw = kw;
            r.kw4 = kw4;
            r.ldD = ldD;
            r.nchunk = nchunk;
            r.nR = nR;
            r.ldLast = ldLast;
            r.strip_row = strip_row;
            r.grow = grow;
          }
          const uint32_t rb = (c >= 0) ? (uint32_t)(kChunk * sizeof(uint16_t)) : 0u;
          mbar_expect_tx(&full[slot], (uint32_t)bytes + rb);
          bulk_g2s(ring + start, src, (uint32_t)bytes, &full[slot]);
          if (c >= 0) bulk_g2s(srow + slot * kChunk, P.srows + srow_off + (int64_t)c * kChunk, rb, &full[slot]);
        }
      }
    }
  }
}

// GS = false: the X strip lives in shared memory (swizzled, written out into the group strip at
// the end).  GS = true ("global strip", subdomains whose strips do not fit on chip, e.g. cfg5): the
// tile solves in place in its T columns of the SYRK group strip in global memory (row-major, G
// wide, L2-resident while the tile runs); the strip rows of the plan are then group-strip rows.
// MINB: CTAs per SM the launch is built for (2: the small-strip tile class, registers capped)
template <int T, bool GS, bool YM, int MINB = 1>
__global__ void __launch_bounds__(TileCfg<T, MINB>::CT + 32, MINB) trsm_smem_kernel(DevPlan P, TrsmLaunch Lc) {
  using Cfg = TileCfg<T, MINB>;
  constexpr int WM = Cfg::WM, WN = Cfg::WN, NWC = Cfg::NWC, CT = Cfg::CT;
  constexpr int KS = kMaxPanel / 4;  // k steps of 4 in a full panel
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const TrsmSmem L = trsm_smem_layout(T, Lc.ring_bytes, Lc.strip_cap, GS, YM);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + L.full);
  uint64_t* empty = reinterpret_cast<uint64_t*>(smem_raw + L.empty);
  SlotRec* rec = reinterpret_cast<SlotRec*>(smem_raw + L.off);
  uint16_t* srow = reinterpret_cast<uint16_t*>(smem_raw + L.srow);
  unsigned char* ring = smem_raw + L.ring;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const I2 task = P.trsm_tasks[Lc.task0 + blockIdx.x];
  const int sub = task.x;
  const Tile tile = P.tiles[task.y];
  const double* __restrict__ PB = P.PB + P.sub_PB_base[sub];
  double* Xs;
  float* Xf = nullptr;  // global strip of an FP32 plan
  const bool f32 = GS && P.fp32;
  int LDX;
  if constexpr (GS) {
    const int64_t off = P.sub_X_base[sub] + P.groups[tile.group].x_off + tile.col_in_group;
    Xs = static_cast<double*>(P.X) + off;
    Xf = static_cast<float*>(P.X) + off;
    LDX = P.G;
  } else {
    Xs = reinterpret_cast<double*>(smem_raw + L.strip);
    LDX = Cfg::LDX;
  }
  // element (row, col) of the strip
  auto xi = [&](int row, int col) -> int {
    if constexpr (GS) {
      return row * LDX + col;
    } else {
      return Cfg::idx(row, col);
    }
  };
  // strip element access (the global strip of an FP32 plan holds floats)
  auto xld = [&](int e) -> double { return f32 ? (double)Xf[e] : Xs[e]; };
  auto xld2 = [&](int e) -> double2 { return f32 ? ld2(Xf + e) : ld2(Xs + e); };
  auto xst2 = [&](int e, double2 v) {
    if (f32) st2(Xf + e, v);
    else st2(Xs + e, v);
  };

  if (tid == 0) {
    for (int k = 0; k < kSlots; k++) {
      mbar_init(&full[k], 1);
      mbar_init(&empty[k], Cfg::NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  if (warp == Cfg::NCW) {  // ---- TMA producer warp
    trsm_producer(P, tile, PB, ring, full, empty, rec, srow, lane, Lc.ring_bytes);
    return;
  }

  // ---- consumers.  X init (row a2): zero the strip (+4 pad rows), scatter B~^T
  const int g = lane >> 2, t4 = lane & 3;
  const int br0 = (warp / NWC) * WM, bc0 = (warp % NWC) * WN;
  if constexpr (GS) {
#if SC_CTA_ZERO_REACH
    // the tile's T columns of the group-strip rows of its own reach (one step's panel per thread);
    // the group's other rows are never written in these columns and stay zero from the allocation
    for (int s = tile.step_begin + tid; s < tile.step_end; s += CT) {
      const Step st = P.steps[s];
      const int nr = P.panels[st.panel].kw;
      for (int r = 0; r < nr; r++)
#pragma unroll
        for (int j = 0; j < T; j += 2) xst2((st.strip_row + r) * LDX + j, make_double2(0.0, 0.0));
    }
#else
    for (int q = tid; q < tile.strip_rows * (T / 2); q += CT) {  // the tile's T columns of every group-strip row
      const int r = q / (T / 2), j = 2 * (q - r * (T / 2));
      xst2(r * LDX + j, make_double2(0.0, 0.0));
    }
#endif
  } else {
    double2* X2 = reinterpret_cast<double2*>(Xs);
    const int nvec = (tile.strip_rows + 4) * LDX / 2;
    for (int q = tid; q < nvec; q += CT) X2[q] = make_double2(0.0, 0.0);
  }
  consumer_sync<CT>();
  for (int q = tile.binit_begin + tid; q < tile.binit_end; q += CT) {
    const BInit bi = P.binit[q];
    if (f32) Xf[xi(bi.strip_row, bi.col)] = (float)bi.val;
    else Xs[xi(bi.strip_row, bi.col)] = bi.val;
  }
  consumer_sync<CT>();

  // ---- stepped supernodal TRSM (row a3).  With W_p = L[R_p, p] inv(L_pp) prepared once per
  // subdomain, step p is two independent products of the SAME operand X_p (final after the earlier
  // steps):  X_p <- inv(L_pp) X_p  and  X[R_p] -= W_p X_p.  No barrier separates them; the solved
  // rows go straight to the group strip in HBM (they are never read again by this tile), and one
  // barrier per step among the warps of a column block orders the R_p updates before the next
  // panel reads its rows.
  const int cgrp = warp % NWC;  // column-block group: the warps that touch these T / NWC columns
  auto group_sync = [&]() {
    if constexpr (NWC == 1) {
      consumer_sync<CT>();
    } else {
      asm volatile("bar.sync %0, %1;\n" ::"r"(2 + cgrp), "n"(CT / NWC) : "memory");  // ids 2..9
    }
  };
  double* Ys = reinterpret_cast<double*>(smem_raw + L.ys);  // Y mode only: 64 x LDX, swizzled
  Group Gt;
  int64_t xg_off = 0;           // this tile's columns of its group strip (shared-strip mode)
  if constexpr (!GS) {
    Gt = P.groups[tile.group];
    xg_off = P.sub_X_base[sub] + Gt.x_off + tile.col_in_group;
  }
  int b = 0;  // block counter (same order as the producer)
  for (int s = tile.step_begin; s < tile.step_end; s++, b++) {
    // the step's geometry arrives with its first block (inv(L_pp))
    const int slot0 = b % kSlots;
    mbar_wait(&full[slot0], (uint32_t)(b / kSlots) & 1u);
    const SlotRec pn = rec[slot0];
    const int kw = pn.kw, kw4 = pn.kw4;
    const int row0 = pn.strip_row;
    // B operand: X_p (rows row0 + 4 ks + t4 share (row & 3), hence one swizzled column per j).  A
    // global strip has no zero pad rows past the last panel: rows >= kw are read as 0.
    double yf[KS][WN];
    {
      const int xb = (row0 + t4) * LDX;
#pragma unroll
      for (int j = 0; j < WN; j++) {
        const int xcol = xi(row0 + t4, (bc0 + j) * 8 + g) - (row0 + t4) * LDX;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
          if (ks % 4 == 0 && 4 * ks >= kw4) break;
          yf[ks][j] = (4 * ks < kw4 && (!GS || 4 * ks + t4 < kw)) ? xld(xb + (4 * ks) * LDX + xcol) : 0.0;
        }
      }
    }
    // X_p <- inv(L_pp) X_p for this warp's row blocks (inv lower triangular: row block i needs
    // k < 8 (i + 1)); kept in registers until the step's barrier
    double yn[WM][WN][2];
    {
      constexpr int YS = MINB >= 2 ? 1 : SC_GEMM1_SPLIT;  // accumulator sets (k steps round-robin)
      double ya[YS][WM][WN][2];
#pragma unroll
      for (int h = 0; h < YS; h++)
#pragma unroll
        for (int i = 0; i < WM; i++)
#pragma unroll
          for (int j = 0; j < WN; j++) ya[h][i][j][0] = ya[h][i][j][1] = 0.0;
      const int slot = slot0;
      const double* A = reinterpret_cast<const double*>(ring + pn.off);
      const int ld = pn.ldD;
      const int kend = min(kw4, (br0 + WM) * 8);
      if (br0 * 8 < kw4) {
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
          if (ks % 4 == 0 && 4 * ks >= kend) break;
          if (4 * ks < kend) {
            double a[WM];
#pragma unroll
            for (int i = 0; i < WM; i++) a[i] = A[(4 * ks + t4) * ld + (br0 + i) * 8 + g];
#pragma unroll
            for (int i = 0; i < WM; i++)
#pragma unroll
              for (int j = 0; j < WN; j++) dmma(ya[ks % YS][i][j][0], ya[ks % YS][i][j][1], a[i], yf[ks][j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
#pragma unroll
      for (int i = 0; i < WM; i++)
#pragma unroll
        for (int j = 0; j < WN; j++) {
          yn[i][j][0] = ya[0][i][j][0];
          yn[i][j][1] = ya[0][i][j][1];
#pragma unroll
          for (int h = 1; h < YS; h++) {
            yn[i][j][0] += ya[h][i][j][0];
            yn[i][j][1] += ya[h][i][j][1];
          }
        }
    }
    if constexpr (YM) {
      // Y mode: the update operand is L[R_p, p] itself, so the chunks need the solved Y = X_p(new):
      // exchanged through Ys among the warps of the column-block group, then held as B fragments
#pragma unroll
      for (int i = 0; i < WM; i++) {
        const int r = (br0 + i) * 8 + g;
#pragma unroll
        for (int j = 0; j < WN; j++)
          if (r < kw4)
            *reinterpret_cast<double2*>(Ys + Cfg::idx(r, (bc0 + j) * 8 + 2 * t4)) = make_double2(yn[i][j][0], yn[i][j][1]);
      }
      group_sync();
#pragma unroll
      for (int j = 0; j < WN; j++) {
        const double* yb = Ys + Cfg::idx(t4, (bc0 + j) * 8 + g);  // rows 4 ks + t4 share the swizzle
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
          if (ks % 4 == 0 && 4 * ks >= kw4) break;
          yf[ks][j] = (4 * ks < kw4) ? yb[4 * ks * Cfg::LDX] : 0.0;
        }
      }
    }
    // X[R_p] -= W_p X_p (W mode) or L[R_p, p] Y (Y mode), one 64-row chunk (one ring block) at a
    // time; chunks update disjoint rows and each warp releases its ring slot itself.  Software
    // pipelined over chunk pairs: the read-modify-write of chunk c - 1 runs while the tensor cores
    // work on chunk c (two accumulator sets, no register copies).
    // (pipelined only where registers allow: 2 output blocks per warp, one CTA per SM)
    constexpr bool PIPE = SC_CHUNK_PIPE && (WM * WN <= 2) && MINB == 1;
    constexpr int KSPLIT = PIPE ? 2 : ((WM * WN <= 2) ? SC_KSPLIT : SC_KSPLIT4);
    struct ChunkAcc {
      double acc[KSPLIT][WM][WN][2];
      double2 xold[WM][WN];
      int sr[WM];
      bool on;
    };
    auto issue = [&](int c, ChunkAcc& R) {
      b++;
      const int rows_c = min(kChunk, pn.nR - c * kChunk);
      const int ld = (c == pn.nchunk - 1) ? pn.ldLast : kLdC;
      const int slot = b % kSlots;
      mbar_wait(&full[slot], (uint32_t)(b / kSlots) & 1u);
      const double* A = reinterpret_cast<const double*>(ring + rec[slot].off);
#pragma unroll
      for (int i = 0; i < WM; i++) R.sr[i] = (int)srow[slot * kChunk + (br0 + i) * 8 + g];
      R.on = br0 * 8 < rows_c;
      if constexpr (GS) {  // global strip: fetch the rows to update before the products
        if (R.on) {
#pragma unroll
          for (int i = 0; i < WM; i++)
#pragma unroll
            for (int j = 0; j < WN; j++)
              R.xold[i][j] = (R.sr[i] == 0xFFFF) ? make_double2(0.0, 0.0) : xld2(xi(R.sr[i], (bc0 + j) * 8 + 2 * t4));
        }
      }
      if (R.on) {
#pragma unroll
        for (int h = 0; h < KSPLIT; h++)
#pragma unroll
          for (int i = 0; i < WM; i++)
#pragma unroll
            for (int j = 0; j < WN; j++) R.acc[h][i][j][0] = R.acc[h][i][j][1] = 0.0;
#pragma unroll
        for (int ks = 0; ks < KS; ks++) {
          if (ks % 4 == 0 && 4 * ks >= kw4) break;  // warp-uniform exit per group of 4 k steps
          if (4 * ks < kw4) {
            double a[WM];
#pragma unroll
            for (int i = 0; i < WM; i++) a[i] = A[(4 * ks + t4) * ld + (br0 + i) * 8 + g];
#pragma unroll
            for (int i = 0; i < WM; i++)
#pragma unroll
              for (int j = 0; j < WN; j++)
                dmma(R.acc[ks % KSPLIT][i][j][0], R.acc[ks % KSPLIT][i][j][1], a[i], yf[ks][j]);
          }
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    };
    auto finish = [&](ChunkAcc& R) {
      if (!R.on) return;
#pragma unroll
      for (int i = 0; i < WM; i++) {
        if (R.sr[i] == 0xFFFF) continue;  // row outside this tile's reach (or padding): update is 0
#pragma unroll
        for (int j = 0; j < WN; j++) {
          double s0 = R.acc[0][i][j][0], s1 = R.acc[0][i][j][1];
#pragma unroll
          for (int h = 1; h < KSPLIT; h++) {
            s0 += R.acc[h][i][j][0];
            s1 += R.acc[h][i][j][1];
          }
          const int e = xi(R.sr[i], (bc0 + j) * 8 + 2 * t4);
          double2 v;
          if constexpr (GS) {
            v = R.xold[i][j];
          } else {
            v = *reinterpret_cast<const double2*>(Xs + e);
          }
          v.x -= s0;
          v.y -= s1;
          if constexpr (GS) {
            xst2(e, v);
          } else {
            *reinterpret_cast<double2*>(Xs + e) = v;
          }
        }
      }
    };
    if constexpr (PIPE) {
      ChunkAcc S0, S1;
      for (int c = 0; c < pn.nchunk; c += 2) {
        issue(c, S0);
        if (c >= 1) finish(S1);  // chunk c - 1
        if (c + 1 < pn.nchunk) issue(c + 1, S1);
        finish(S0);
      }
      if (pn.nchunk > 0 && (pn.nchunk & 1) == 0) finish(S1);
    } else {
      ChunkAcc S0;
      for (int c = 0; c < pn.nchunk; c++) {
        issue(c, S0);
        finish(S0);
      }
    }
    // the column-block group's R_p updates are visible before the next panel reads its rows, and
    // every warp of the group has read X_p: store the solved rows (final) into the group strip
    group_sync();
#pragma unroll
    for (int i = 0; i < WM; i++) {
      const int r = (br0 + i) * 8 + g;
      if (r < kw) {
#pragma unroll
        for (int j = 0; j < WN; j++) {
          const double2 v = make_double2(yn[i][j][0], yn[i][j][1]);
          if constexpr (GS) {
            xst2(xi(row0 + r, (bc0 + j) * 8 + 2 * t4), v);
          } else {
            const int64_t e = xg_off + (int64_t)(pn.grow + r) * P.G + (bc0 + j) * 8 + 2 * t4;
            if (P.fp32) st2(static_cast<float*>(P.X) + e, v);
            else st2(static_cast<double*>(P.X) + e, v);
          }
        }
      }
    }
  }
}


// ------------------------------------------------------------------------------------------------
// Warp TRSM (rows a1+a2+a3 fused for narrow panels, e.g. 2D): one warp per (subdomain, tile of
// T = 8 NB columns), no CTA barriers, no prep.  The tile's X strip lives in its T columns of the
// SYRK group strip (global memory, L2-resident while the tile runs).  Per step (factor panel p in
// the tile's reach, kw <= 32):
//   X_p <- L_pp^{-1} X_p   blocked by 8: each 8x8 diagonal block by substitution in registers
//                          (lanes = (row g, column pair 2t)), the blocks below by DMMA;
//   X[R_p] -= L[R_p,p] X_p DMMA over 8-row blocks of the pruned rows R_p, read-modify-write of the
//                          strip rows (row map = the group strip's srows).
// Every A fragment is gathered straight from the caller's CSC values through the plan's fragment
// gather map (Panel::gx_off), so L crosses HBM once and nothing is staged.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(void* dst, const void* src, int src_bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(smem_u32(dst)), "l"(src), "r"(src_bytes)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <typename ST>
__device__ __forceinline__ double gather_l(const ST* __restrict__ Lv, int32_t q) {
  return q >= 0 ? (double)__ldg(Lv + q) : 0.0;
}

#ifndef SC_WARP_ZERO_REACH
#define SC_WARP_ZERO_REACH 1
#endif
#ifndef SC_WARP_WPC
#define SC_WARP_WPC 1  // warps (tiles) per CTA (1: a finished warp frees its slot at once; 4 measured 4 % slower)
#endif
#ifndef SC_WARP_PER_SM
#define SC_WARP_PER_SM 12  // resident warps per SM the registers are sized for: no spills at 168 registers
                           // (measured, 4-warp CTAs: cfg2 TRSM 1.15 ms at 12 warps vs 1.24 at 16, 1.54 at 20)
#endif
constexpr int kWarpTri = 10 * 64;  // staged triangle values per warp: <= 10 8x8 blocks (kw <= 32)


template <int BYTES>
__device__ __forceinline__ void cp_async_el(void* dst, const void* src, int src_bytes) {  // 4 or 8 bytes
  asm volatile("cp.async.ca.shared.global [%0], [%1], %2, %3;\n" ::"r"(smem_u32(dst)), "l"(src), "n"(BYTES),
               "r"(src_bytes)
               : "memory");
}

// Warp TRSM staging buffer Ys (32 rows of the tile's T columns): NB = 2 rows are 16 doubles (128 B)
// with the 16-byte units XOR-swizzled by row (unit ^ (4 (row & 1) | (row & 2))), so the B-fragment
// reads (rows 4ks + t, column 8j + g), the C-fragment double2 accesses (row 8K + g, columns 8j + 2t),
// the row-wise cp.async / double2 copies and the column-per-lane triangle reads are all free of bank
// conflicts; NB = 1 keeps a padded row of 12 doubles.
template <int NB>
__device__ __forceinline__ int ysi(int row, int col) {
  if constexpr (NB == 2) return row * 16 + ((((col >> 1) ^ (((row & 1) << 2) | (row & 2))) << 1) | (col & 1));
  else return row * 12 + col;
}
template <int NB>
__host__ __device__ constexpr int ys_ld() { return NB == 2 ? 16 : 12; }

// R maps of a batch (lane-contiguous int2 per pair of k steps) and its strip rows
template <int KSMAX, int NRBB>
__device__ __forceinline__ void warp_r_idx(const int32_t* __restrict__ gr, const uint16_t* __restrict__ srw, int R0,
                                           int nRB, int KS, int lane, int2 (&q)[8], int (&row)[4]) {
  const int g = lane >> 2;
#pragma unroll
  for (int r = 0; r < NRBB; r++) {
    const bool on = R0 + r < nRB;
    row[r] = on ? (int)__ldg(srw + 8 * (R0 + r) + g) : 0xFFFF;
    const int2* gi = reinterpret_cast<const int2*>(gr) + (int64_t)(R0 + r) * (KS / 2) * 32 + lane;
#pragma unroll
    for (int k2 = 0; k2 < KSMAX / 2; k2++) q[r * (KSMAX / 2) + k2] = (on && 2 * k2 < KS) ? __ldg(gi + 32 * k2) : make_int2(-1, -1);
  }
}
// R-row update (X[R_p] -= L[R_p, p] Y) in batches of NRBB 8-row blocks (KS <= KSMAX k steps).
// q / row hold the batch's gather map / row map (loaded during the previous batch or before the
// triangle solve); per batch: gather the L values (HBM) and the old X rows (L2), load the next
// batch's maps, D = X - L Y by DMMA with Y's B fragments from shared memory, store.  (Measured and
// dropped: the next batch's L values gathered before this batch's DMMAs, the first batch's before the
// triangle solve, the step's maps staged in shared memory -- the kernel is bound by the L1 data
// pipe, not by the latency those hide.)
template <int NB, int KSMAX, int NRBB, typename ST>
__device__ __forceinline__ void warp_r_run(const ST* __restrict__ Lv, const int32_t* __restrict__ gr,
                                          const uint16_t* __restrict__ srw, ST* __restrict__ Xs, const int G,
                                          const double* __restrict__ Ys, const int nRB, const int KS, const int lane,
                                          int2 (&q)[8], int (&row)[4]) {
  const int g = lane >> 2, t = lane & 3;
  for (int R0 = 0; R0 < nRB; R0 += NRBB) {
    double a[NRBB][KSMAX];
    double2 xo[NRBB][NB];
    int rc[NRBB];
#pragma unroll
    for (int r = 0; r < NRBB; r++) {
      rc[r] = row[r];
#pragma unroll
      for (int k2 = 0; k2 < KSMAX / 2; k2++) {
        a[r][2 * k2] = -gather_l(Lv, q[r * (KSMAX / 2) + k2].x);
        a[r][2 * k2 + 1] = -gather_l(Lv, q[r * (KSMAX / 2) + k2].y);
      }
#pragma unroll
      for (int j = 0; j < NB; j++)
        xo[r][j] = rc[r] != 0xFFFF ? ld2(Xs + (int64_t)rc[r] * G + 8 * j + 2 * t) : make_double2(0.0, 0.0);
    }
    if (R0 + NRBB < nRB) warp_r_idx<KSMAX, NRBB>(gr, srw, R0 + NRBB, nRB, KS, lane, q, row);
#pragma unroll
    for (int ks = 0; ks < KSMAX; ks++) {
      if (ks >= KS) break;
#pragma unroll
      for (int j = 0; j < NB; j++) {
        const double b = Ys[ysi<NB>(4 * ks + t, 8 * j + g)];
#pragma unroll
        for (int r = 0; r < NRBB; r++) dmma(xo[r][j].x, xo[r][j].y, a[r][ks], b);
      }
    }
#pragma unroll
    for (int r = 0; r < NRBB; r++)
      if (rc[r] != 0xFFFF) {
#pragma unroll
        for (int j = 0; j < NB; j++) st2(Xs + (int64_t)rc[r] * G + 8 * j + 2 * t, xo[r][j]);
      }
  }
}

// Gathers of a panel's triangle values (fragment order) into Ts with cp.async (no registers held
// while they travel; structural zeros zero-filled).
template <typename ST>
__device__ __forceinline__ void warp_tri_gather(const ST* __restrict__ Lv, const int2 (&q)[10], int ntb, ST* Ts,
                                                int lane) {
  constexpr int B = sizeof(ST);
#pragma unroll
  for (int b = 0; b < 10; b++)
    if (b < ntb) {
      cp_async_el<B>(Ts + 64 * b + lane, Lv + (q[b].x >= 0 ? q[b].x : 0), q[b].x >= 0 ? B : 0);
      cp_async_el<B>(Ts + 64 * b + 32 + lane, Lv + (q[b].y >= 0 ? q[b].y : 0), q[b].y >= 0 ? B : 0);
    }
}
__device__ __forceinline__ void warp_tri_idx(const int32_t* __restrict__ gx, int ntb, int lane, int2 (&q)[10]) {
#pragma unroll
  for (int b = 0; b < 10; b++) q[b] = b < ntb ? __ldg(reinterpret_cast<const int2*>(gx + 64 * b) + lane) : make_int2(-1, -1);
}

// One warp per (subdomain, tile), software-pipelined over the tile's steps: the next panel's
// descriptors and triangle gather map are loaded during the current step and its triangle values are
// gathered (cp.async) as soon as the current triangle is solved; the first R batch's maps are
// loaded before the triangle solve.  Per warp shared memory: X_p / Y (32 x LDY), the triangle
// values (block b, k step s: Ts[64 b + 32 s + lane]) and the reciprocal pivots.
__device__ __forceinline__ WStep ld_wstep(const WStep* p) {
  const int4 u = __ldg(reinterpret_cast<const int4*>(p)), v = __ldg(reinterpret_cast<const int4*>(p) + 1);
  WStep w;
  w.strip_row = u.x, w.a = u.y, w.kw = u.z, w.nR = u.w;
  w.gx_off = (int64_t)(((uint64_t)(uint32_t)v.y << 32) | (uint32_t)v.x);
  w.srow_off = (int64_t)(((uint64_t)(uint32_t)v.w << 32) | (uint32_t)v.z);
  return w;
}
template <int NB, typename ST>
__global__ void __launch_bounds__(32 * SC_WARP_WPC, SC_WARP_PER_SM / SC_WARP_WPC) trsm_warp_kernel(DevPlan P, int t0, int ntask) {
  constexpr int T = 8 * NB, LDY = ys_ld<NB>();
  __shared__ __align__(16) double wsm[SC_WARP_WPC][32 * LDY + kWarpTri + 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int wt = blockIdx.x * SC_WARP_WPC + wid;
  if (wt >= ntask) return;
  double* __restrict__ Ys = wsm[wid];
  ST* __restrict__ Ts = reinterpret_cast<ST*>(Ys + 32 * LDY);  // triangle values as stored (ST)
  double* __restrict__ Rv = Ys + 32 * LDY + kWarpTri;
  const I2 task = P.trsm_tasks[t0 + wt];
  const int sub = task.x;
  const Tile tile = P.tiles[task.y];
  const ST* __restrict__ Lv = static_cast<const ST*>(P.Lptr[sub]);
  const int G = P.G;
  ST* __restrict__ Xs = static_cast<ST*>(P.X) + P.sub_X_base[sub] + P.groups[tile.group].x_off + tile.col_in_group;
  const int g = lane >> 2, t = lane & 3;
  constexpr int VPR = T / 2, RPI = 32 / VPR;  // double2 per strip row, rows per warp instruction
  const int vr0 = lane / VPR, vc2 = 2 * (lane % VPR);
  WStep ws_n{}, ws_nn{};  // descriptors of the next two steps
  int2 qt[10];
  if (tile.step_begin < tile.step_end) {
    ws_n = ld_wstep(P.wsteps + tile.step_begin);
    if (tile.step_begin + 1 < tile.step_end) ws_nn = ld_wstep(P.wsteps + tile.step_begin + 1);
    const int k8 = (ws_n.kw + 7) >> 3;
    warp_tri_idx(P.gidx + ws_n.gx_off, k8 * (k8 + 1) / 2, lane, qt);
    warp_tri_gather(Lv, qt, k8 * (k8 + 1) / 2, Ts, lane);
  }
  // X init (row a2): zero the tile's columns of the group-strip rows of its own reach (the panels it
  // visits; the group's other rows are never written in these columns and stay zero from the
  // allocation), scatter B~^T
#if SC_WARP_ZERO_REACH
  for (int s0 = tile.step_begin; s0 < tile.step_end; s0 += 32) {
    int r0 = 0, nr = 0;
    if (s0 + lane < tile.step_end) {
      const WStep w = ld_wstep(P.wsteps + s0 + lane);
      r0 = w.strip_row;
      nr = w.kw;
    }
    const int ns = min(32, tile.step_end - s0);
    for (int j = 0; j < ns; j++) {
      const int rj = __shfl_sync(0xffffffffu, r0, j), nj = __shfl_sync(0xffffffffu, nr, j);
      for (int r = vr0; r < nj; r += RPI) st2(Xs + (int64_t)(rj + r) * G + vc2, make_double2(0.0, 0.0));
    }
  }
#else
  for (int r = vr0; r < tile.strip_rows; r += RPI) st2(Xs + (int64_t)r * G + vc2, make_double2(0.0, 0.0));
#endif
  __syncwarp();
  for (int q = tile.binit_begin + lane; q < tile.binit_end; q += 32) {
    const BInit bi = P.binit[q];
    Xs[(int64_t)bi.strip_row * G + bi.col] = (ST)bi.val;
  }
  __syncwarp();
  for (int s = tile.step_begin; s < tile.step_end; s++) {
    const WStep st = ws_n;
    const int kw = st.kw, kw8 = (kw + 7) >> 3, KS = 2 * kw8;
    const int32_t* __restrict__ gx = P.gidx + st.gx_off;
    ST* __restrict__ xp = Xs + (int64_t)st.strip_row * G;
    // X_p -> Ys (rows kw..8 kw8 zero-filled): cp.async for FP64 strips, converting loads for FP32
    if constexpr (sizeof(ST) == 8) {
      for (int r = vr0; r < 8 * kw8; r += RPI)
        cp_async16(Ys + ysi<NB>(r, vc2), xp + (int64_t)(r < kw ? r : 0) * G + vc2, r < kw ? 16 : 0);
    } else {
      for (int r = vr0; r < 8 * kw8; r += RPI)
        *reinterpret_cast<double2*>(Ys + ysi<NB>(r, vc2)) = r < kw ? ld2(xp + (int64_t)r * G + vc2) : make_double2(0.0, 0.0);
    }
    cp_async_commit();
    const bool more = s + 1 < tile.step_end;
    if (more) {  // next step's triangle gather map (its descriptor was loaded a step earlier), and the
                 // descriptor of the step after it
      ws_n = ws_nn;
      const int k8 = (ws_n.kw + 7) >> 3;
      warp_tri_idx(P.gidx + ws_n.gx_off, k8 * (k8 + 1) / 2, lane, qt);
      if (s + 2 < tile.step_end) ws_nn = ld_wstep(P.wsteps + s + 2);
    }
    // first R batch's maps (they travel during the triangle solve)
    const int nRB = (st.nR + 7) >> 3;
    const int32_t* __restrict__ gr = gx + 64 * (kw8 * (kw8 + 1) / 2);
    const uint16_t* __restrict__ srw = P.srows + st.srow_off;
    int2 qr[8];
    int rr[4];
    if (KS <= 4) warp_r_idx<4, 4>(gr, srw, 0, nRB, KS, lane, qr, rr);
    else warp_r_idx<8, 2>(gr, srw, 0, nRB, KS, lane, qr, rr);
    cp_async_wait<0>();  // this step's triangle values (issued during the previous step) and X_p
    __syncwarp();
    {  // reciprocal pivots, one row per lane
      const int K = lane >> 3, gg = lane & 7;
      const bool live = lane < kw;
      const double d = live ? (double)Ts[64 * warp_tri_block(K, K, kw8) + 32 * (gg >> 2) + 4 * gg + (gg & 3)] : 1.0;
      if (live && (!(d > 0.0) || !isfinite(d))) flag_zero_pivot(P, sub, st.a + lane);
      Rv[lane] = live ? 1.0 / d : 0.0;
    }
    __syncwarp();
    // X_p <- L_pp^{-1} X_p over 8-row blocks K: X_K -= L_KJ Y_J (J < K, DMMA on C fragments), then
    // the 8x8 diagonal block by substitution, one column per lane (L entries broadcast from Ts)
    for (int K = 0; K < kw8; K++) {
      if (K > 0) {
        double2 x[NB];
#pragma unroll
        for (int j = 0; j < NB; j++) x[j] = *reinterpret_cast<const double2*>(Ys + ysi<NB>(8 * K + g, 8 * j + 2 * t));
        for (int J = 0; J < K; J++) {
          const ST* tb = Ts + 64 * warp_tri_block(J, K, kw8);
          const double a0 = -(double)tb[lane], a1 = -(double)tb[32 + lane];
#pragma unroll
          for (int j = 0; j < NB; j++) {
            dmma(x[j].x, x[j].y, a0, Ys[ysi<NB>(8 * J + t, 8 * j + g)]);
            dmma(x[j].x, x[j].y, a1, Ys[ysi<NB>(8 * J + 4 + t, 8 * j + g)]);
          }
        }
#pragma unroll
        for (int j = 0; j < NB; j++) *reinterpret_cast<double2*>(Ys + ysi<NB>(8 * K + g, 8 * j + 2 * t)) = x[j];
        __syncwarp();
      }
      if (lane < T) {
        const ST* tb = Ts + 64 * warp_tri_block(K, K, kw8);
        double xv[8];
#pragma unroll
        for (int i = 0; i < 8; i++) xv[i] = Ys[ysi<NB>(8 * K + i, lane)];
#pragma unroll
        for (int k = 0; k < 8; k++) {
          xv[k] *= Rv[8 * K + k];
#pragma unroll
          for (int i = k + 1; i < 8; i++) xv[i] = fma(-(double)tb[32 * (k >> 2) + 4 * i + (k & 3)], xv[k], xv[i]);
        }
#pragma unroll
        for (int i = 0; i < 8; i++) Ys[ysi<NB>(8 * K + i, lane)] = xv[i];
      }
      __syncwarp();
    }
    // Ts is free: gather the next step's triangle while this step's R rows are updated
    if (more) {
      const int k8 = (ws_n.kw + 7) >> 3;
      warp_tri_gather(Lv, qt, k8 * (k8 + 1) / 2, Ts, lane);
    }
    cp_async_commit();
    // the solved rows are final: into the group strip
    for (int r = vr0; r < kw; r += RPI)
      st2(xp + (int64_t)r * G + vc2, *reinterpret_cast<const double2*>(Ys + ysi<NB>(r, vc2)));
    if (KS <= 4) warp_r_run<NB, 4, 4, ST>(Lv, gr, srw, Xs, G, Ys, nRB, KS, lane, qr, rr);
    else warp_r_run<NB, 8, 2, ST>(Lv, gr, srw, Xs, G, Ys, nRB, KS, lane, qr, rr);
    __syncwarp();  // this step's strip writes are visible to every lane of the next step
  }
  cp_async_wait<0>();
}

// ------------------------------------------------------------------------------------------------
// SYRK over G-column groups: F'[I,J] = sum_seg X_I[seg]^T X_J[seg] (lower part of F' only)
// ------------------------------------------------------------------------------------------------
#ifndef SC_SYRK_KC
#define SC_SYRK_KC 32
#endif
constexpr int kKC = SC_SYRK_KC;  // k rows staged per chunk

#ifndef SC_SYRK_KSPLIT
#define SC_SYRK_KSPLIT 0  // 1: k-split G = 32 SYRK (measured 2x slower on cfg2: short k ranges, reduction cost)
#endif
template <int G>
struct SyrkCfg {              // (G/8)^2 output blocks of 8x8 over 8 warps
  // G = 32 (2D): every warp holds all 4 x 4 output blocks and takes every 8th k step of a chunk
  // (16 DMMAs per 8 fragment loads instead of 2 per 3), partial tiles summed over the warps in a
  // fixed tree order at the end
  static constexpr bool KSPLIT = (G == 32) && SC_SYRK_KSPLIT;
  static constexpr int NB = G / 8;
  static constexpr int WN = KSPLIT ? NB : (G == 64) ? 4 : (G == 32 ? 2 : 1);
  static constexpr int WM = KSPLIT ? NB : (G == 64) ? 2 : 1;
  static constexpr int NWC = NB / WN;
  static constexpr int ACTIVE = KSPLIT ? 8 : (NB / WM) * NWC;   // warps with work (4 for G = 16)
};

// smem row stride (elements) of a staged X chunk: conflict-free fragment loads for 8- and 4-byte
// elements
template <int G, typename ST>
__host__ __device__ constexpr int syrk_ld() {
  return G + (sizeof(ST) == 8 ? 4 : 8);
}
template <int G, typename ST = double>
__host__ __device__ constexpr size_t syrk_smem_bytes() {
  // 2 stages x (X_I chunk, X_J chunk); the k-split G = 32 kernel reuses it for its warp reduction
  // (4 partial 32 x 32 tiles of doubles)
  return (G == 32 && SC_SYRK_KSPLIT && sizeof(ST) * 4 * kKC * syrk_ld<G, ST>() < 4 * 16 * 64 * sizeof(double))
             ? 4 * 16 * 64 * sizeof(double)
             : sizeof(ST) * 4 * kKC * syrk_ld<G, ST>();
}

template <int G, typename ST>
__global__ void __launch_bounds__(kThreads) syrk_pair_kernel(DevPlan P, int t0) {
  constexpr int kLdG = syrk_ld<G, ST>(), kGroup = G;
  extern __shared__ __align__(16) unsigned char syrk_smem[];
  ST* Sbuf = reinterpret_cast<ST*>(syrk_smem);
  constexpr int WM = SyrkCfg<G>::WM, WN = SyrkCfg<G>::WN, NWC = SyrkCfg<G>::NWC;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool active = warp < SyrkCfg<G>::ACTIVE;
  const int g = lane >> 2, t4 = lane & 3;
  const I2 task = P.syrk_tasks[t0 + blockIdx.x];
  const int sub = task.x;
  const Pair pr = P.pairs[task.y];
  const Group gI = P.groups[pr.I], gJ = P.groups[pr.J];
  const ST* __restrict__ XI = static_cast<const ST*>(P.X) + P.sub_X_base[sub] + gI.x_off;
  const ST* __restrict__ XJ = static_cast<const ST*>(P.X) + P.sub_X_base[sub] + gJ.x_off;
  constexpr bool KSPLIT = SyrkCfg<G>::KSPLIT;
  const int br0 = KSPLIT ? 0 : (warp / NWC) * WM, bc0 = KSPLIT ? 0 : (warp % NWC) * WN;
  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  // k chunks of kKC rows over the segments, two-stage cp.async pipeline (load chunk i+1 while
  // the tensor cores work on chunk i)
  int csg = pr.seg_begin, ck0 = 0;  // cursor of the next chunk to load
  auto load = [&](int stage) -> int {
    int kn = 0;
    if (csg < pr.seg_end) {
      const Seg s = P.segs[csg];
      kn = min(kKC, s.len - ck0);
      ST* As = Sbuf + (2 * stage) * kKC * kLdG;
      ST* Bs = As + kKC * kLdG;
      // thread -> (row r0 + u * RSTEP, 16-byte column vector j): fixed per thread, only the row
      // bases move
      constexpr int VEC = 16 / sizeof(ST), CP = kGroup / VEC, RSTEP = kThreads / CP;
      const int r0 = tid / CP, j = VEC * (tid % CP);
      const ST* srcI = XI + (int64_t)(s.offI + ck0) * kGroup + j;
      const ST* srcJ = XJ + (int64_t)(s.offJ + ck0) * kGroup + j;
#pragma unroll
      for (int r = r0; r < kKC; r += RSTEP) {
        const int ok = r < kn;
        const int rr = ok ? r : 0;
        cp_async16(As + r * kLdG + j, srcI + rr * kGroup, ok ? 16 : 0);
        cp_async16(Bs + r * kLdG + j, srcJ + rr * kGroup, ok ? 16 : 0);
      }
      ck0 += kKC;
      if (ck0 >= s.len) {
        csg++;
        ck0 = 0;
      }
    }
    cp_async_commit();
    return kn;
  };
  int kn_next = load(0);
  for (int it = 0; kn_next > 0; it++) {
    const int cur = it & 1, kn = kn_next;
    kn_next = load(cur ^ 1);
    cp_async_wait<1>();
    __syncthreads();
    const ST* As = Sbuf + (2 * cur) * kKC * kLdG;
    const ST* Bs = As + kKC * kLdG;
    const int kn4 = (kn + 3) & ~3;
    if (active) {
      auto kstep = [&](int k) {
        double a[WM], b[WN];
#pragma unroll
        for (int i = 0; i < WM; i++) a[i] = (double)As[(k + t4) * kLdG + (br0 + i) * 8 + g];
#pragma unroll
        for (int j = 0; j < WN; j++) b[j] = (double)Bs[(k + t4) * kLdG + (bc0 + j) * 8 + g];
#pragma unroll
        for (int i = 0; i < WM; i++)
#pragma unroll
          for (int j = 0; j < WN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
      };
      if constexpr (KSPLIT) {  // this warp's k steps of the chunk
        for (int k = 4 * warp; k < kn4; k += 4 * (kThreads / 32)) kstep(k);
      } else if (kn4 == kKC) {  // full chunk: fixed trip count, fully unrolled
#pragma unroll
        for (int k = 0; k < kKC; k += 4) kstep(k);
      } else {
        for (int k = 0; k < kn4; k += 4) kstep(k);
      }
    }
    __syncthreads();
  }
  cp_async_wait<0>();
  if constexpr (KSPLIT) {  // sum the warps' partial tiles: 8 -> 4 -> 2 -> 1, fixed order
    double* R = reinterpret_cast<double*>(syrk_smem);  // >= 4 x (WM x WN x 64) doubles (the stage buffers)
    static_assert(4 * WM * WN * 64 * sizeof(double) <= syrk_smem_bytes<G, ST>(), "reduction buffer");
#pragma unroll
    for (int half = 4; half >= 1; half >>= 1) {
      if (warp >= half && warp < 2 * half) {
#pragma unroll
        for (int i = 0; i < WM; i++)
#pragma unroll
          for (int j = 0; j < WN; j++) {
            R[(((warp - half) * WM + i) * WN + j) * 64 + 2 * lane] = acc[i][j][0];
            R[(((warp - half) * WM + i) * WN + j) * 64 + 2 * lane + 1] = acc[i][j][1];
          }
      }
      __syncthreads();
      if (warp < half) {
#pragma unroll
        for (int i = 0; i < WM; i++)
#pragma unroll
          for (int j = 0; j < WN; j++) {
            acc[i][j][0] += R[((warp * WM + i) * WN + j) * 64 + 2 * lane];
            acc[i][j][1] += R[((warp * WM + i) * WN + j) * 64 + 2 * lane + 1];
          }
      }
      __syncthreads();
    }
    if (warp != 0) return;
  }
  if (!active) return;
  ST* __restrict__ F = static_cast<ST*>(P.F) + P.sub_F_base[sub];
  const bool diag = (pr.I == pr.J);
#pragma unroll
  for (int i = 0; i < WM; i++) {
    const int r = (br0 + i) * 8 + g;  // row within group I
    if (r >= gI.width) continue;
#pragma unroll
    for (int j = 0; j < WN; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = (bc0 + j) * 8 + 2 * t4 + h;  // column within group J
        if (c >= gJ.width || (diag && r < c)) continue;
        F[f_index(gI.col0 + r, gJ.col0 + c)] = (ST)acc[i][j][h];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// SYRK with 16-column groups (small operators, e.g. 2D): one warp per 16 x 16 output tile (2 x 2 DMMA
// blocks), fragments loaded straight from the group strips (L2-resident while the subdomain's tiles
// run), k loop unrolled so several k steps' loads are in flight.  16-column groups restrict each
// tile's k range to the rows both 16-column strips hold: 1.35x the useful flops instead of 1.94x with
// 32-column groups (cfg2), and the strips themselves shrink to the tile-exact reach.
// ------------------------------------------------------------------------------------------------
#ifndef SC_SYRK16_BATCH
#define SC_SYRK16_BATCH 2  // k steps whose fragment loads are issued together
#endif
#ifndef SC_SYRK16_WPC
#define SC_SYRK16_WPC 1    // warps (output tiles) per CTA: 1 (a finished tile frees its slot at once)
#endif
template <typename ST>
__global__ void __launch_bounds__(32 * SC_SYRK16_WPC) syrk_warp16_kernel(DevPlan P, int t0, int ntask) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int ti = blockIdx.x * SC_SYRK16_WPC + wid;
  if (ti >= ntask) return;
  const I2 task = P.syrk_tasks[t0 + ti];
  const int sub = task.x;
  const Pair pr = P.pairs[task.y];
  const Group gI = P.groups[pr.I], gJ = P.groups[pr.J];
  const ST* __restrict__ XI = static_cast<const ST*>(P.X) + P.sub_X_base[sub] + gI.x_off;
  const ST* __restrict__ XJ = static_cast<const ST*>(P.X) + P.sub_X_base[sub] + gJ.x_off;
  const int g = lane >> 2, t = lane & 3;
  double acc[2][2][2];
#pragma unroll
  for (int i = 0; i < 2; i++)
#pragma unroll
    for (int j = 0; j < 2; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
  for (int s0 = pr.seg_begin; s0 < pr.seg_end; s0 += 32) {  // segment descriptors 32 at a time (one per lane)
    Seg my{};
    if (s0 + lane < pr.seg_end) my = P.segs[s0 + lane];
    const int ns = min(32, pr.seg_end - s0);
    for (int sj = 0; sj < ns; sj++) {
    const int offI = __shfl_sync(0xffffffffu, my.offI, sj), offJ = __shfl_sync(0xffffffffu, my.offJ, sj);
    const int len = __shfl_sync(0xffffffffu, my.len, sj);
    const ST* ai = XI + (int64_t)(offI + t) * 16 + g;  // A[i][k] = X_I[k][i], lane (g, t): row k = t
    const ST* bj = XJ + (int64_t)(offJ + t) * 16 + g;  // B[k][j] = X_J[k][j]
    // 4 k steps (16 rows) per batch: all 16 fragment loads issued before the batch's 16 DMMAs (the
    // compiler otherwise reuses the fragment registers and serialises one load latency per k step)
    for (int k0 = 0; k0 < len; k0 += 4 * SC_SYRK16_BATCH) {
      double a0[SC_SYRK16_BATCH], a1[SC_SYRK16_BATCH], b0[SC_SYRK16_BATCH], b1[SC_SYRK16_BATCH];
#pragma unroll
      for (int u = 0; u < SC_SYRK16_BATCH; u++) {
        const int k = k0 + 4 * u;
        const bool ok = k + t < len;
        const int64_t o = (int64_t)k * 16;
        a0[u] = ok ? (double)ai[o] : 0.0;
        a1[u] = ok ? (double)ai[o + 8] : 0.0;
        b0[u] = ok ? (double)bj[o] : 0.0;
        b1[u] = ok ? (double)bj[o + 8] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < SC_SYRK16_BATCH; u++) {
        dmma(acc[0][0][0], acc[0][0][1], a0[u], b0[u]);
        dmma(acc[0][1][0], acc[0][1][1], a0[u], b1[u]);
        dmma(acc[1][0][0], acc[1][0][1], a1[u], b0[u]);
        dmma(acc[1][1][0], acc[1][1][1], a1[u], b1[u]);
      }
    }
    }
  }
  ST* __restrict__ F = static_cast<ST*>(P.F) + P.sub_F_base[sub];
  const bool diag = pr.I == pr.J;
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const int r = 8 * i + g;
    if (r >= gI.width) continue;
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = 8 * j + 2 * t + h;
        if (c >= gJ.width || (diag && r < c)) continue;
        F[f_index(gI.col0 + r, gJ.col0 + c)] = (ST)acc[i][j][h];
      }
  }
}

// ------------------------------------------------------------------------------------------------
// Apply: y_i = F'_i x_i (x_i(a) = lambda[slm_i(a)]) from the lower triangle; deterministic sum.
// ------------------------------------------------------------------------------------------------
// One 64 x 64 tile (rb >= cb) of the lower F' per CTA, read once from HBM: u = F'_tile x_cols
// (row partial sums) and v = F'_tile^T x_rows (column partial sums; strictly lower part on the
// diagonal tiles, F' above its diagonal is never written and stays 0).  y = sum of the partials of
// a row's tiles, in a fixed order (deterministic, no atomics).
__device__ __forceinline__ int64_t apply_tile_index(int rb, int cb) { return (int64_t)rb * (rb + 1) / 2 + cb; }

// Warp w holds columns 8w..8w+7 of the tile, lane l rows l and l + 32, straight from HBM into
// registers (each load instruction reads 32 consecutive doubles of one column): column sums by warp
// shuffles, row sums over the 8 warps through a 4 KB shared reduction.
#ifndef SC_APPLY_TPC
#define SC_APPLY_TPC 4
#endif
constexpr int kApplyTPC = SC_APPLY_TPC;  // tiles per CTA

// ------------------------------------------------------------------------------------------------
// Input-split SYRK ("Splitting of the input matrix"; SURVEY f3 ablation): the k
// loop of F = X^T X is cut into block rows -- here the plan's common-row segments of each group pair
// -- and each block row's small SYRK touches only the output block of the columns that are non-zero
// in it; the partial results are summed into F' (zeroed first) with FP64 atomics, so the summation
// order (and the last bits of F) varies from run to run.  The default output-split kernels above
// write every F' entry once.
// ------------------------------------------------------------------------------------------------
template <typename ST>
__global__ void __launch_bounds__(256) syrk_input_split_kernel(DevPlan P, const SplitTask* __restrict__ tasks,
                                                               int64_t t0, int64_t ntask) {
  const int lane = threadIdx.x & 31;
  const int64_t ti = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5);
  if (ti >= ntask) return;
  const SplitTask tk = tasks[t0 + ti];
  const Pair pr = P.pairs[tk.pair];
  const Seg sg = P.segs[tk.seg];
  const Group gI = P.groups[pr.I], gJ = P.groups[pr.J];
  const int G = P.G, ib = tk.ij >> 2, jb = tk.ij & 3;
  const ST* __restrict__ XI = static_cast<const ST*>(P.X) + P.sub_X_base[tk.sub] + gI.x_off + 16 * ib;
  const ST* __restrict__ XJ = static_cast<const ST*>(P.X) + P.sub_X_base[tk.sub] + gJ.x_off + 16 * jb;
  const int g = lane >> 2, t = lane & 3;
  const ST* ai = XI + (int64_t)(sg.offI + t) * G + g;
  const ST* bj = XJ + (int64_t)(sg.offJ + t) * G + g;
  double acc[2][2][2] = {};
  for (int k = 0; k < sg.len; k += 4) {
    const bool ok = k + t < sg.len;
    const int64_t o = (int64_t)k * G;
    const double a0 = ok ? (double)ai[o] : 0.0, a1 = ok ? (double)ai[o + 8] : 0.0;
    const double b0 = ok ? (double)bj[o] : 0.0, b1 = ok ? (double)bj[o + 8] : 0.0;
    dmma(acc[0][0][0], acc[0][0][1], a0, b0);
    dmma(acc[0][1][0], acc[0][1][1], a0, b1);
    dmma(acc[1][0][0], acc[1][0][1], a1, b0);
    dmma(acc[1][1][0], acc[1][1][1], a1, b1);
  }
  ST* __restrict__ F = static_cast<ST*>(P.F) + P.sub_F_base[tk.sub];
  const bool diag = pr.I == pr.J;
#pragma unroll
  for (int i = 0; i < 2; i++) {
    const int r = 16 * ib + 8 * i + g;
    if (r >= gI.width) continue;
#pragma unroll
    for (int j = 0; j < 2; j++)
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = 16 * jb + 8 * j + 2 * t + h;
        if (c >= gJ.width || (diag && r < c)) continue;
        atomicAdd(F + f_index(gI.col0 + r, gJ.col0 + c), (ST)acc[i][j][h]);
      }
  }
}

template <typename ST>
__global__ void __launch_bounds__(kThreads) apply_tile_kernel(DevPlan P, const double* __restrict__ lambda, int ntask) {
  constexpr int AT = kApplyTile;
  static_assert(AT == 64 && kThreads == 256, "apply tile mapping");
  __shared__ double red[kThreads / 32][AT];
  for (int it = 0; it < kApplyTPC; it++) {
  const int ti = blockIdx.x * kApplyTPC + it;
  if (ti >= ntask) return;
  if (it > 0) __syncthreads();  // red reused
  const ApplyTask task = P.apply_tasks[ti];
  const int sub = task.sub, rb = task.rb, cb = task.cb;
  const int m = P.sub_m[sub];
  const int r0 = rb * AT, c0 = cb * AT;
  const int nr = min(AT, m - r0), nc = min(AT, m - c0);
  const ST* __restrict__ F = static_cast<const ST*>(P.F) + P.sub_F_base[sub];
  const int64_t* __restrict__ slm = P.slm + P.sub_slm_off[sub];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const bool diag = (rb == cb);
  const int rA = lane, rB = lane + 32;
  const double xA = (rA < nr) ? __ldg(lambda + slm[r0 + rA]) : 0.0;
  const double xB = (rB < nr) ? __ldg(lambda + slm[r0 + rB]) : 0.0;
  double fa[8], fb[8], xc[8];
  const ST* __restrict__ Ft = F + apply_tile_index(rb, cb) * AT * AT;  // packed lower tile, ld 64
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int c = warp * 8 + k;
    const ST* col = Ft + (int64_t)c * AT;
    const bool cv = c < nc;
    fa[k] = (cv && rA < nr) ? (double)__ldg(col + rA) : 0.0;
    fb[k] = (cv && rB < nr) ? (double)__ldg(col + rB) : 0.0;
    xc[k] = cv ? __ldg(lambda + slm[c0 + c]) : 0.0;
  }
  double* part = P.part + P.sub_part_off[sub] + apply_tile_index(rb, cb) * 2 * AT;
  double uA = 0.0, uB = 0.0;
#pragma unroll
  for (int k = 0; k < 8; k++) {
    const int c = warp * 8 + k;
    uA = fma(fa[k], xc[k], uA);
    uB = fma(fb[k], xc[k], uB);
    // column sum v_c = sum_r F[r][c] x_r (strictly lower part on a diagonal tile)
    double v = ((diag && rA <= c) ? 0.0 : fa[k] * xA) + ((diag && rB <= c) ? 0.0 : fb[k] * xB);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) part[AT + c] = v;
  }
  red[warp][rA] = uA;
  red[warp][rB] = uB;
  __syncthreads();
  if (tid < AT) {
    double u = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; w++) u += red[w][tid];
    part[tid] = u;
  }
  }
}

__global__ void __launch_bounds__(kThreads) apply_scatter_kernel(DevPlan P, double* __restrict__ q, int64_t nl) {
  constexpr int AT = kApplyTile;
  const int64_t gidx = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (gidx >= nl) return;
  double s = 0.0;
  for (int64_t p = P.qg_ptr[gidx]; p < P.qg_ptr[gidx + 1]; p++) {
    const int64_t sa = P.qg_sub_a[p];
    const int sub = (int)(sa >> 32), a = (int)(sa & 0xffffffff);
    const int nab = (P.sub_m[sub] + AT - 1) / AT;
    const double* part = P.part + P.sub_part_off[sub];
    const int b = a / AT, r = a - b * AT;
    for (int cb = 0; cb <= b; cb++) s += part[apply_tile_index(b, cb) * 2 * AT + r];           // row sums
    for (int rb = b; rb < nab; rb++) s += part[apply_tile_index(rb, b) * 2 * AT + AT + r];    // column sums
  }
  q[gidx] = s;
}


// ------------------------------------------------------------------------------------------------
// Implicit apply (row f2; eq. dualop_apply_impl): q = sum_i B~_i K_i^{-1} B~_i^T lambda_i
// without F, by one forward and one backward substitution with the prepared factor panels (the
// panel buffers of the last sc_prepare_factor / sc_assemble_batch).  One CTA per subdomain; its
// work vector (n doubles, permuted order) in shared memory when it fits, else in global memory.
//   forward, panels ascending:  y_p = inv(L_pp) x_p;  x[R_p] -= L[R_p,p] y_p   (W mode: W_p x_p)
//   backward, descending:       z_p = inv(L_pp)^T (y_p - L[R_p,p]^T z[R_p])   (W mode:
//                               z_p = inv(L_pp)^T y_p - W_p^T z[R_p])
// ------------------------------------------------------------------------------------------------
// sc_get_F_device: F(sigma(a), sigma(b)) = F'(max(a,b), min(a,b)) for one subdomain, full symmetric,
// original multiplier order, column-major with leading dimension ld
template <typename ST>
__global__ void __launch_bounds__(256) export_F_kernel(DevPlan P, int sub, double* __restrict__ out, int64_t ld) {
  const int m = P.sub_m[sub];
  const int r = blockIdx.y * 16 + (threadIdx.x >> 4), c = blockIdx.x * 16 + (threadIdx.x & 15);
  if (r >= m || c > r) return;
  const ST* F = static_cast<const ST*>(P.F) + P.sub_F_base[sub];
  const int32_t* sg = P.ssig + P.sub_slm_off[sub];
  const double v = (double)F[f_index(r, c)];
  const int64_t sr = sg[r], sc = sg[c];
  out[sc * ld + sr] = v;
  out[sr * ld + sc] = v;
}

__global__ void __launch_bounds__(kThreads) implicit_scatter_kernel(DevPlan P, double* __restrict__ q, int64_t nl) {
  const int64_t gidx = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (gidx >= nl) return;
  double s = 0.0;
  for (int64_t p = P.qg_ptr[gidx]; p < P.qg_ptr[gidx + 1]; p++) {
    const int64_t sa = P.qg_sub_a[p];
    s += P.upart[P.sub_slm_off[(int)(sa >> 32)] + (sa & 0xffffffff)];
  }
  q[gidx] = s;
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
namespace {

using TrsmFn = void (*)(DevPlan, TrsmLaunch);
int trsm_threads(int T, int minb = 1) {
  switch (T) {
    case 8: return minb == 2 ? TileCfg<8, 2>::CT + 32 : TileCfg<8>::CT + 32;
    case 16: return minb == 2 ? TileCfg<16, 2>::CT + 32 : TileCfg<16>::CT + 32;
    case 32: return TileCfg<32>::CT + 32;
    default: return TileCfg<64>::CT + 32;
  }
}
template <bool YM>
TrsmFn trsm_kernel_ptr_m(int T, bool gs) {
  switch (T) {
    case 8: return gs ? trsm_smem_kernel<8, true, YM> : trsm_smem_kernel<8, false, YM>;
    case 16: return gs ? trsm_smem_kernel<16, true, YM> : trsm_smem_kernel<16, false, YM>;
    case 32: return gs ? trsm_smem_kernel<32, true, YM> : trsm_smem_kernel<32, false, YM>;
    default: return gs ? trsm_smem_kernel<64, true, YM> : trsm_smem_kernel<64, false, YM>;
  }
}
TrsmFn trsm_kernel_ptr(int T, bool gs, bool wmode) {
  return wmode ? trsm_kernel_ptr_m<false>(T, gs) : trsm_kernel_ptr_m<true>(T, gs);
}
// global strips at two CTAs per SM (T = 16, plan option gs2)
TrsmFn trsm_kernel_ptr_gs2(bool wmode, int ctas = 2) {
  if (ctas == 3) return wmode ? trsm_smem_kernel<16, true, false, 3> : trsm_smem_kernel<16, true, true, 3>;
  return wmode ? trsm_smem_kernel<16, true, false, 2> : trsm_smem_kernel<16, true, true, 2>;
}

// small-strip class (shared strips, T <= 16 only), two CTAs per SM
TrsmFn trsm_kernel_ptr2(int T, bool wmode) {
  switch (T) {
    case 8: return wmode ? trsm_smem_kernel<8, false, false, 2> : trsm_smem_kernel<8, false, true, 2>;
    default: return wmode ? trsm_smem_kernel<16, false, false, 2> : trsm_smem_kernel<16, false, true, 2>;
  }
}

template <typename V>
sc_status upload(Plan& P, const std::vector<V>& v, const V** dst, std::string& err) {
  void* d = nullptr;
  size_t bytes = std::max<size_t>(v.size() * sizeof(V), 16);
  CUDA_TRY(cudaMalloc(&d, bytes));
  P.allocations.push_back(d);
  if (!v.empty()) CUDA_TRY(cudaMemcpy(d, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
  *dst = static_cast<const V*>(d);
  return SC_OK;
}

template <typename V>
sc_status alloc_zero(Plan& P, int64_t count, V** dst, std::string& err) {
  void* d = nullptr;
  size_t bytes = std::max<size_t>((size_t)count * sizeof(V), 16);
  CUDA_TRY(cudaMalloc(&d, bytes));
  P.allocations.push_back(d);
  CUDA_TRY(cudaMemset(d, 0, bytes));
  *dst = static_cast<V*>(d);
  return SC_OK;
}

#define TRY(x)                   \
  do {                           \
    sc_status s_ = (x);          \
    if (s_ != SC_OK) return s_;  \
  } while (0)

}  // namespace

sc_status upload_plan(Plan& P, std::string& err) {
  CUDA_TRY(cudaSetDevice(P.opt.device));
  // shared-memory fit checks before any allocation
  if (P.ring_bytes <= 0 && !P.warp_trsm) {
    err = "X strip of " + std::to_string(P.max_strip_rows) + " rows x " + std::to_string(P.T) +
          " columns leaves no room for the L-block ring in shared memory; use smaller tile_cols";
    return SC_ERR_INVALID_ARG;
  }
  P.smem_trsm = P.warp_trsm ? 0 : trsm_smem_layout(P.T, P.ring_bytes, P.max_strip_rows, P.gstrip, !P.wmode).total;
  if (P.ntrsm_small > 0) P.smem_trsm_small = trsm_smem_layout(P.T, P.ring_small, P.strip_small, false, !P.wmode).total;
  {
    int dev_smem = 0;
    CUDA_TRY(cudaDeviceGetAttribute(&dev_smem, cudaDevAttrMaxSharedMemoryPerBlockOptin, P.opt.device));
    if (P.smem_trsm > (size_t)dev_smem) {
      err = "X strip of " + std::to_string(P.max_strip_rows) + " rows x " + std::to_string(P.T) +
            " columns does not fit in shared memory (" + std::to_string(P.smem_trsm) + " > " + std::to_string(dev_smem) +
            " bytes); use smaller tile_cols";
      return SC_ERR_INVALID_ARG;
    }
  }
  DevPlan& D = P.dev;
  std::memset(&D, 0, sizeof(D));
  // concatenate class data
  std::vector<Panel> panels;
  std::vector<int32_t> Rrows, dest;
  std::vector<int64_t> csc_off;
  std::vector<Tile> tiles;
  std::vector<Step> steps;
  std::vector<uint16_t> srows;
  std::vector<Group> groups;
  std::vector<Reach> greach;
  std::vector<BInit> binit;
  std::vector<Pair> pairs;
  std::vector<Seg> segs;
  std::vector<int32_t> gidx;
  for (auto& C : P.classes) {
    csc_off.push_back((int64_t)dest.size());
    dest.insert(dest.end(), C.dest.begin(), C.dest.end());
    const size_t p0 = panels.size();
    panels.insert(panels.end(), C.panels.begin(), C.panels.end());
    for (size_t q = p0; q < panels.size(); q++) panels[q].gx_off += (int64_t)gidx.size();
    gidx.insert(gidx.end(), C.gidx.begin(), C.gidx.end());
    Rrows.insert(Rrows.end(), C.Rrows.begin(), C.Rrows.end());
    tiles.insert(tiles.end(), C.tiles.begin(), C.tiles.end());
    steps.insert(steps.end(), C.steps.begin(), C.steps.end());
    srows.insert(srows.end(), C.srows.begin(), C.srows.end());
    groups.insert(groups.end(), C.groups.begin(), C.groups.end());
    greach.insert(greach.end(), C.greach.begin(), C.greach.end());
    binit.insert(binit.end(), C.binit.begin(), C.binit.end());
    pairs.insert(pairs.end(), C.pairs.begin(), C.pairs.end());
    segs.insert(segs.end(), C.segs.begin(), C.segs.end());
  }
  TRY(upload(P, panels, &D.panels, err));
  TRY(upload(P, gidx, &D.gidx, err));
  TRY(upload(P, Rrows, &D.Rrows, err));
  TRY(upload(P, dest, &D.dest, err));
  TRY(upload(P, csc_off, &D.cls_csc_off, err));
  TRY(upload(P, tiles, &D.tiles, err));
  TRY(upload(P, steps, &D.steps, err));
  if (P.warp_trsm) {
    std::vector<WStep> ws(steps.size());
    for (size_t q = 0; q < steps.size(); q++) {
      const Panel& pn = panels[(size_t)steps[q].panel];
      ws[q] = WStep{steps[q].strip_row, pn.a, pn.kw, pn.nR, pn.gx_off, steps[q].srow_off};
    }
    TRY(upload(P, ws, &D.wsteps, err));
  }
  TRY(upload(P, srows, &D.srows, err));
  TRY(upload(P, groups, &D.groups, err));
  TRY(upload(P, greach, &D.greach, err));
  TRY(upload(P, binit, &D.binit, err));
  TRY(upload(P, pairs, &D.pairs, err));
  TRY(upload(P, segs, &D.segs, err));
  TRY(upload(P, P.sub_cls, &D.sub_cls, err));
  {
    std::vector<int32_t> cp0(P.cls_panel_begin);
    cp0.push_back((int32_t)panels.size());
    TRY(upload(P, cp0, &D.cls_panel0, err));
    std::vector<int64_t> ib0;
    std::vector<int32_t> ibp, ibr;
    std::vector<double> ibv;
    for (auto& C : P.classes) {
      ib0.push_back((int64_t)ibp.size());
      for (int32_t v : C.ib_ptr) ibp.push_back(v + (int32_t)ibr.size());
      ibr.insert(ibr.end(), C.ib_row.begin(), C.ib_row.end());
      ibv.insert(ibv.end(), C.ib_val.begin(), C.ib_val.end());
    }
    TRY(upload(P, ib0, &D.cls_ib0, err));
    TRY(upload(P, ibp, &D.ib_ptr, err));
    TRY(upload(P, ibr, &D.ib_row, err));
    TRY(upload(P, ibv, &D.ib_val, err));
    TRY(alloc_zero(P, (int64_t)P.slm.size(), &D.upart, err));
  }
  TRY(upload(P, P.sub_X_base, &D.sub_X_base, err));
  TRY(upload(P, P.sub_F_base, &D.sub_F_base, err));
  TRY(upload(P, P.sub_PB_base, &D.sub_PB_base, err));
  TRY(upload(P, P.sub_m, &D.sub_m, err));
  TRY(upload(P, P.prep_tasks, &D.prep_tasks, err));
  TRY(upload(P, P.prep_small_tasks, &D.prep_small_tasks, err));
  TRY(upload(P, P.trsm_tasks, &D.trsm_tasks, err));
  TRY(upload(P, P.syrk_tasks, &D.syrk_tasks, err));
  if (P.syrk_input) {  // (sub, pair, segment, 16 x 16 sub-tile) tasks of the input-split SYRK
    std::vector<SplitTask> st;
    P.split_sub_begin.assign((size_t)P.nsub + 1, 0);
    const int nb = P.G / 16;
    size_t q = 0;
    for (int32_t i = 0; i < P.nsub; i++) {
      P.split_sub_begin[(size_t)i] = (int64_t)st.size();
      for (; q < P.syrk_tasks.size() && P.syrk_tasks[q].x == i; q++) {
        const Pair& pr = pairs[(size_t)P.syrk_tasks[q].y];
        for (int32_t sg = pr.seg_begin; sg < pr.seg_end; sg++)
          for (int ib = 0; ib < nb; ib++)
            for (int jb = 0; jb < nb; jb++)
              if (!(pr.I == pr.J && jb > ib)) st.push_back(SplitTask{i, P.syrk_tasks[q].y, sg, ib * 4 + jb});
      }
    }
    P.split_sub_begin[(size_t)P.nsub] = (int64_t)st.size();
    TRY(upload(P, st, &P.d_split, err));
  }
  TRY(upload(P, P.apply_tasks, &D.apply_tasks, err));
  TRY(upload(P, P.sub_slm_off, &D.sub_slm_off, err));
  TRY(upload(P, P.slm, &D.slm, err));
  TRY(upload(P, P.ssig, &D.ssig, err));
  TRY(upload(P, P.sub_part_off, &D.sub_part_off, err));
  TRY(upload(P, P.qg_ptr, &D.qg_ptr, err));
  TRY(upload(P, P.qg_sub_a, &D.qg_sub_a, err));
  {  // X strips and F' lower tiles in the plan's storage precision
    char* xb = nullptr;
    char* fb = nullptr;
    TRY(alloc_zero(P, P.X_doubles * P.esz, &xb, err));
    TRY(alloc_zero(P, P.F_doubles * P.esz, &fb, err));
    D.X = xb;
    D.F = fb;
  }
  if (!P.warp_trsm) TRY(alloc_zero(P, P.PB_doubles, &D.PB, err));  // warp TRSM: only for the implicit apply, lazily
  TRY(alloc_zero(P, P.part_doubles, &D.part, err));
  TRY(alloc_zero(P, 1 + (int64_t)P.nsub, &D.err, err));
  double** dl = nullptr;
  TRY(alloc_zero(P, std::max(P.nsub, 1), &dl, err));
  P.d_Lptr = dl;
  D.Lptr = reinterpret_cast<const void* const*>(dl);
  void* hp = nullptr;
  CUDA_TRY(cudaMallocHost(&hp, sizeof(double*) * (size_t)std::max(P.nsub, 1)));
  P.h_Lptr_pinned = static_cast<const void**>(hp);
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  P.lptr_event = ev;
  D.nsub = P.nsub;
  D.max_n = P.max_n;
  D.T = P.T;
  D.G = P.G;
  D.wmode = P.wmode ? 1 : 0;
  D.fp32 = P.esz == 4 ? 1 : 0;
  if (P.ntrsm_small > 0) {  // small-strip tile class: its own launch on a side stream
    CUDA_TRY(cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&P.side_stream), cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(&P.ev_fork), cudaEventDisableTiming));
    CUDA_TRY(cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(&P.ev_join), cudaEventDisableTiming));
  }
  // every kernel: the largest shared-memory carveout (the default left prep_small<16> at 3 CTAs/SM)
  auto smem_attr = [&](const void* fn, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared);
    return e;
  };
  CUDA_TRY(smem_attr((const void*)prep_panel_kernel<true>, kPrepSmem));
  CUDA_TRY(smem_attr((const void*)prep_panel_kernel<false>, kPrepSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<8, true>, SmallCfg<8>::kSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<8, false>, SmallCfg<8>::kSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<16, true>, SmallCfg<16>::kSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<16, false>, SmallCfg<16>::kSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<32, true>, SmallCfg<32>::kSmem));
  CUDA_TRY(smem_attr((const void*)prep_small_kernel<32, false>, SmallCfg<32>::kSmem));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<16, double>, syrk_smem_bytes<16, double>()));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<32, double>, syrk_smem_bytes<32, double>()));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<64, double>, syrk_smem_bytes<64, double>()));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<16, float>, syrk_smem_bytes<16, float>()));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<32, float>, syrk_smem_bytes<32, float>()));
  CUDA_TRY(smem_attr((const void*)syrk_pair_kernel<64, float>, syrk_smem_bytes<64, float>()));
  for (const void* fn : {(const void*)trsm_warp_kernel<1, double>, (const void*)trsm_warp_kernel<2, double>,
                         (const void*)trsm_warp_kernel<1, float>, (const void*)trsm_warp_kernel<2, float>})
    CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, (int)cudaSharedmemCarveoutMaxShared));
  if (!P.warp_trsm)
    CUDA_TRY(smem_attr((const void*)(P.gs2 ? trsm_kernel_ptr_gs2(P.wmode, P.gs2) : trsm_kernel_ptr(P.T, P.gstrip, P.wmode)),
                       P.smem_trsm));
  if (P.ntrsm_small > 0) CUDA_TRY(smem_attr((const void*)trsm_kernel_ptr2(P.T, P.wmode), P.smem_trsm_small));
  double total = (double)P.esz * (P.X_doubles + P.F_doubles) + 8.0 * ((P.warp_trsm ? 0 : P.PB_doubles) + P.part_doubles) +
                 4.0 * gidx.size();
  total += dest.size() * 4.0 + Rrows.size() * 4.0 + panels.size() * sizeof(Panel) + tiles.size() * sizeof(Tile) +
           steps.size() * sizeof(Step) + groups.size() * sizeof(Group) +
           greach.size() * sizeof(Reach) + binit.size() * sizeof(BInit) + pairs.size() * sizeof(Pair) +
           segs.size() * sizeof(Seg) + P.slm.size() * 8.0 + P.qg_sub_a.size() * 8.0 + P.qg_ptr.size() * 8.0;
  P.stats.device_bytes = total;
  P.on_device = true;
  return SC_OK;
}

// Releases everything the plan allocated on the device / pinned host, whether or not upload_plan
// completed (a failed upload must not orphan its allocations).
void free_plan_device(Plan& P) {
  if (P.opt.device < 0) return;
  cudaSetDevice(P.opt.device);
  cudaDeviceSynchronize();
  free_factor_device(P);
  for (void* p : P.allocations) cudaFree(p);
  P.allocations.clear();
  if (P.h_Lptr_pinned) cudaFreeHost((void*)P.h_Lptr_pinned);
  P.h_Lptr_pinned = nullptr;
  if (P.lptr_event) cudaEventDestroy((cudaEvent_t)P.lptr_event);
  P.lptr_event = nullptr;
  if (P.side_stream) cudaStreamDestroy(static_cast<cudaStream_t>(P.side_stream));
  if (P.ev_fork) cudaEventDestroy(static_cast<cudaEvent_t>(P.ev_fork));
  if (P.ev_join) cudaEventDestroy(static_cast<cudaEvent_t>(P.ev_join));
  P.side_stream = P.ev_fork = P.ev_join = nullptr;
  for (int i = 0; i < 2; i++)
    if (P.ov_stream[i]) cudaStreamDestroy(static_cast<cudaStream_t>(P.ov_stream[i]));
  P.ov_stream[0] = P.ov_stream[1] = nullptr;
  for (void* e : P.ev_ov) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  P.ev_ov.clear();
  if (P.copy_stream) cudaStreamDestroy(static_cast<cudaStream_t>(P.copy_stream));
  if (P.ev_start) cudaEventDestroy(static_cast<cudaEvent_t>(P.ev_start));
  for (void* e : P.ev_chunk) cudaEventDestroy(static_cast<cudaEvent_t>(e));
  P.ev_chunk.clear();
  P.copy_stream = P.ev_start = nullptr;
  if (P.d_Lstage) cudaFree(P.d_Lstage);
  P.d_Lstage = nullptr;
  if (P.d_hsrc) cudaFree(P.d_hsrc);
  if (P.d_Lstage_off) cudaFree(P.d_Lstage_off);
  if (P.h_hsrc) cudaFreeHost((void*)P.h_hsrc);
  if (P.ev_hsrc) cudaEventDestroy(static_cast<cudaEvent_t>(P.ev_hsrc));
  P.d_hsrc = nullptr;
  P.d_Lstage_off = nullptr;
  P.h_hsrc = nullptr;
  P.ev_hsrc = nullptr;
  P.on_device = false;
}

template <bool WMODE>
static void launch_prep_small(int bkt, int t0, int t1, Plan& P, cudaStream_t stream) {
  const int nt = t1 - t0;
  if (bkt == 0) {
    using C8 = SmallCfg<8>;
    prep_small_kernel<8, WMODE><<<(nt + C8::WARPS - 1) / C8::WARPS, 32 * C8::WARPS, C8::kSmem, stream>>>(P.dev, t0, t1);
  } else if (bkt == 1) {
    using C16 = SmallCfg<16>;
    prep_small_kernel<16, WMODE><<<(nt + C16::WARPS - 1) / C16::WARPS, 32 * C16::WARPS, C16::kSmem, stream>>>(P.dev, t0, t1);
  } else {
    using C32 = SmallCfg<32>;
    prep_small_kernel<32, WMODE><<<(nt + C32::WARPS - 1) / C32::WARPS, 32 * C32::WARPS, C32::kSmem, stream>>>(P.dev, t0, t1);
  }
}

// first task of subdomain >= sub in a subdomain-major task list
static int task_lb(const std::vector<I2>& v, int lo, int hi, int32_t sub) {
  return (int)(std::lower_bound(v.begin() + lo, v.begin() + hi, sub, [](const I2& t, int32_t s) { return t.x < s; }) -
               v.begin());
}

static sc_status set_Lptr(Plan& P, const void* const* Lptr_host, cudaStream_t stream, std::string& err) {
  bool same = (int32_t)P.last_Lptr.size() == P.nsub;
  for (int32_t i = 0; same && i < P.nsub; i++) same = (P.last_Lptr[(size_t)i] == Lptr_host[i]);
  if (same) return SC_OK;
  for (int32_t i = 0; i < P.nsub; i++)
    if (!Lptr_host[i] && P.sub_nnz[(size_t)i] > 0) {
      err = "L_values[" + std::to_string(i) + "] is NULL";
      return SC_ERR_INVALID_ARG;
    }
  CUDA_TRY(cudaEventSynchronize((cudaEvent_t)P.lptr_event));  // previous upload consumed the buffer
  for (int32_t i = 0; i < P.nsub; i++) P.h_Lptr_pinned[i] = Lptr_host[i];
  CUDA_TRY(cudaMemcpyAsync(P.d_Lptr, P.h_Lptr_pinned, sizeof(double*) * (size_t)P.nsub, cudaMemcpyHostToDevice, stream));
  CUDA_TRY(cudaEventRecord((cudaEvent_t)P.lptr_event, stream));
  P.last_Lptr.assign(Lptr_host, Lptr_host + P.nsub);
  return SC_OK;
}

// prep kernels (factor panels) for the subdomains [s0, s1)
static sc_status launch_prep_range(Plan& P, int32_t s0, int32_t s1, cudaStream_t stream, std::string& err) {
  const bool all = s0 == 0 && s1 == P.nsub;
  {
    const int npr = (int)P.prep_tasks.size();
    const int a = all ? 0 : task_lb(P.prep_tasks, 0, npr, s0), b = all ? npr : task_lb(P.prep_tasks, 0, npr, s1);
    if (b > a) {
      if (P.wmode) prep_panel_kernel<true><<<b - a, kThreads, kPrepSmem, stream>>>(P.dev, a);
      else prep_panel_kernel<false><<<b - a, kThreads, kPrepSmem, stream>>>(P.dev, a);
      CUDA_TRY(cudaGetLastError());
    }
  }
  for (int bkt = 0; bkt < 3; bkt++) {  // small panels bucketed by padded width 8 / 16 / 32
    const int lo = P.small_begin[bkt], hi = P.small_begin[bkt + 1];
    const int t0 = all ? lo : task_lb(P.prep_small_tasks, lo, hi, s0);
    const int t1 = all ? hi : task_lb(P.prep_small_tasks, lo, hi, s1), nt = t1 - t0;
    if (nt <= 0) continue;
    if (P.wmode) {
      launch_prep_small<true>(bkt, t0, t1, P, stream);
    } else {
      launch_prep_small<false>(bkt, t0, t1, P, stream);
    }
    CUDA_TRY(cudaGetLastError());
  }
  return SC_OK;
}

// All phases (prep, TRSM, SYRK) for the subdomains [s0, s1) on `stream`; timing events only for the
// whole batch.
static sc_status launch_trsm_range(Plan& P, int32_t s0, int32_t s1, cudaStream_t stream, std::string& err) {
  const bool all = s0 == 0 && s1 == P.nsub;
  if (P.warp_trsm) {
    const int ntr = (int)P.trsm_tasks.size();
    const int a = all ? 0 : task_lb(P.trsm_tasks, 0, ntr, s0), b = all ? ntr : task_lb(P.trsm_tasks, 0, ntr, s1);
    if (b > a) {
      constexpr int W = SC_WARP_WPC, NT = 32 * SC_WARP_WPC;
      const int nb = (b - a + W - 1) / W;  // W warps (tiles) per CTA
      if (P.esz == 4) {
        if (P.T == 8) trsm_warp_kernel<1, float><<<nb, NT, 0, stream>>>(P.dev, a, b - a);
        else trsm_warp_kernel<2, float><<<nb, NT, 0, stream>>>(P.dev, a, b - a);
      } else {
        if (P.T == 8) trsm_warp_kernel<1, double><<<nb, NT, 0, stream>>>(P.dev, a, b - a);
        else trsm_warp_kernel<2, double><<<nb, NT, 0, stream>>>(P.dev, a, b - a);
      }
      CUDA_TRY(cudaGetLastError());
    }
    return SC_OK;
  }
  {
    // tiles with small strips (2 CTAs per SM) and the rest (1 CTA per SM): two launches, the large
    // ones on a side stream so both classes share the SMs and neither launch's tail idles them
    const int ntr = (int)P.trsm_tasks.size(), nsm = P.ntrsm_small;
    const TrsmFn fn = P.gs2 ? trsm_kernel_ptr_gs2(P.wmode, P.gs2) : trsm_kernel_ptr(P.T, P.gstrip, P.wmode),
                 fn2 = trsm_kernel_ptr2(P.T, P.wmode);
    const int thr = P.gs2 ? trsm_threads(16, 2) : trsm_threads(P.T);
    const int sa = all ? 0 : task_lb(P.trsm_tasks, 0, nsm, s0), sb = all ? nsm : task_lb(P.trsm_tasks, 0, nsm, s1);
    const int la = all ? nsm : task_lb(P.trsm_tasks, nsm, ntr, s0), lb = all ? ntr : task_lb(P.trsm_tasks, nsm, ntr, s1);
    const int ns = sb - sa, nl = lb - la;
    if (ns > 0 && nl > 0) {
      cudaStream_t side = static_cast<cudaStream_t>(P.side_stream);
      CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_fork), stream));
      CUDA_TRY(cudaStreamWaitEvent(side, static_cast<cudaEvent_t>(P.ev_fork), 0));
      fn<<<nl, thr, P.smem_trsm, side>>>(P.dev, TrsmLaunch{la, P.ring_bytes, P.max_strip_rows, 0});
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_join), side));
      fn2<<<ns, trsm_threads(P.T, 2), P.smem_trsm_small, stream>>>(P.dev, TrsmLaunch{sa, P.ring_small, P.strip_small, 0});
      CUDA_TRY(cudaGetLastError());
      CUDA_TRY(cudaStreamWaitEvent(stream, static_cast<cudaEvent_t>(P.ev_join), 0));
    } else if (ns > 0) {
      fn2<<<ns, trsm_threads(P.T, 2), P.smem_trsm_small, stream>>>(P.dev, TrsmLaunch{sa, P.ring_small, P.strip_small, 0});
    } else if (nl > 0) {
      fn<<<nl, thr, P.smem_trsm, stream>>>(P.dev, TrsmLaunch{la, P.ring_bytes, P.max_strip_rows, 0});
    }
    CUDA_TRY(cudaGetLastError());
  }
  return SC_OK;
}

static sc_status launch_syrk_range(Plan& P, int32_t s0, int32_t s1, cudaStream_t stream, std::string& err) {
  const bool all = s0 == 0 && s1 == P.nsub;
  if (P.syrk_input) {  // f3 ablation: zero F' of the range, then the input-split kernel's atomics
    const int64_t f0 = P.sub_F_base[(size_t)s0], f1 = s1 < P.nsub ? P.sub_F_base[(size_t)s1] : P.F_doubles;
    CUDA_TRY(cudaMemsetAsync(static_cast<char*>(P.dev.F) + (size_t)P.esz * f0, 0, (size_t)P.esz * (f1 - f0), stream));
    const int64_t a = P.split_sub_begin[(size_t)s0], n = P.split_sub_begin[(size_t)s1] - a;
    if (n > 0) {
      const unsigned nb = (unsigned)((n + 7) / 8);
      if (P.esz == 4) syrk_input_split_kernel<float><<<nb, 256, 0, stream>>>(P.dev, P.d_split, a, n);
      else syrk_input_split_kernel<double><<<nb, 256, 0, stream>>>(P.dev, P.d_split, a, n);
      CUDA_TRY(cudaGetLastError());
    }
    return SC_OK;
  }
  {
    const int nsy = (int)P.syrk_tasks.size();
    const int a = all ? 0 : task_lb(P.syrk_tasks, 0, nsy, s0), b = all ? nsy : task_lb(P.syrk_tasks, 0, nsy, s1);
    if (b > a && P.G == 16) {  // warp per 16 x 16 output tile
      const int nt = b - a;
      constexpr int W = SC_SYRK16_WPC;
      if (P.esz == 4) syrk_warp16_kernel<float><<<(nt + W - 1) / W, 32 * W, 0, stream>>>(P.dev, a, nt);
      else syrk_warp16_kernel<double><<<(nt + W - 1) / W, 32 * W, 0, stream>>>(P.dev, a, nt);
      CUDA_TRY(cudaGetLastError());
    } else if (b > a) {
      if (P.esz == 4) {
        switch (P.G) {
          case 16: syrk_pair_kernel<16, float><<<b - a, kThreads, syrk_smem_bytes<16, float>(), stream>>>(P.dev, a); break;
          case 32: syrk_pair_kernel<32, float><<<b - a, kThreads, syrk_smem_bytes<32, float>(), stream>>>(P.dev, a); break;
          default: syrk_pair_kernel<64, float><<<b - a, kThreads, syrk_smem_bytes<64, float>(), stream>>>(P.dev, a); break;
        }
      } else {
        switch (P.G) {
          case 16: syrk_pair_kernel<16, double><<<b - a, kThreads, syrk_smem_bytes<16, double>(), stream>>>(P.dev, a); break;
          case 32: syrk_pair_kernel<32, double><<<b - a, kThreads, syrk_smem_bytes<32, double>(), stream>>>(P.dev, a); break;
          default: syrk_pair_kernel<64, double><<<b - a, kThreads, syrk_smem_bytes<64, double>(), stream>>>(P.dev, a); break;
        }
      }
      CUDA_TRY(cudaGetLastError());
    }
  }
  return SC_OK;
}

// All phases (prep, TRSM, SYRK) for the subdomains [s0, s1) on `stream`; timing events only for the
// whole batch.
static sc_status launch_range(Plan& P, int32_t s0, int32_t s1, cudaStream_t stream, bool timing, std::string& err) {
  if (timing && P.tev[0]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[0], stream));
  sc_status st = P.warp_trsm ? SC_OK : launch_prep_range(P, s0, s1, stream, err);  // warp TRSM: no prep
  if (st != SC_OK) return st;
  if (timing && P.tev[1]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[1], stream));
  st = launch_trsm_range(P, s0, s1, stream, err);
  if (st != SC_OK) return st;
  if (timing && P.tev[2]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[2], stream));
  st = launch_syrk_range(P, s0, s1, stream, err);
  if (st != SC_OK) return st;
  if (timing && P.tev[3]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[3], stream));
  return SC_OK;
}

// Phase-overlapped batch (P.overlap chunks of subdomains): prep of chunk k+1 (on `stream`), TRSM of
// chunk k and SYRK of chunk k-1 (two plan-owned streams) run concurrently, ordered per chunk by events.
static sc_status launch_overlapped(Plan& P, cudaStream_t stream, std::string& err) {
  const int K = P.overlap;
  if (!P.ov_stream[0]) {
    for (int i = 0; i < 2; i++)
      CUDA_TRY(cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&P.ov_stream[i]), cudaStreamNonBlocking));
  }
  while ((int)P.ev_ov.size() < 2 * K + 2) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P.ev_ov.push_back(e);
  }
  cudaStream_t ts = static_cast<cudaStream_t>(P.ov_stream[0]), ss = static_cast<cudaStream_t>(P.ov_stream[1]);
  auto ev = [&](int i) { return static_cast<cudaEvent_t>(P.ev_ov[(size_t)i]); };
  if (P.tev[0]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[0], stream));
  CUDA_TRY(cudaEventRecord(ev(0), stream));
  CUDA_TRY(cudaStreamWaitEvent(ts, ev(0), 0));
  CUDA_TRY(cudaStreamWaitEvent(ss, ev(0), 0));
  for (int k = 0; k < K; k++) {
    const int32_t s0 = (int32_t)((int64_t)P.nsub * k / K), s1 = (int32_t)((int64_t)P.nsub * (k + 1) / K);
    sc_status st = P.warp_trsm ? SC_OK : launch_prep_range(P, s0, s1, stream, err);
    if (st != SC_OK) return st;
    CUDA_TRY(cudaEventRecord(ev(2 + 2 * k), stream));
    CUDA_TRY(cudaStreamWaitEvent(ts, ev(2 + 2 * k), 0));
    st = launch_trsm_range(P, s0, s1, ts, err);
    if (st != SC_OK) return st;
    CUDA_TRY(cudaEventRecord(ev(3 + 2 * k), ts));
    CUDA_TRY(cudaStreamWaitEvent(ss, ev(3 + 2 * k), 0));
    st = launch_syrk_range(P, s0, s1, ss, err);
    if (st != SC_OK) return st;
  }
  if (P.tev[1]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[1], stream));  // all prep issued/done on stream
  if (P.tev[2]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[2], ts));
  CUDA_TRY(cudaEventRecord(ev(1), ss));
  CUDA_TRY(cudaStreamWaitEvent(stream, ev(1), 0));
  if (P.tev[3]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[3], stream));
  return SC_OK;
}

sc_status launch_assemble(Plan& P, const void* const* Lptr_host, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  sc_status st = set_Lptr(P, Lptr_host, stream, err);
  if (st != SC_OK) return st;
  P.last_stream = stream_v;
  CUDA_TRY(cudaMemsetAsync(P.dev.err, 0, sizeof(unsigned long long) * (1 + (size_t)P.nsub), stream));
  if (P.overlap > 1 && P.nsub >= 2 * P.overlap) return launch_overlapped(P, stream, err);
  return launch_range(P, 0, P.nsub, stream, true, err);
}

// Host-resident L (row f1 "host-fed pipeline"): the batch is cut into chunks of
// subdomains; chunk k's pinned-host -> device copies run on a plan-owned copy stream while the
// kernels of chunk k-1 run on `stream` (one event per chunk), so the H2D transfer (PCIe-bound) hides
// the assembly.
// Plan-owned device staging of every subdomain's L values (host-fed paths): allocate it once, point
// the plan's L table at it, reset the sticky errors.  dptrs receives the per-subdomain staging pointers.
sc_status assemble_stage_begin(Plan& P, std::vector<void*>& dptrs, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  if (!P.d_Lstage) {
    P.Lstage_off.assign((size_t)P.nsub + 1, 0);
    for (int32_t i = 0; i < P.nsub; i++) P.Lstage_off[(size_t)i + 1] = P.Lstage_off[(size_t)i] + P.sub_nnz[(size_t)i];
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, std::max<size_t>((size_t)P.esz * (size_t)P.Lstage_off.back(), 16)));
    P.d_Lstage = d;
  }
  if (!P.copy_stream) {
    CUDA_TRY(cudaStreamCreateWithFlags(reinterpret_cast<cudaStream_t*>(&P.copy_stream), cudaStreamNonBlocking));
    CUDA_TRY(cudaEventCreateWithFlags(reinterpret_cast<cudaEvent_t*>(&P.ev_start), cudaEventDisableTiming));
  }
  dptrs.assign((size_t)P.nsub, nullptr);
  for (int32_t i = 0; i < P.nsub; i++) dptrs[(size_t)i] = static_cast<char*>(P.d_Lstage) + P.esz * P.Lstage_off[(size_t)i];
  std::vector<const void*> cp(dptrs.begin(), dptrs.end());
  sc_status st = set_Lptr(P, cp.data(), stream, err);
  if (st != SC_OK) return st;
  P.last_stream = stream_v;
  CUDA_TRY(cudaMemsetAsync(P.dev.err, 0, sizeof(unsigned long long) * (1 + (size_t)P.nsub), stream));
  return SC_OK;
}

sc_status assemble_range(Plan& P, int32_t s0, int32_t s1, void* stream, std::string& err) {
  return launch_range(P, s0, s1, static_cast<cudaStream_t>(stream), false, err);
}

sc_status assemble_host_pipelined(Plan& P, const void* const* Lhost, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  for (int32_t i = 0; i < P.nsub; i++)
    if (P.sub_nnz[(size_t)i] > 0 && !Lhost[i]) {
      err = "L_values_host[" + std::to_string(i) + "] is NULL";
      return SC_ERR_INVALID_ARG;
    }
  std::vector<void*> dptrs;
  sc_status st = assemble_stage_begin(P, dptrs, stream_v, err);
  if (st != SC_OK) return st;
  const int32_t nchunk = std::max<int32_t>(1, std::min<int32_t>(16, P.nsub / 64));
  while ((int32_t)P.ev_chunk.size() < nchunk) {
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P.ev_chunk.push_back(e);
  }
  cudaStream_t cs = static_cast<cudaStream_t>(P.copy_stream);
  // the staging buffer is reused: copies wait for everything enqueued on `stream` before this call
  CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_start), stream));
  CUDA_TRY(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(P.ev_start), 0));
  // pinned (device-mapped) host arrays: one gather kernel per chunk on the copy stream (reads host
  // memory over PCIe; no per-array copy calls); otherwise cudaMemcpyAsync per host-contiguous run
  bool mapped = true;
  std::vector<const void*> hdev((size_t)P.nsub, nullptr);
  for (int32_t i = 0; i < P.nsub && mapped; i++) {
    if (P.sub_nnz[(size_t)i] == 0) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, Lhost[i]) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
      cudaGetLastError();
      mapped = false;
    } else {
      hdev[(size_t)i] = at.devicePointer;
    }
  }
  if (mapped) {
    if (!P.d_hsrc) {
      void* d = nullptr;
      CUDA_TRY(cudaMalloc(&d, sizeof(void*) * (size_t)std::max(P.nsub, 1)));
      P.d_hsrc = d;
      int64_t* o = nullptr;
      CUDA_TRY(cudaMalloc(&o, sizeof(int64_t) * ((size_t)P.nsub + 1)));
      CUDA_TRY(cudaMemcpy(o, P.Lstage_off.data(), sizeof(int64_t) * ((size_t)P.nsub + 1), cudaMemcpyHostToDevice));
      P.d_Lstage_off = o;
      void* hp = nullptr;
      CUDA_TRY(cudaMallocHost(&hp, sizeof(void*) * (size_t)std::max(P.nsub, 1)));
      P.h_hsrc = static_cast<const void**>(hp);
      cudaEvent_t ev;
      CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(ev, cs));
      P.ev_hsrc = ev;
    }
    CUDA_TRY(cudaEventSynchronize(static_cast<cudaEvent_t>(P.ev_hsrc)));
    for (int32_t i = 0; i < P.nsub; i++) P.h_hsrc[i] = hdev[(size_t)i] ? hdev[(size_t)i] : Lhost[0];
    CUDA_TRY(cudaMemcpyAsync(P.d_hsrc, P.h_hsrc, sizeof(void*) * (size_t)P.nsub, cudaMemcpyHostToDevice, cs));
    CUDA_TRY(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_hsrc), cs));
  }
  for (int32_t k = 0; k < nchunk; k++) {
    const int32_t s0 = (int32_t)((int64_t)P.nsub * k / nchunk), s1 = (int32_t)((int64_t)P.nsub * (k + 1) / nchunk);
    if (mapped) {
      st = gather_host_range(reinterpret_cast<const void* const*>(P.d_hsrc), P.d_Lstage_off, P.d_Lstage, s0, s1, P.esz,
                             cs, err);
      if (st != SC_OK) return st;
    } else {
      int32_t i = s0;
      while (i < s1) {  // one cudaMemcpyAsync per run of host-contiguous subdomains
        if (P.sub_nnz[(size_t)i] == 0) {
          i++;
          continue;
        }
        const char* src = static_cast<const char*>(Lhost[i]);
        size_t bytes = (size_t)P.esz * (size_t)P.sub_nnz[(size_t)i];
        int32_t j = i + 1;
        while (j < s1 && P.sub_nnz[(size_t)j] > 0 && static_cast<const char*>(Lhost[j]) == src + bytes) {
          bytes += (size_t)P.esz * (size_t)P.sub_nnz[(size_t)j];
          j++;
        }
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(P.d_Lstage) + P.esz * P.Lstage_off[(size_t)i], src, bytes,
                                 cudaMemcpyHostToDevice, cs));
        i = j;
      }
    }
    cudaEvent_t e = static_cast<cudaEvent_t>(P.ev_chunk[(size_t)k]);
    CUDA_TRY(cudaEventRecord(e, cs));
    CUDA_TRY(cudaStreamWaitEvent(stream, e, 0));
    st = launch_range(P, s0, s1, stream, false, err);
    if (st != SC_OK) return st;
  }
  return SC_OK;
}

sc_status launch_apply(Plan& P, const double* lambda, double* q, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  P.last_stream = stream_v;
  const int na = (int)P.apply_tasks.size();
  if (na > 0) {
    if (P.esz == 4) apply_tile_kernel<float><<<(na + kApplyTPC - 1) / kApplyTPC, kThreads, 0, stream>>>(P.dev, lambda, na);
    else apply_tile_kernel<double><<<(na + kApplyTPC - 1) / kApplyTPC, kThreads, 0, stream>>>(P.dev, lambda, na);
    CUDA_TRY(cudaGetLastError());
  }
  if (P.n_lambda > 0) {
    const int64_t nb = (P.n_lambda + kThreads - 1) / kThreads;
    apply_scatter_kernel<<<(unsigned)nb, kThreads, 0, stream>>>(P.dev, q, P.n_lambda);
    CUDA_TRY(cudaGetLastError());
  }
  return SC_OK;
}

sc_status launch_prepare(Plan& P, const void* const* Lptr_host, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  sc_status st = ensure_factor_plan(P, err);
  if (st != SC_OK) return st;
  st = set_Lptr(P, Lptr_host, stream, err);
  if (st != SC_OK) return st;
  P.last_stream = stream_v;
  CUDA_TRY(cudaMemsetAsync(P.dev.err, 0, sizeof(unsigned long long) * (1 + (size_t)P.nsub), stream));
  return launch_stage(P, stream_v, err);
}

sc_status launch_apply_implicit(Plan& P, const double* lambda, double* q, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  if (!P.fac.ready || !P.fac.w_ready) {
    err = "no factor in the workspace: call sc_prepare_factor or sc_factorize_batch first";
    return SC_ERR_STATE;
  }
  P.last_stream = stream_v;
  sc_status st = launch_implicit_solve(P, lambda, stream_v, err);
  if (st != SC_OK) return st;
  if (P.n_lambda > 0) {
    const int64_t nb = (P.n_lambda + kThreads - 1) / kThreads;
    implicit_scatter_kernel<<<(unsigned)nb, kThreads, 0, stream>>>(P.dev, q, P.n_lambda);
    CUDA_TRY(cudaGetLastError());
  }
  return SC_OK;
}

sc_status device_check(Plan& P, std::string& err) {
  CUDA_TRY(cudaSetDevice(P.opt.device));
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(P.last_stream)));
  unsigned long long flag = 0;
  CUDA_TRY(cudaMemcpy(&flag, P.dev.err, sizeof(flag), cudaMemcpyDeviceToHost));
  if (flag) {
    err = "non-positive or non-finite diagonal of L in subdomain " + std::to_string((flag >> 32) - 1) + " column " +
          std::to_string(flag & 0xffffffffull);
    return SC_ERR_ZERO_PIVOT;
  }
  return SC_OK;
}

// zero-pivot flag of subdomain i only (other subdomains' F stay readable)
static sc_status device_check_sub(Plan& P, int32_t i, std::string& err) {
  CUDA_TRY(cudaSetDevice(P.opt.device));
  CUDA_TRY(cudaStreamSynchronize(static_cast<cudaStream_t>(P.last_stream)));
  unsigned long long flag = 0;
  CUDA_TRY(cudaMemcpy(&flag, P.dev.err + 1 + i, sizeof(flag), cudaMemcpyDeviceToHost));
  if (flag) {
    err = "non-positive or non-finite diagonal of L in subdomain " + std::to_string(i) + " column " +
          std::to_string(flag - 1);
    return SC_ERR_ZERO_PIVOT;
  }
  return SC_OK;
}

// `count` stored elements from element offset `off` of a device array in the plan's precision, as doubles
static sc_status copy_elements(Plan& P, const void* base, int64_t off, int64_t count, double* out, std::string& err) {
  if (P.esz == 8) {
    CUDA_TRY(cudaMemcpy(out, static_cast<const double*>(base) + off, 8 * (size_t)count, cudaMemcpyDeviceToHost));
    return SC_OK;
  }
  std::vector<float> tmp((size_t)count);
  CUDA_TRY(cudaMemcpy(tmp.data(), static_cast<const float*>(base) + off, 4 * (size_t)count, cudaMemcpyDeviceToHost));
  for (int64_t k = 0; k < count; k++) out[k] = (double)tmp[(size_t)k];
  return SC_OK;
}

sc_status copy_F_lower(Plan& P, int32_t i, std::vector<double>& out, std::string& err) {
  TRY(device_check_sub(P, i, err));
  const int64_t m = P.sub_m[(size_t)i], len = f_tiles((int)m) * kApplyTile * kApplyTile;
  out.resize((size_t)len);
  if (m > 0) TRY(copy_elements(P, P.dev.F, P.sub_F_base[(size_t)i], len, out.data(), err));
  return SC_OK;
}

sc_status export_F_device(Plan& P, int32_t i, double* F, int64_t ld, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  const int m = P.sub_m[(size_t)i];
  if (m == 0) return SC_OK;
  P.last_stream = stream_v;
  const dim3 grid((unsigned)((m + 15) / 16), (unsigned)((m + 15) / 16));
  if (P.esz == 4) export_F_kernel<float><<<grid, 256, 0, stream>>>(P.dev, i, F, ld);
  else export_F_kernel<double><<<grid, 256, 0, stream>>>(P.dev, i, F, ld);
  CUDA_TRY(cudaGetLastError());
  return SC_OK;
}

sc_status copy_X_strips(Plan& P, int32_t i, std::vector<double>& out, std::string& err) {
  TRY(device_check_sub(P, i, err));
  const ClassPlan& C = P.classes[(size_t)P.sub_cls[(size_t)i]];
  out.resize((size_t)C.x_doubles);
  if (C.x_doubles > 0)
    TRY(copy_elements(P, P.dev.X, P.sub_X_base[(size_t)i], C.x_doubles, out.data(), err));
  return SC_OK;
}

}  // namespace sc
