// factor.cu — numeric factorization on the device (§2.2, the
// numeric stage of the two-stage factorization; §4.5, its share of the preprocessing).
//
//   factor_kernel   left-looking supernodal Cholesky  P K_reg P^T = L L^T  for a whole batch.  One
//                   warp task per frame: the diagonal block of a factor panel (<= 32 columns) or 32 of
//                   the rows below it.  A persistent grid pulls tasks from a queue ordered so that every
//                   dependency comes first (factor_plan.cpp); a task waits (acquire) until the
//                   descendant panels it reads are complete, accumulates their updates
//                   L[rows, d] L[cols, d]^T with FP64 DMMA (m8n8k4) straight into the frame layout
//                   (fragments gathered by row lookup in R_d, so no scatter of partial results),
//                   subtracts from the K entries, then
//                     diagonal frame: Cholesky of the block in the warp's shared memory and the inverse
//                                     of the triangle (kept in the workspace for the row frames);
//                     row frame:      X = S inv(L_pp)^T by DMMA;
//                   and writes the finished rows to the workspace (read by ancestor panels) and to the
//                   caller's CSC values of L, then publishes (release) its completion.
// Deadlock freedom: a warp only waits for tasks that precede its own in the queue; those were taken
// earlier by running warps which themselves only wait for earlier tasks, so no residency assumption
// is needed.  Deterministic: every value is produced by one warp in a fixed order.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "sc_internal.h"

namespace sc {

namespace {

#define FCUDA(expr)                                                      \
  do {                                                                   \
    cudaError_t e_ = (expr);                                             \
    if (e_ != cudaSuccess) {                                             \
      err = std::string(#expr) + ": " + cudaGetErrorString(e_);          \
      return e_ == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA; \
    }                                                                    \
  } while (0)
#define FTRY(x)                  \
  do {                           \
    sc_status s_ = (x);          \
    if (s_ != SC_OK) return s_;  \
  } while (0)

constexpr int kFWarps = 4;              // warps per CTA (independent workers)
#ifndef SC_FPREFETCH
#define SC_FPREFETCH 0                  // software-pipelined k loop of the updates (costs spills at 128 regs)
#endif
#ifndef SC_FENCE_RELEASE
#define SC_FENCE_RELEASE 0              // 1: __threadfence + atomicAdd for the completion flags
#endif
#ifndef SC_FMINB
#define SC_FMINB 4                      // CTAs per SM the factor kernel's registers are sized for
#endif
constexpr int kSLd = kFW + 1;           // per-warp frame buffer: 32 x 33 doubles (column 32: 1 / l_jj)
constexpr int kFSmem = kFWarps * kFW * kSLd * 8;

__device__ __forceinline__ void fdmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
// Completion flags: producers write their results, then add to the flag with a release reduction.  Consumers spin with relaxed loads (no L1 invalidation per poll -- an ld.acquire costs a
// CCTL.IVALL each time) and, once every flag a warp needs is set, one fence.acq_rel.gpu completes the
// acquire pattern; the data itself is read with ld.global.cg (L2).
__device__ __forceinline__ int ld_relaxed(const int* p) {
  int v;
  asm volatile("ld.relaxed.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void fence_acq_rel() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
// Completion: the lanes' results are ordered before lane 0 by __syncwarp; a release reduction makes
// them visible with the flag (release patterns are cumulative), cheaper than __threadfence + atomicAdd
__device__ __forceinline__ void red_release_add(int* p, int v) {
#if SC_FENCE_RELEASE
  __threadfence();
  atomicAdd(p, v);
#else
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
#endif
}


__global__ void __launch_bounds__(32 * kFWarps, SC_FMINB) factor_kernel(DevFactor F, int64_t t0, int64_t t1, int slot,
                                                                 int stage) {
  extern __shared__ double fsm[];
  __shared__ int frow_s[kFWarps][kFW], rmap_s[kFWarps][kFW], cmap_s[kFWarps][kFW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* S = fsm + warp * kFW * kSLd;
  int* frow = frow_s[warp];
  int* rmap = rmap_s[warp];
  int* cmap = cmap_s[warp];
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = t0 + atomicAdd(F.queue + slot, 1);
    task = __shfl_sync(~0u, task, 0);
    if (task >= t1) break;
    const FTask tk = F.tasks[task];
    const bool part = tk.nf < 0;  // partial update task of a split frame (SC_FACTOR_SPLIT)
    if (part && stage) continue;  // staging has no updates
    const FPart pt = part ? F.parts[tk.frame] : FPart{};
    for (int fi = 0; fi < (part ? 1 : tk.nf); fi++) {
    const FFrame fr = F.frames[part ? pt.frame : tk.frame + fi];
    const FPanel pn = F.panels[fr.panel];
    const int sub = tk.sub;
    int* flags = F.flags + (F.sub_flag_base[sub] - F.cls_panel0[F.sub_cls[sub]]);  // indexed by global panel
    double* W = F.W + F.sub_W_base[sub];
    const bool diag = fr.r0 < 0;
    const int kw = pn.kw, nI = (fr.nrow + 7) >> 3, nJ = pn.kw8 >> 3;
    // the frame's row values (ascending), for the row lookups of the descendants' rows
    frow[lane] = lane < fr.nrow ? (diag ? pn.a + lane : __ldg(F.Rrows + pn.R_off + fr.r0 + lane)) : INT32_MAX;
    double acc[4][4][2];
#pragma unroll
    for (int I = 0; I < 4; I++)
#pragma unroll
      for (int J = 0; J < 4; J++) acc[I][J][0] = acc[I][J][1] = 0.0;

    // ---- updates from the finished descendant panels (left-looking), 32 list entries at a time:
    // lane l loads entry l's descriptor and its panel, waits (acquire) for that panel; then the
    // entries are processed in list order (deterministic)
    const int ub = part ? pt.u_begin : fr.u_begin, ue = part ? pt.u_end : fr.u_end;
    for (int u0 = ub; u0 < (stage ? ub : ue); u0 += 32) {
      const int nu = min(32, ue - u0);
      FFUpd U{};
      int dkw = 0, dkw8 = 0, dR = 0;
      int64_t dw = 0;
      if (lane < nu) {
        U = F.fupd[u0 + lane];
        const FPanel dn = F.panels[U.d];
        dkw = dn.kw;
        dkw8 = dn.kw8;
        dR = dn.R_off;
        dw = dn.w_off;
        const int* fl = flags + U.d;
        while ((ld_relaxed(fl) & 0xFFFF) < dn.nframe) __nanosleep(32);
      }
      __syncwarp();
      if (lane == 0) fence_acq_rel();
      __syncwarp();
      for (int j = 0; j < nu; j++) {
        const int s0 = __shfl_sync(~0u, U.s0, j), s1 = __shfl_sync(~0u, U.s1, j);
        const int k0 = __shfl_sync(~0u, U.k0, j), k1 = __shfl_sync(~0u, U.k1, j);
        const int ukw = __shfl_sync(~0u, dkw, j), ukw8 = __shfl_sync(~0u, dkw8, j), uR = __shfl_sync(~0u, dR, j);
        const int64_t uw = __shfl_sync(~0u, dw, j);
        const int32_t* Rd = F.Rrows + uR;
        // columns: R_d[s0, s1) are columns of this panel (value - a); rows: R_d[k0, k1) -> frame rows
        cmap[lane] = -1;
        rmap[lane] = -1;
        __syncwarp();
        if (lane < s1 - s0) cmap[__ldg(Rd + s0 + lane) - pn.a] = s0 + lane;
        if (diag) {
          if (lane < s1 - s0) rmap[__ldg(Rd + s0 + lane) - pn.a] = s0 + lane;
        } else {
          for (int w0 = k0; w0 < k1; w0 += 32) {
            if (w0 + lane < k1) {
              const int v = __ldg(Rd + w0 + lane);
              int lo = 0;  // first frame row >= v (frame rows ascending, padded with INT32_MAX)
#pragma unroll
              for (int step = 16; step > 0; step >>= 1)
                if (frow[lo + step - 1] < v) lo += step;
              if (frow[lo] == v) rmap[lo] = w0 + lane;
            }
          }
        }
        __syncwarp();
        const int ridx = rmap[lane], cidx = cmap[lane];
        const unsigned rm = __ballot_sync(~0u, ridx >= 0), cm = __ballot_sync(~0u, cidx >= 0);
        if (!rm || !cm) continue;
        // DMMA fragments gathered straight from the workspace rows of d (row-major, kw8 wide; L2):
        // A = L[frame rows, d] (row ridx), B = L[frame columns, d] (row cidx)
        const double* Wd = W + uw + t;
        int oa[4], ob[4];  // row offsets of the fragments' rows in d's workspace, -1 = zero / inactive block
#pragma unroll
        for (int I = 0; I < 4; I++) {
          const int r = __shfl_sync(~0u, ridx, 8 * I + g);
          oa[I] = (I < nI && ((rm >> (8 * I)) & 0xFFu) && r >= 0) ? r * ukw8 : -1;
        }
#pragma unroll
        for (int J = 0; J < 4; J++) {
          const int c = __shfl_sync(~0u, cidx, 8 * J + g);
          ob[J] = (J < nJ && ((cm >> (8 * J)) & 0xFFu) && c >= 0) ? c * ukw8 : -1;
        }
        bool ra[4], ca[4];  // warp-uniform block activity
#pragma unroll
        for (int I = 0; I < 4; I++) ra[I] = I < nI && ((rm >> (8 * I)) & 0xFFu);
#pragma unroll
        for (int J = 0; J < 4; J++) ca[J] = J < nJ && ((cm >> (8 * J)) & 0xFFu);
        for (int kb = 0; kb < ukw; kb += 4) {  // kb + t < ukw8: the padding columns of a row are zeros
          double a[4], b[4];
#pragma unroll
          for (int I = 0; I < 4; I++) a[I] = oa[I] >= 0 ? __ldcg(Wd + oa[I] + kb) : 0.0;
#pragma unroll
          for (int J = 0; J < 4; J++) b[J] = ob[J] >= 0 ? __ldcg(Wd + ob[J] + kb) : 0.0;
#pragma unroll
          for (int I = 0; I < 4; I++)
#pragma unroll
            for (int J = 0; J < 4; J++)
              if (ra[I] && ca[J] && (!diag || J <= I)) fdmma(acc[I][J][0], acc[I][J][1], a[I], b[J]);
        }
      }
    }


    if (part) {  // partial block -> its slot ([value][lane], coalesced), then release
      double* pb = F.pbuf + (F.sub_part_base[sub] + pt.slot) * 1024;
#pragma unroll
      for (int I = 0; I < 4; I++)
#pragma unroll
        for (int J = 0; J < 4; J++) {
          pb[((I * 4 + J) * 2) * 32 + lane] = acc[I][J][0];
          pb[((I * 4 + J) * 2 + 1) * 32 + lane] = acc[I][J][1];
        }
      __syncwarp();
      if (lane == 0) red_release_add(F.pflags + F.sub_part_base[sub] + pt.slot, 1);
      break;
    }
    if (!stage && fr.part_end > fr.part_begin) {  // the split-off partial blocks, in slot order
      for (int q = fr.part_begin; q < fr.part_end; q++) {
        const int64_t slot = F.sub_part_base[sub] + q;
        if (lane == 0) {
          while (ld_relaxed(F.pflags + slot) < 1) __nanosleep(32);
          fence_acq_rel();
        }
        __syncwarp();
        const double* pb = F.pbuf + slot * 1024;
#pragma unroll
        for (int I = 0; I < 4; I++)
#pragma unroll
          for (int J = 0; J < 4; J++) {
            acc[I][J][0] += __ldcg(pb + ((I * 4 + J) * 2) * 32 + lane);
            acc[I][J][1] += __ldcg(pb + ((I * 4 + J) * 2 + 1) * 32 + lane);
          }
      }
    }

    // ---- S = K entries - updates (frame layout, row-major in the warp's shared buffer); stage mode:
    // S = the frame's entries of the given L (zeros elsewhere)
    __syncwarp();
    if (stage) {
      for (int e = lane; e < kFW * kSLd; e += 32) S[e] = 0.0;
      __syncwarp();
      for (int e = fr.l_begin + lane; e < fr.l_end; e += 32) {
        const FEnt en = F.lent[e];
        S[(en.pos >> 5) * kSLd + (en.pos & 31)] =
            F.fp32 ? (double)__ldg(static_cast<const float*>(F.Lin[sub]) + en.q)
                   : __ldg(static_cast<const double*>(F.Lin[sub]) + en.q);
      }
    } else {
#pragma unroll
      for (int I = 0; I < 4; I++)
#pragma unroll
        for (int J = 0; J < 4; J++)
          if (I < nI && J < nJ) {
            S[(8 * I + g) * kSLd + 8 * J + 2 * t] = -acc[I][J][0];
            S[(8 * I + g) * kSLd + 8 * J + 2 * t + 1] = -acc[I][J][1];
          }
      __syncwarp();
      const double* Kv = static_cast<const double*>(F.Kptr[sub]);
      for (int e = fr.k_begin + lane; e < fr.k_end; e += 32) {
        const FEnt en = F.kent[e];
        S[(en.pos >> 5) * kSLd + (en.pos & 31)] += __ldg(Kv + en.q);
      }
    }
    __syncwarp();

    if (diag && stage) {  // the triangle is given: pivots checked, reciprocals for the inverse
      if (lane < kw) {
        const double d = S[lane * kSLd + lane];
        if (!(d > 0.0) || !isfinite(d)) {
          atomicCAS(F.err, 0ull, ((unsigned long long)(sub + 1) << 32) | (unsigned long long)(pn.a + lane));
          atomicCAS(F.err + 1 + sub, 0ull, (unsigned long long)(pn.a + lane) + 1ull);
        }
        S[lane * kSLd + kFW] = 1.0 / d;
      }
      __syncwarp();
    }
    if (diag) {
      // ---- Cholesky of the diagonal block, left-looking by columns (lane = row): column j needs the
      // finished columns k < j only, so every lane runs the same k loop (no divergence) and one
      // __syncwarp per column suffices
      for (int j = 0; j < (stage ? 0 : kw); j++) {
        double v = S[lane * kSLd + j];
        for (int k = 0; k < j; k++) v = fma(-S[lane * kSLd + k], S[j * kSLd + k], v);
        double djj = __shfl_sync(~0u, v, j);
        if (!(djj > 0.0) || !isfinite(djj)) {
          if (lane == 0) {
            atomicCAS(F.err, 0ull, ((unsigned long long)(sub + 1) << 32) | (unsigned long long)(pn.a + j));
            atomicCAS(F.err + 1 + sub, 0ull, (unsigned long long)(pn.a + j) + 1ull);
          }
          djj = 1.0;
        }
        const double l = sqrt(djj), rl = 1.0 / l;
        if (lane == j) {
          S[j * kSLd + j] = l;
          S[j * kSLd + kFW] = rl;
        }
        if (lane > j && lane < kw) S[lane * kSLd + j] = v * rl;
        __syncwarp();
      }
      // ---- inverse of the triangle: lane c computes column c (forward substitution, registers)
      double x[kFW];
#pragma unroll
      for (int i = 0; i < kFW; i++) {
        double s = (i == lane) ? 1.0 : 0.0;
        if (i < kw && i > lane) {
#pragma unroll
          for (int k = 0; k < i; k++)
            if (k >= lane) s -= S[i * kSLd + k] * x[k];
        }
        x[i] = (i < kw && i >= lane) ? s * S[i * kSLd + kFW] : 0.0;
      }
      double* Winv = W + pn.inv_off;
      if (lane < pn.kw8) {
#pragma unroll
        for (int i = 0; i < kFW; i++)
          if (i < pn.kw8) Winv[lane * pn.kw8 + i] = x[i];
      }
    } else if (stage) {  // the rows of the given L go to the workspace as they are (row-major, kw8 wide)
      double* Wp = W + pn.w_off;
      if (lane < fr.nrow)
        for (int c = 0; c < pn.kw8; c += 2)
          *reinterpret_cast<double2*>(Wp + (int64_t)(fr.r0 + lane) * pn.kw8 + c) =
              make_double2(S[lane * kSLd + c], S[lane * kSLd + c + 1]);
    } else {
      // ---- wait for the panel's own diagonal frame, then X = S inv(L_pp)^T
      if (lane == 0) {
        const int* fl = flags + fr.panel;
        while (!(ld_relaxed(fl) & 0x10000)) __nanosleep(32);
        fence_acq_rel();
      }
      __syncwarp();
      const double* Winv = W + pn.inv_off;
      const int ld8 = pn.kw8;
#pragma unroll
      for (int I = 0; I < 4; I++)
#pragma unroll
        for (int J = 0; J < 4; J++) acc[I][J][0] = acc[I][J][1] = 0.0;
      for (int k0 = 0; k0 < pn.kw8; k0 += 4) {
        double a[4], b[4];
#pragma unroll
        for (int I = 0; I < 4; I++) a[I] = I < nI ? S[(8 * I + g) * kSLd + k0 + t] : 0.0;
#pragma unroll
        for (int J = 0; J < 4; J++) b[J] = J < nJ ? __ldcg(Winv + (int64_t)(k0 + t) * ld8 + 8 * J + g) : 0.0;
#pragma unroll
        for (int I = 0; I < 4; I++)
#pragma unroll
          for (int J = 0; J < 4; J++)
            if (I < nI && J < nJ) fdmma(acc[I][J][0], acc[I][J][1], a[I], b[J]);
      }
      __syncwarp();
      double* Wp = W + pn.w_off;
#pragma unroll
      for (int I = 0; I < 4; I++)
#pragma unroll
        for (int J = 0; J < 4; J++)
          if (I < nI && J < nJ) {
            const int r = 8 * I + g, c = 8 * J + 2 * t;
            S[r * kSLd + c] = acc[I][J][0];
            S[r * kSLd + c + 1] = acc[I][J][1];
            if (r < fr.nrow)  // row-major, kw8 wide (the padding columns are exact zeros)
              *reinterpret_cast<double2*>(Wp + (int64_t)(fr.r0 + r) * pn.kw8 + c) = make_double2(acc[I][J][0], acc[I][J][1]);
          }
    }
    __syncwarp();
    // ---- L values of this frame into the caller's CSC array
    if (stage) {
    } else if (F.fp32) {
      float* Lo = static_cast<float*>(F.Lout[sub]);
      for (int e = fr.l_begin + lane; e < fr.l_end; e += 32) {
        const FEnt en = F.lent[e];
        Lo[en.q] = (float)S[(en.pos >> 5) * kSLd + (en.pos & 31)];
      }
    } else {
      double* Lo = static_cast<double*>(F.Lout[sub]);
      for (int e = fr.l_begin + lane; e < fr.l_end; e += 32) {
        const FEnt en = F.lent[e];
        Lo[en.q] = S[(en.pos >> 5) * kSLd + (en.pos & 31)];
      }
    }
    __syncwarp();
    if (lane == 0) {
      red_release_add(flags + fr.panel, diag ? 0x10001 : 1);
    }
    }  // frames of the task
  }
}

// ------------------------------------------------------------------------------------------------
// Implicit apply on the factor workspace (eq. dualop_apply_impl):
// x = P B~^T lambda_i, y = L^{-1} x (forward), z = L^{-T} y (backward), u = B~ P^T z; no F.  One warp
// task per (subdomain, factor panel), pulled from a queue in level order (forward) or its reverse
// (backward), with per-panel completion flags (acquire/release) like the factorization: all panels
// of all subdomains whose dependencies are done run concurrently.  Each entry of the factor is read
// once per direction; every sum has a fixed order (deterministic).
//   forward  (panel p): b_c = sum over the permuted row a_p + c of B~^T lambda (CSR by row);
//                       b -= L[cols of p, d] y_d for the descendants d (their rows R_d[s0, s1));
//                       y_p = inv(L_pp) b.
//   backward (panel p): v = y_p - L[R_p, p]^T z[R_p] (after the ancestors owning R_p);
//                       z_p = inv(L_pp)^T v.
// ------------------------------------------------------------------------------------------------
__device__ __forceinline__ void wait_flag(const int* f, int target) {
  while (ld_relaxed(f) < target) __nanosleep(32);
}

// b = P B~^T lambda_i for every permuted row of every subdomain (by row, fixed order), into the work
// vectors; the forward tasks then read their b_p with one load
__global__ void __launch_bounds__(256) implicit_b_kernel(DevFactor F, const double* __restrict__ lambda, int nmax) {
  const int sub = blockIdx.y, cls = F.sub_cls[sub];
  const int n = (int)(F.sub_x_base[sub + 1] - F.sub_x_base[sub]);
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  const int32_t* rp = F.bt_rp + F.cls_bt0[cls];
  const int64_t* slm = F.slm + F.sub_slm_off[sub];
  double b = 0.0;
  for (int e = rp[r]; e < rp[r + 1]; e++) b = fma(F.bt_v[e], __ldg(lambda + slm[F.bt_a[e]]), b);
  F.xv[F.sub_x_base[sub] + r] = b;
  (void)nmax;
}

__global__ void __launch_bounds__(32 * kFWarps) implicit_fwd_kernel(DevFactor F, int64_t ntask) {
  __shared__ double acc_s[kFWarps][kFW];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* acc = acc_s[warp];
  // one task at a time: grabbing the next task early would hold it back while this one runs (its
  // dependants would wait longer: measured cfg2 4.3 vs 3.4 ms per apply)
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = atomicAdd(F.queue + 2, 1);
    task = __shfl_sync(~0u, task, 0);
    if (task >= ntask) break;
    const I2 pt = F.ptasks[task];
    const bool part = pt.y < 0;  // partial updates of a split diagonal frame
    const FPart pp = part ? F.parts[-1 - pt.y] : FPart{};
    const FFrame fr = F.frames[part ? pp.frame : F.panels[pt.y].frame_begin];
    const FPanel pn = F.panels[fr.panel];
    const int pg = fr.panel;
    const int sub = pt.x, cls = F.sub_cls[sub];
    int* flags = F.flags + (F.sub_flag_base[sub] - F.cls_panel0[cls]);
    const double* W = F.W + F.sub_W_base[sub];
    double* x = F.xv + F.sub_x_base[sub];
    const int kw = pn.kw;
    const double b = !part && lane < kw ? x[pn.a + lane] : 0.0;  // P B~^T lambda (implicit_b_kernel)
    acc[lane] = 0.0;
    const int ub = part ? pp.u_begin : fr.u_begin, ue = part ? pp.u_end : fr.u_end;
    for (int u0 = ub; u0 < ue; u0 += 32) {
      const int nu = min(32, ue - u0);
      FFUpd U{};
      int dkw = 0, dnR = 0, dR = 0, da = 0;
      int64_t dw = 0;
      if (lane < nu) {
        U = F.fupd[u0 + lane];
        const FPanel dn = F.panels[U.d];
        dkw = dn.kw;
        dnR = dn.kw8;  // row stride of the workspace rows
        dR = dn.R_off;
        da = dn.a;
        dw = dn.w_off;
        wait_flag(flags + U.d, 1);
      }
      __syncwarp();
      if (lane == 0) fence_acq_rel();
      __syncwarp();
      for (int j = 0; j < nu; j++) {
        const int s0 = __shfl_sync(~0u, U.s0, j), s1 = __shfl_sync(~0u, U.s1, j);
        const int ukw = __shfl_sync(~0u, dkw, j), ukw8 = __shfl_sync(~0u, dnR, j), uR = __shfl_sync(~0u, dR, j);
        const int ua = __shfl_sync(~0u, da, j);
        const int64_t uw = __shfl_sync(~0u, dw, j);
        if (lane < s1 - s0) {
          const double* row = W + uw + (int64_t)(s0 + lane) * ukw8;  // row-major, kw8 wide
          double v = 0.0;
#pragma unroll
          for (int h = 0; h < kFW; h += 16) {  // 16 loads in flight, then the fixed-order sum
            double w[16], xk[16];
#pragma unroll
            for (int k = 0; k < 16; k += 2) {
              const double2 w2 = h + k < ukw ? __ldcg(reinterpret_cast<const double2*>(row + h + k)) : make_double2(0.0, 0.0);
              w[k] = w2.x;
              w[k + 1] = w2.y;
            }
#pragma unroll
            for (int k = 0; k < 16; k++) xk[k] = h + k < ukw ? __ldcg(x + ua + h + k) : 0.0;
#pragma unroll
            for (int k = 0; k < 16; k++) v = fma(w[k], xk[k], v);
          }
          acc[__ldg(F.Rrows + uR + s0 + lane) - pn.a] += v;
        }
        __syncwarp();
      }
    }
    __syncwarp();
    if (part) {  // partial sums -> the part's slot, then release
      const int64_t slot = F.sub_part_base[sub] + pp.slot;
      F.pbuf[slot * 1024 + lane] = acc[lane];
      __syncwarp();
      if (lane == 0) red_release_add(F.pflags + slot, 1);
      continue;
    }
    for (int q = fr.part_begin; q < fr.part_end; q++) {  // the split-off partial sums, in slot order
      const int64_t slot = F.sub_part_base[sub] + q;
      if (lane == 0) {
        while (ld_relaxed(F.pflags + slot) < 1) __nanosleep(32);
        fence_acq_rel();
      }
      __syncwarp();
      acc[lane] += __ldcg(F.pbuf + slot * 1024 + lane);
      __syncwarp();
    }
    const double v = lane < kw ? b - acc[lane] : 0.0;
    const double* inv = W + pn.inv_off;  // column-major kw8 x kw8: inv[i][k] at k kw8 + i
    double y = 0.0;
#pragma unroll
    for (int k = 0; k < kFW; k++) {
      const double vk = __shfl_sync(~0u, v, k);
      const double iv = (k < kw && lane >= k && lane < kw) ? __ldcg(inv + (int64_t)k * pn.kw8 + lane) : 0.0;
      y = fma(iv, vk, y);
    }
    if (lane < kw) x[pn.a + lane] = y;
    __syncwarp();
    if (lane == 0) {
      red_release_add(flags + pg, 1);
    }
  }
}

__global__ void __launch_bounds__(32 * kFWarps) implicit_bwd_kernel(DevFactor F, int64_t ntask) {
  const int lane = threadIdx.x & 31;
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = atomicAdd(F.queue + 3, 1);
    task = __shfl_sync(~0u, task, 0);
    if (task >= ntask) break;
    const I2 pt = F.ptasks[ntask - 1 - task];
    if (pt.y < 0) continue;  // partial forward task: nothing to do backward
    const FPanel pn = F.panels[pt.y];
    const int sub = pt.x, cls = F.sub_cls[sub];
    int* flags = F.flags + (F.sub_flag_base[sub] - F.cls_panel0[cls]);
    const double* W = F.W + F.sub_W_base[sub];
    double* x = F.xv + F.sub_x_base[sub];
    const int kw = pn.kw;
    for (int a0 = pn.anc_begin + lane; a0 < pn.anc_end; a0 += 32) wait_flag(flags + F.anc[a0].d, 2);
    __syncwarp();
    if (lane == 0) fence_acq_rel();
    __syncwarp();
    // s_k = sum_r L[R_p[r], a + k] z[R_p[r]]: lanes over rows, 32 partial sums per lane
    double part[kFW];
#pragma unroll
    for (int k = 0; k < kFW; k++) part[k] = 0.0;
    const double* Wp = W + pn.w_off;
    for (int r0 = 0; r0 < pn.nR; r0 += 32) {
      const int r = r0 + lane;
      const double z = r < pn.nR ? __ldcg(x + __ldg(F.Rrows + pn.R_off + r)) : 0.0;
      const double* row = Wp + (int64_t)r * pn.kw8;  // row-major, kw8 wide
#pragma unroll
      for (int k = 0; k < kFW; k += 2)
        if (k < kw && r < pn.nR) {
          const double2 w2 = __ldcg(reinterpret_cast<const double2*>(row + k));
          part[k] = fma(w2.x, z, part[k]);
          part[k + 1] = fma(w2.y, z, part[k + 1]);
        }
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < kFW; k++) {
      if (k < kw) {
        double v = part[k];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(~0u, v, o);
        if (lane == k) s = v;
      }
    }
    const double v = lane < kw ? __ldcg(x + pn.a + lane) - s : 0.0;
    const double* inv = W + pn.inv_off;  // z_j = sum_{i >= j} inv[i][j] v_i
    double z = 0.0;
#pragma unroll
    for (int i = 0; i < kFW; i++) {
      const double vi = __shfl_sync(~0u, v, i);
      const double iv = (i < kw && lane <= i && lane < kw) ? __ldcg(inv + (int64_t)lane * pn.kw8 + i) : 0.0;
      z = fma(iv, vi, z);
    }
    __syncwarp();
    if (lane < kw) x[pn.a + lane] = z;
    __syncwarp();
    if (lane == 0) {
      red_release_add(flags + pt.y, 1);
    }
  }
}

// u[a] = (B~ P^T z)_a per subdomain and stepped column, into DevPlan::upart (then the plan's
// deterministic scatter-sum over subdomains)
__global__ void __launch_bounds__(256) implicit_gather_kernel(DevPlan P, const double* __restrict__ xv,
                                                              const int64_t* __restrict__ sub_x_base) {
  const int sub = blockIdx.x, cls = P.sub_cls[sub], m = P.sub_m[sub];
  const int32_t* ibp = P.ib_ptr + P.cls_ib0[cls];
  const double* x = xv + sub_x_base[sub];
  double* u = P.upart + P.sub_slm_off[sub];
  for (int a = threadIdx.x; a < m; a += blockDim.x) {
    double s = 0.0;
    for (int e = ibp[a]; e < ibp[a + 1]; e++) s = fma(P.ib_val[e], x[P.ib_row[e]], s);
    u[a] = s;
  }
}

// ------------------------------------------------------------------------------------------------
// Host -> device gather of many small pinned host arrays in one launch: the kernel reads mapped
// (pinned, UVA) host memory over PCIe directly, one block per array, so a batch of a thousand
// 160-KB K arrays costs one launch instead of a thousand cudaMemcpyAsync calls.
// ------------------------------------------------------------------------------------------------
template <typename E>
__global__ void __launch_bounds__(256) gather_host_kernel(const E* const* __restrict__ src,
                                                          const int64_t* __restrict__ off, E* __restrict__ dst,
                                                          int s0, int s1) {
  for (int sgi = s0 + blockIdx.x; sgi < s1; sgi += gridDim.x) {
    const E* a = src[sgi];
    const int64_t o = off[sgi], n = off[sgi + 1] - o;
    E* d = dst + o;
    constexpr int V = 16 / sizeof(E);  // elements per 16-byte vector
    if ((((uintptr_t)a | (uintptr_t)d) & 15) == 0) {
      const int64_t nv = n / V;
      for (int64_t i = threadIdx.x; i < nv; i += blockDim.x)
        reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(a)[i];
      for (int64_t i = nv * V + threadIdx.x; i < n; i += blockDim.x) d[i] = a[i];
    } else {
      for (int64_t i = threadIdx.x; i < n; i += blockDim.x) d[i] = a[i];
    }
  }
}

template <typename V>
sc_status fupload(FactorPlan& F, const std::vector<V>& v, const V** dst, std::string& err) {
  void* d = nullptr;
  FCUDA(cudaMalloc(&d, std::max<size_t>(v.size() * sizeof(V), 16)));
  F.allocations.push_back(d);
  if (!v.empty()) FCUDA(cudaMemcpy(d, v.data(), v.size() * sizeof(V), cudaMemcpyHostToDevice));
  *dst = static_cast<const V*>(d);
  return SC_OK;
}
template <typename V>
sc_status falloc(FactorPlan& F, int64_t count, V** dst, std::string& err) {
  void* d = nullptr;
  FCUDA(cudaMalloc(&d, std::max<size_t>((size_t)count * sizeof(V), 16)));
  F.allocations.push_back(d);
  *dst = static_cast<V*>(d);
  return SC_OK;
}

constexpr int kQueueSlots = 64;  // one task counter per launch of a call (chunks of the host pipeline)

// upload the per-call K / L pointer tables (pinned staging guarded by an event)
sc_status set_ptrs(Plan& P, const void* const* K, void* const* L, cudaStream_t stream, std::string& err) {
  FactorPlan& F = P.fac;
  FCUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(F.ptr_event)));
  for (int32_t i = 0; i < P.nsub; i++) {
    F.h_ptrs[i] = const_cast<void*>(K[i]);
    F.h_ptrs[P.nsub + i] = L[i];
  }
  FCUDA(cudaMemcpyAsync(F.d_ptrs, F.h_ptrs, sizeof(void*) * 2 * (size_t)P.nsub, cudaMemcpyHostToDevice, stream));
  FCUDA(cudaEventRecord(static_cast<cudaEvent_t>(F.ptr_event), stream));
  return SC_OK;
}

int factor_grid(int64_t ntask) {
  static int nsm = 0, per_sm = 0;
  if (!nsm) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, factor_kernel, 32 * kFWarps, kFSmem);
    per_sm = std::max(per_sm, 1);
  }
  const int64_t want = (ntask + kFWarps - 1) / kFWarps;
  return (int)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)nsm * per_sm));
}

sc_status factor_range(Plan& P, int64_t t0, int64_t t1, int slot, cudaStream_t stream, std::string& err,
                       int stage = 0) {
  if (t1 <= t0) return SC_OK;
  factor_kernel<<<factor_grid(t1 - t0), 32 * kFWarps, kFSmem, stream>>>(P.fac.dev, t0, t1, slot, stage);
  FCUDA(cudaGetLastError());
  return SC_OK;
}

}  // namespace

void free_factor_device(Plan& P) {
  FactorPlan& F = P.fac;
  if (F.allocations.empty() && !F.h_ptrs) return;
  cudaSetDevice(P.opt.device);
  cudaDeviceSynchronize();
  for (void* p : F.allocations) cudaFree(p);
  F.allocations.clear();
  if (F.h_ptrs) cudaFreeHost(F.h_ptrs);
  F.h_ptrs = nullptr;
  if (F.ptr_event) cudaEventDestroy(static_cast<cudaEvent_t>(F.ptr_event));
  F.ptr_event = nullptr;
  if (F.d_Kstage) cudaFree(F.d_Kstage);
  F.d_Kstage = nullptr;
  if (F.d_hptrs) cudaFree(F.d_hptrs);
  if (F.d_Kstage_off) cudaFree(F.d_Kstage_off);
  if (F.h_hptrs) cudaFreeHost((void*)F.h_hptrs);
  F.d_hptrs = nullptr;
  F.d_Kstage_off = nullptr;
  F.h_hptrs = nullptr;
  if (F.hptr_event) cudaEventDestroy(static_cast<cudaEvent_t>(F.hptr_event));
  F.hptr_event = nullptr;


  F.d_ptrs = nullptr;
  F.ready = false;
}

sc_status upload_factor_plan(Plan& P, std::string& err) {
  FactorPlan& F = P.fac;
  FCUDA(cudaSetDevice(P.opt.device));
  DevFactor D{};
  FTRY(fupload(F, F.panels, &D.panels, err));
  FTRY(fupload(F, F.Rrows, &D.Rrows, err));
  FTRY(fupload(F, F.fupd, &D.fupd, err));
  FTRY(fupload(F, F.frames, &D.frames, err));
  FTRY(fupload(F, F.kent, &D.kent, err));
  FTRY(fupload(F, F.lent, &D.lent, err));
  FTRY(fupload(F, F.tasks, &D.tasks, err));
  FTRY(fupload(F, P.sub_cls, &D.sub_cls, err));
  FTRY(fupload(F, F.sub_W_base, &D.sub_W_base, err));
  FTRY(fupload(F, F.sub_flag_base, &D.sub_flag_base, err));
  FTRY(fupload(F, F.cls_panel0, &D.cls_panel0, err));
  FTRY(fupload(F, F.anc, &D.anc, err));
  FTRY(fupload(F, F.ptasks, &D.ptasks, err));
  {  // split frames: partial tasks, their slots and blocks
    std::vector<FPart> pv(F.parts);
    if (pv.empty()) pv.push_back(FPart{});
    FTRY(fupload(F, pv, &D.parts, err));
    FTRY(fupload(F, F.cls_part0, &D.cls_part0, err));
    FTRY(fupload(F, F.sub_part_base, &D.sub_part_base, err));
    FTRY(falloc(F, std::max<int64_t>(F.nparts, 1), &D.pflags, err));
    FTRY(falloc(F, std::max<int64_t>(F.nparts, 1) * 1024, &D.pbuf, err));
  }
  FTRY(fupload(F, F.bt_rp, &D.bt_rp, err));
  FTRY(fupload(F, F.bt_a, &D.bt_a, err));
  FTRY(fupload(F, F.bt_v, &D.bt_v, err));
  FTRY(fupload(F, F.cls_bt0, &D.cls_bt0, err));
  FTRY(fupload(F, F.sub_x_base, &D.sub_x_base, err));
  FTRY(falloc(F, F.sub_x_base.back(), &D.xv, err));
  D.Lin = P.dev.Lptr;
  D.slm = P.dev.slm;
  D.sub_slm_off = P.dev.sub_slm_off;
  FTRY(falloc(F, F.W_doubles, &D.W, err));

  FTRY(falloc(F, F.nflags, &D.flags, err));
  FTRY(falloc(F, kQueueSlots, &D.queue, err));
  void** dp = nullptr;
  FTRY(falloc(F, 2 * (int64_t)std::max(P.nsub, 1), &dp, err));
  F.d_ptrs = dp;
  D.Kptr = reinterpret_cast<const void* const*>(dp);
  D.Lout = dp + P.nsub;
  void* hp = nullptr;
  FCUDA(cudaMallocHost(&hp, sizeof(void*) * 2 * (size_t)std::max(P.nsub, 1)));
  F.h_ptrs = static_cast<void**>(hp);
  cudaEvent_t ev;
  FCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  F.ptr_event = ev;
  FCUDA(cudaEventRecord(ev, 0));
  FCUDA(cudaFuncSetAttribute((const void*)factor_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kFSmem));
  D.err = P.dev.err;
  D.fp32 = P.esz == 4 ? 1 : 0;
  F.dev = D;
  F.ready = true;
  return SC_OK;
}

// Mapped-host gather of arrays [s0, s1) (element size esz) into dst at the offsets `off` (device).
sc_status gather_host_range(const void* const* d_src, const int64_t* d_off, void* d_dst, int32_t s0, int32_t s1,
                            int esz, void* stream_v, std::string& err) {
  if (s1 <= s0) return SC_OK;
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  const int grid = std::max(1, std::min(s1 - s0, 256));
  if (esz == 8)
    gather_host_kernel<double><<<grid, 256, 0, stream>>>(reinterpret_cast<const double* const*>(d_src), d_off,
                                                          static_cast<double*>(d_dst), s0, s1);
  else
    gather_host_kernel<float><<<grid, 256, 0, stream>>>(reinterpret_cast<const float* const*>(d_src), d_off,
                                                         static_cast<float*>(d_dst), s0, s1);
  FCUDA(cudaGetLastError());
  return SC_OK;
}

sc_status ensure_factor_plan(Plan& P, std::string& err) {
  if (P.fac.ready) return SC_OK;
  sc_status st = build_factor_plan(P, nullptr, P.nsub, err);
  if (st == SC_OK) st = upload_factor_plan(P, err);
  if (st != SC_OK) {
    free_factor_device(P);
    P.fac = FactorPlan();
    return st;
  }
  P.stats.device_bytes += 8.0 * (double)(P.fac.W_doubles + P.fac.sub_x_base.back());
  return SC_OK;
}

sc_status launch_factorize(Plan& P, const void* const* Kptr, void* const* Lout, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  FactorPlan& F = P.fac;
  FCUDA(cudaSetDevice(P.opt.device));
  for (int32_t i = 0; i < P.nsub; i++) {
    if (!Kptr[i] && F.sub_nnzK[(size_t)i] > 0) {
      err = "K_values[" + std::to_string(i) + "] is NULL";
      return SC_ERR_INVALID_ARG;
    }
    if (!Lout[i] && P.sub_nnz[(size_t)i] > 0) {
      err = "L_values[" + std::to_string(i) + "] is NULL";
      return SC_ERR_INVALID_ARG;
    }
  }
  FTRY(set_ptrs(P, Kptr, Lout, stream, err));
  P.last_stream = stream_v;
  F.w_ready = true;  // the workspace holds this factorization (implicit apply)
  FCUDA(cudaMemsetAsync(P.dev.err, 0, sizeof(unsigned long long) * (1 + (size_t)P.nsub), stream));
  FCUDA(cudaMemsetAsync(F.dev.flags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nflags, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.pflags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nparts, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  return factor_range(P, 0, F.task_chunk[0], 0, stream, err);
}

// Stage the workspace from the plan's current L table (sc_prepare_factor): W <- L[R_p, p] and
// inv(L_pp) for every panel, no factorization.
sc_status launch_stage(Plan& P, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  FactorPlan& F = P.fac;
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  FTRY(factor_range(P, 0, F.task_chunk[0], 0, stream, err, 1));
  F.w_ready = true;
  return SC_OK;
}

// Implicit apply: forward and backward substitution over the workspace, then u = B~ P^T z into the
// plan's per-(subdomain, multiplier) buffer (the caller's scatter-sum follows).
sc_status launch_implicit_solve(Plan& P, const double* lambda, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  FactorPlan& F = P.fac;
  const int64_t nt = (int64_t)F.ptasks.size();
  FCUDA(cudaMemsetAsync(F.dev.flags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nflags, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.pflags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nparts, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  if (nt > 0) {
    static int nsm = 0;
    if (!nsm) {
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
    }
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((nt + kFWarps - 1) / kFWarps, (int64_t)nsm * 8));
    int nmax = 0;
    for (int32_t i = 0; i < P.nsub; i++) nmax = std::max(nmax, (int)(F.sub_x_base[(size_t)i + 1] - F.sub_x_base[(size_t)i]));
    implicit_b_kernel<<<dim3((unsigned)((nmax + 255) / 256), (unsigned)P.nsub), 256, 0, stream>>>(F.dev, lambda, nmax);
    FCUDA(cudaGetLastError());
    implicit_fwd_kernel<<<grid, 32 * kFWarps, 0, stream>>>(F.dev, nt);
    FCUDA(cudaGetLastError());
    implicit_bwd_kernel<<<grid, 32 * kFWarps, 0, stream>>>(F.dev, nt);
    FCUDA(cudaGetLastError());
  }
  if (P.nsub > 0) {
    implicit_gather_kernel<<<P.nsub, 256, 0, stream>>>(P.dev, F.dev.xv, F.dev.sub_x_base);
    FCUDA(cudaGetLastError());
  }
  return SC_OK;
}

// Host-fed path: H2D of every subdomain's K values (per chunk of subdomains on the plan's copy stream),
// then one factorization of the whole batch (level order over all subdomains: its critical path is
// one panel chain, where per-chunk factorizations would serialise one chain per chunk) into the plan's
// L staging buffer, then the assembly, both on `stream`.
sc_status factorize_assemble_host(Plan& P, const void* const* Khost, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  FactorPlan& F = P.fac;
  FCUDA(cudaSetDevice(P.opt.device));
  for (int32_t i = 0; i < P.nsub; i++)
    if (!Khost[i] && F.sub_nnzK[(size_t)i] > 0) {
      err = "K_values_host[" + std::to_string(i) + "] is NULL";
      return SC_ERR_INVALID_ARG;
    }
  if (!F.d_Kstage) {
    F.Kstage_off.assign((size_t)P.nsub + 1, 0);
    for (int32_t i = 0; i < P.nsub; i++) F.Kstage_off[(size_t)i + 1] = F.Kstage_off[(size_t)i] + F.sub_nnzK[(size_t)i];
    void* d = nullptr;
    FCUDA(cudaMalloc(&d, std::max<size_t>(8 * (size_t)F.Kstage_off.back(), 16)));
    F.d_Kstage = d;
  }
  std::vector<void*> Lst;
  FTRY(assemble_stage_begin(P, Lst, stream_v, err));  // L staging + pointer table + error reset
  std::vector<const void*> Kd((size_t)P.nsub);
  for (int32_t i = 0; i < P.nsub; i++) Kd[(size_t)i] = static_cast<char*>(F.d_Kstage) + 8 * F.Kstage_off[(size_t)i];
  FTRY(set_ptrs(P, Kd.data(), Lst.data(), stream, err));
  F.w_ready = true;
  FCUDA(cudaMemsetAsync(F.dev.flags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nflags, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.pflags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nparts, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  // pinned (device-mapped) host arrays: one gather kernel on `stream`; otherwise cudaMemcpyAsync per
  // host-contiguous run on the copy stream
  bool mapped = true;
  std::vector<const void*> hdev((size_t)P.nsub, nullptr);
  for (int32_t i = 0; i < P.nsub && mapped; i++) {
    if (F.sub_nnzK[(size_t)i] == 0) continue;
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, Khost[i]) != cudaSuccess || at.type != cudaMemoryTypeHost || !at.devicePointer) {
      cudaGetLastError();
      mapped = false;
    } else {
      hdev[(size_t)i] = at.devicePointer;
    }
  }
  if (mapped) {
    if (!F.d_hptrs) {
      void* d = nullptr;
      FCUDA(cudaMalloc(&d, sizeof(void*) * (size_t)std::max(P.nsub, 1)));
      F.d_hptrs = d;
      int64_t* o = nullptr;
      FCUDA(cudaMalloc(&o, sizeof(int64_t) * ((size_t)P.nsub + 1)));
      FCUDA(cudaMemcpy(o, F.Kstage_off.data(), sizeof(int64_t) * ((size_t)P.nsub + 1), cudaMemcpyHostToDevice));
      F.d_Kstage_off = o;
      void* hp = nullptr;
      FCUDA(cudaMallocHost(&hp, sizeof(void*) * (size_t)std::max(P.nsub, 1)));
      F.h_hptrs = static_cast<const void**>(hp);
      cudaEvent_t ev;
      FCUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
      FCUDA(cudaEventRecord(ev, stream));
      F.hptr_event = ev;
    }
    FCUDA(cudaEventSynchronize(static_cast<cudaEvent_t>(F.hptr_event)));  // the last upload consumed the pinned table
    for (int32_t i = 0; i < P.nsub; i++) F.h_hptrs[i] = hdev[(size_t)i] ? hdev[(size_t)i] : Khost[0];
    FCUDA(cudaMemcpyAsync(F.d_hptrs, F.h_hptrs, sizeof(void*) * (size_t)P.nsub, cudaMemcpyHostToDevice, stream));
    FCUDA(cudaEventRecord(static_cast<cudaEvent_t>(F.hptr_event), stream));
    gather_host_kernel<double><<<std::max(1, std::min(P.nsub, 1024)), 256, 0, stream>>>(
        static_cast<const double* const*>(F.d_hptrs), F.d_Kstage_off, static_cast<double*>(F.d_Kstage), 0, P.nsub);
    FCUDA(cudaGetLastError());
  } else {
    cudaStream_t cs = static_cast<cudaStream_t>(P.copy_stream);
    // the K staging buffer is reused: the copies wait for everything enqueued on `stream` before this call
    FCUDA(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_start), stream));
    FCUDA(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(P.ev_start), 0));
    int32_t i = 0;
    while (i < P.nsub) {  // one copy per run of host-contiguous subdomains
      if (F.sub_nnzK[(size_t)i] == 0) {
        i++;
        continue;
      }
      const char* src = static_cast<const char*>(Khost[i]);
      size_t bytes = 8 * (size_t)F.sub_nnzK[(size_t)i];
      int32_t j = i + 1;
      while (j < P.nsub && F.sub_nnzK[(size_t)j] > 0 && static_cast<const char*>(Khost[j]) == src + bytes) {
        bytes += 8 * (size_t)F.sub_nnzK[(size_t)j];
        j++;
      }
      FCUDA(cudaMemcpyAsync(static_cast<char*>(F.d_Kstage) + 8 * F.Kstage_off[(size_t)i], src, bytes,
                            cudaMemcpyHostToDevice, cs));
      i = j;
    }
    if (P.ev_chunk.empty()) {
      cudaEvent_t e;
      FCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      P.ev_chunk.push_back(e);
    }
    cudaEvent_t ec = static_cast<cudaEvent_t>(P.ev_chunk[0]);
    FCUDA(cudaEventRecord(ec, cs));
    FCUDA(cudaStreamWaitEvent(stream, ec, 0));
  }
  FTRY(factor_range(P, 0, F.task_chunk[0], 0, stream, err));
  return assemble_range(P, 0, P.nsub, stream_v, err);
}

}  // namespace sc
