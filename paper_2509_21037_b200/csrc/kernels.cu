// kernels.cu — the device hot path (sm_100a, FP64).
//
//   trsm_tile_kernel<T>  "X init + stepped supernodal TRSM" (SURVEY §8 rows a2+a3): one CTA per
//                        (subdomain, RHS column tile).  Zeroes the tile's X strip, scatters the
//                        permuted B~^T, then walks the factor panels of the tile's reach
//                        in order: diagonal-block forward substitution (warp-per-column with shuffle
//                        broadcasts), then the pruned sub-diagonal update X[R] -= L[R,panel] X[panel]
//                        as an FP64 DMMA (mma.sync m8n8k4) gather-GEMM-scatter.
//   syrk_pair_kernel<T>  "block-sparse SYRK" (row a4): one CTA per output tile (I >= J) of F'
//                        = X^T X, k restricted to rows both strips hold, DMMA tiles.
//   apply_*              "explicit apply" (row a6): batched symmetric mat-vec on the lower F'
//                        with the stepped-order gather of lambda and a deterministic scatter-sum.
#include <cuda_runtime.h>

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

// Shared-memory strides (in doubles) chosen == 4 (mod 16) so the fragment loads
// (4 consecutive k rows x 8 consecutive columns) hit 16 distinct 8-byte bank pairs per phase.
constexpr int kLdL = kChunk + 4;   // L chunk / triangle, column-major [col][row]

template <int T>
struct TileCfg {
  static constexpr int LDX = T + 4;            // X rows, row-major [row][col]
  static constexpr int NB = T / 8;             // 8-wide column blocks in a tile
  // update GEMM C(64 x T): warps as (8/NWC) x NWC, each WM x WN blocks of 8x8
  static constexpr int WN = (T == 64) ? 4 : 2;
  static constexpr int NWC = NB / WN;
  static constexpr int WM = 8 / (8 / NWC);     // block rows per warp so that all 8 rows covered
};

template <int T>
__global__ void __launch_bounds__(kThreads) trsm_tile_kernel(DevPlan P) {
  using Cfg = TileCfg<T>;
  constexpr int LDX = Cfg::LDX;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  double* Xs = reinterpret_cast<double*>(smem_raw);                 // [kMaxPanel][LDX]
  double* Ls = Xs + kMaxPanel * LDX;                                // [kMaxPanel][kLdL] triangle
  double* Lc = Ls + kMaxPanel * kLdL;                               // [kMaxPanel][kLdL] chunk
  int64_t* colS = reinterpret_cast<int64_t*>(Lc + kMaxPanel * kLdL);  // [kMaxPanel]
  int32_t* rowsS = reinterpret_cast<int32_t*>(colS + kMaxPanel);      // [kChunk]
  uint16_t* map = reinterpret_cast<uint16_t*>(rowsS + kChunk);        // [max_n]

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const I2 task = P.trsm_tasks[blockIdx.x];
  const int sub = task.x;
  const Tile tile = P.tiles[task.y];
  const int cls = P.sub_cls[sub];
  const int64_t* __restrict__ colptr = P.colptr + P.cls_colptr_off[cls];
  const double* __restrict__ Lv = P.Lptr[sub];
  double* __restrict__ X = P.X + P.sub_X_base[sub] + tile.x_off;

  // ---- X init (row a2): zero the strip, build the row map, scatter B~^T
  {
    const int64_t nvec = (int64_t)tile.strip_rows * T / 2;
    double2* X2 = reinterpret_cast<double2*>(X);
    for (int64_t q = tid; q < nvec; q += kThreads) X2[q] = make_double2(0.0, 0.0);
    for (int q = tile.reach_begin + warp; q < tile.reach_end; q += kThreads / 32) {
      const Reach R = P.reach[q];
      for (int r = R.e + lane; r < R.c1; r += 32) map[r] = (uint16_t)(R.off + (r - R.e));
    }
  }
  __syncthreads();
  for (int q = tile.binit_begin + tid; q < tile.binit_end; q += kThreads) {
    const BInit b = P.binit[q];
    X[(int64_t)b.strip_row * T + b.col] = b.val;
  }
  __syncthreads();

  // ---- stepped supernodal TRSM (row a3)
  for (int st = tile.step_begin; st < tile.step_end; st++) {
    const Step S = P.steps[st];
    const int kw = S.kw, e = S.e;
    const int kw4 = (kw + 3) & ~3;
    if (tid < kw) colS[tid] = colptr[e + tid];
    __syncthreads();
    // panel triangle L[e:e+kw, e:e+kw] -> Ls (column-major, zero outside the lower triangle)
    for (int q = tid; q < kMaxPanel * kMaxPanel; q += kThreads) {
      const int c = q >> 6, r = q & 63;
      double v = 0.0;
      if (c < kw && r < kw && r >= c) v = Lv[colS[c] + (r - c)];
      Ls[c * kLdL + r] = v;
    }
    // panel rows of X -> Xs (rows kw..kw4 zero for the k padding of the update GEMM)
    for (int q = tid; q < kw4 * T; q += kThreads) {
      const int r = q / T, j = q - r * T;
      Xs[r * LDX + j] = (r < kw) ? X[(int64_t)(S.strip_row + r) * T + j] : 0.0;
    }
    __syncthreads();
    // diagonal block: forward substitution, warp w owns columns j = w + 8q, lanes own rows
    {
      constexpr int CPW = T / 8;
      double x0[CPW], x1[CPW];
#pragma unroll
      for (int q = 0; q < CPW; q++) {
        const int j = warp + 8 * q;
        x0[q] = (lane < kw) ? Xs[lane * LDX + j] : 0.0;
        x1[q] = (lane + 32 < kw) ? Xs[(lane + 32) * LDX + j] : 0.0;
      }
      for (int c = 0; c < kw; c++) {
        const double d = Ls[c * kLdL + c];
        if (!(d > 0.0) || !isfinite(d)) {
          if (tid == 0 && warp == 0)
            atomicCAS(P.err, 0ull, ((unsigned long long)(sub + 1) << 32) | (unsigned long long)(e + c));
        }
        const double rcp = 1.0 / d;
        const double l0 = (lane > c) ? Ls[c * kLdL + lane] : 0.0;
        const double l1 = (lane + 32 > c) ? Ls[c * kLdL + lane + 32] : 0.0;
#pragma unroll
        for (int q = 0; q < CPW; q++) {
          const double xc = __shfl_sync(0xffffffffu, (c < 32) ? x0[q] : x1[q], c & 31) * rcp;
          if (c < 32) {
            if (lane == c) x0[q] = xc;
          } else {
            if (lane == c - 32) x1[q] = xc;
          }
          x0[q] = fma(-l0, xc, x0[q]);
          x1[q] = fma(-l1, xc, x1[q]);
        }
      }
#pragma unroll
      for (int q = 0; q < CPW; q++) {
        const int j = warp + 8 * q;
        if (lane < kw) Xs[lane * LDX + j] = x0[q];
        if (lane + 32 < kw) Xs[(lane + 32) * LDX + j] = x1[q];
      }
    }
    __syncthreads();
    // solved panel rows are final: store them
    for (int q = tid; q < kw * T; q += kThreads) {
      const int r = q / T, j = q - r * T;
      X[(int64_t)(S.strip_row + r) * T + j] = Xs[r * LDX + j];
    }
    // pruned sub-diagonal update, chunks of 64 rows: rows [e+kw, c1) of the supernode, then R_s
    const int nin = S.c1 - e - kw;
    const int M = nin + S.nR;
    for (int m0 = 0; m0 < M; m0 += kChunk) {
      if (tid < kChunk) {
        const int k = m0 + tid;
        int row = -1;
        if (k < M) row = (k < nin) ? (S.strip_row + kw + k) : (int)map[P.Rrows[S.R_off + (k - nin)]];
        rowsS[tid] = row;
      }
      for (int q = tid; q < kw4 * kChunk; q += kThreads) {
        const int c = q >> 6, k = q & 63;
        double v = 0.0;
        if (c < kw && m0 + k < M) v = Lv[colS[c] + (kw - c) + m0 + k];
        Lc[c * kLdL + k] = v;
      }
      __syncthreads();
      {
        constexpr int WM = Cfg::WM, WN = Cfg::WN, NWC = Cfg::NWC;
        const int br0 = (warp / NWC) * WM, bc0 = (warp % NWC) * WN;
        double acc[WM][WN][2];
#pragma unroll
        for (int i = 0; i < WM; i++)
#pragma unroll
          for (int j = 0; j < WN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;
        for (int k = 0; k < kw4; k += 4) {
          double a[WM], b[WN];
#pragma unroll
          for (int i = 0; i < WM; i++) a[i] = Lc[(k + t4) * kLdL + (br0 + i) * 8 + g];
#pragma unroll
          for (int j = 0; j < WN; j++) b[j] = Xs[(k + t4) * LDX + (bc0 + j) * 8 + g];
#pragma unroll
          for (int i = 0; i < WM; i++)
#pragma unroll
            for (int j = 0; j < WN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
#pragma unroll
        for (int i = 0; i < WM; i++) {
          const int row = rowsS[(br0 + i) * 8 + g];
          if (row < 0) continue;
#pragma unroll
          for (int j = 0; j < WN; j++) {
            double2* p = reinterpret_cast<double2*>(X + (int64_t)row * T + (bc0 + j) * 8 + 2 * t4);
            double2 v = *p;
            v.x -= acc[i][j][0];
            v.y -= acc[i][j][1];
            *p = v;
          }
        }
      }
      __syncthreads();
    }
  }
}

// ------------------------------------------------------------------------------------------------
// SYRK: F'[I,J] = sum_seg X_I[seg]^T X_J[seg]  (T x T output tile, lower part of F' only)
// ------------------------------------------------------------------------------------------------
template <int T>
struct SyrkCfg {
  static constexpr int LDX = T + 4;
  static constexpr int NB = T / 8;                       // block rows/cols of the output tile
  static constexpr int NBLK = NB * NB;                   // 8x8 output blocks
  static constexpr int PER_WARP = (NBLK + 7) / 8;        // blocks per warp (T=16: 1 with 4 idle warps)
  static constexpr int WN = (T == 64) ? 4 : (T == 32 ? 2 : 1);
  static constexpr int WM = PER_WARP / WN;
  static constexpr int NWC = NB / WN;
};
constexpr int kKC = 32;  // k rows staged per chunk

template <int T>
__global__ void __launch_bounds__(kThreads) syrk_pair_kernel(DevPlan P) {
  using Cfg = SyrkCfg<T>;
  constexpr int LDX = Cfg::LDX;
  __shared__ __align__(16) double As[kKC * LDX];
  __shared__ __align__(16) double Bs[kKC * LDX];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const I2 task = P.syrk_tasks[blockIdx.x];
  const int sub = task.x;
  const Pair pr = P.pairs[task.y];
  const Tile tI = P.tiles[pr.I], tJ = P.tiles[pr.J];
  const double* __restrict__ XI = P.X + P.sub_X_base[sub] + tI.x_off;
  const double* __restrict__ XJ = P.X + P.sub_X_base[sub] + tJ.x_off;
  constexpr int WM = Cfg::WM, WN = Cfg::WN, NWC = Cfg::NWC;
  const bool active = warp < (Cfg::NB / WM) * NWC;
  const int br0 = (warp / NWC) * WM, bc0 = (warp % NWC) * WN;
  double acc[WM][WN][2];
#pragma unroll
  for (int i = 0; i < WM; i++)
#pragma unroll
    for (int j = 0; j < WN; j++) acc[i][j][0] = acc[i][j][1] = 0.0;

  for (int sg = pr.seg_begin; sg < pr.seg_end; sg++) {
    const Seg s = P.segs[sg];
    for (int k0 = 0; k0 < s.len; k0 += kKC) {
      const int kn = min(kKC, s.len - k0);
      for (int q = tid; q < kKC * T; q += kThreads) {
        const int r = q / T, j = q - r * T;
        As[r * LDX + j] = (r < kn) ? XI[(int64_t)(s.offI + k0 + r) * T + j] : 0.0;
        Bs[r * LDX + j] = (r < kn) ? XJ[(int64_t)(s.offJ + k0 + r) * T + j] : 0.0;
      }
      __syncthreads();
      if (active) {
        const int kn4 = (kn + 3) & ~3;
        for (int k = 0; k < kn4; k += 4) {
          double a[WM], b[WN];
#pragma unroll
          for (int i = 0; i < WM; i++) a[i] = As[(k + t4) * LDX + (br0 + i) * 8 + g];
#pragma unroll
          for (int j = 0; j < WN; j++) b[j] = Bs[(k + t4) * LDX + (bc0 + j) * 8 + g];
#pragma unroll
          for (int i = 0; i < WM; i++)
#pragma unroll
            for (int j = 0; j < WN; j++) dmma(acc[i][j][0], acc[i][j][1], a[i], b[j]);
        }
      }
      __syncthreads();
    }
  }
  if (!active) return;
  const int m = P.sub_m[sub];
  double* __restrict__ F = P.F + P.sub_F_base[sub];
  const bool diag = (pr.I == pr.J);
#pragma unroll
  for (int i = 0; i < WM; i++) {
    const int r = (br0 + i) * 8 + g;  // row within tile I
    if (r >= tI.width) continue;
#pragma unroll
    for (int j = 0; j < WN; j++) {
#pragma unroll
      for (int h = 0; h < 2; h++) {
        const int c = (bc0 + j) * 8 + 2 * t4 + h;  // column within tile J
        if (c >= tJ.width || (diag && r < c)) continue;
        F[(int64_t)(tJ.col0 + c) * m + (tI.col0 + r)] = acc[i][j][h];
      }
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Apply: y_i = F'_i x_i (x_i(a) = lambda[slm_i(a)]) from the lower triangle; deterministic sum.
// ------------------------------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads) apply_partial_kernel(DevPlan P, const double* __restrict__ lambda) {
  __shared__ double xs[32];
  __shared__ double zred[kThreads / 32][32];
  const ApplyTask task = P.apply_tasks[blockIdx.x];
  const int sub = task.sub, b0 = task.b0;
  const int m = P.sub_m[sub];
  const int nb = min(32, m - b0);
  const double* __restrict__ F = P.F + P.sub_F_base[sub];
  const int64_t* slm = P.slm + P.sub_slm_off[sub];
  double* part = P.part + P.sub_part_off[sub] + (int64_t)(b0 / 32) * m;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid < 32) xs[tid] = (tid < nb) ? lambda[slm[b0 + tid]] : 0.0;
  __syncthreads();
  double z[32];
#pragma unroll
  for (int j = 0; j < 32; j++) z[j] = 0.0;
  for (int a = b0 + tid; a < m; a += kThreads) {
    const double xa = lambda[slm[a]];
    double w = 0.0;
#pragma unroll
    for (int j = 0; j < 32; j++) {
      if (j < nb) {
        const int b = b0 + j;
        if (a >= b) {
          const double f = F[(int64_t)b * m + a];
          z[j] = fma(f, xa, z[j]);        // column dot: (F' x) contribution to row b
          if (a > b) w = fma(f, xs[j], w);  // row a contribution from column b
        }
      }
    }
    part[a] = w;
  }
#pragma unroll
  for (int j = 0; j < 32; j++) {
    double v = z[j];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) zred[warp][j] = v;
  }
  __syncthreads();
  if (tid < nb) {
    double v = 0.0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; w++) v += zred[w][tid];
    part[b0 + tid] += v;
  }
}

__global__ void __launch_bounds__(kThreads) apply_scatter_kernel(DevPlan P, double* __restrict__ q, int64_t nl) {
  const int64_t gidx = (int64_t)blockIdx.x * kThreads + threadIdx.x;
  if (gidx >= nl) return;
  double s = 0.0;
  for (int64_t p = P.qg_ptr[gidx]; p < P.qg_ptr[gidx + 1]; p++) {
    const int64_t sa = P.qg_sub_a[p];
    const int sub = (int)(sa >> 32), a = (int)(sa & 0xffffffff);
    const int m = P.sub_m[sub];
    const double* part = P.part + P.sub_part_off[sub];
    for (int blk = 0; blk <= a / 32; blk++) s += part[(int64_t)blk * m + a];
  }
  q[gidx] = s;
}

// ------------------------------------------------------------------------------------------------
// host side
// ------------------------------------------------------------------------------------------------
namespace {

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

size_t trsm_smem_bytes(int T, int max_n) {
  size_t b = sizeof(double) * (size_t)(kMaxPanel * (T + 4) + 2 * kMaxPanel * kLdL);
  b += sizeof(int64_t) * kMaxPanel + sizeof(int32_t) * kChunk;
  b += sizeof(uint16_t) * (size_t)std::max(max_n, 1);
  return (b + 15) & ~(size_t)15;
}

#define TRY(x)                   \
  do {                           \
    sc_status s_ = (x);          \
    if (s_ != SC_OK) return s_;  \
  } while (0)

}  // namespace

sc_status upload_plan(Plan& P, std::string& err) {
  CUDA_TRY(cudaSetDevice(P.opt.device));
  DevPlan& D = P.dev;
  std::memset(&D, 0, sizeof(D));
  // concatenate class data
  std::vector<int64_t> colptr, cls_off;
  std::vector<int32_t> Rrows;
  std::vector<Tile> tiles;
  std::vector<Step> steps;
  std::vector<Reach> reach;
  std::vector<BInit> binit;
  std::vector<Pair> pairs;
  std::vector<Seg> segs;
  for (auto& C : P.classes) {
    cls_off.push_back((int64_t)colptr.size());
    colptr.insert(colptr.end(), C.colptr.begin(), C.colptr.end());
    Rrows.insert(Rrows.end(), C.Rrows.begin(), C.Rrows.end());
    tiles.insert(tiles.end(), C.tiles.begin(), C.tiles.end());
    steps.insert(steps.end(), C.steps.begin(), C.steps.end());
    reach.insert(reach.end(), C.reach.begin(), C.reach.end());
    binit.insert(binit.end(), C.binit.begin(), C.binit.end());
    pairs.insert(pairs.end(), C.pairs.begin(), C.pairs.end());
    segs.insert(segs.end(), C.segs.begin(), C.segs.end());
  }
  TRY(upload(P, colptr, &D.colptr, err));
  TRY(upload(P, cls_off, &D.cls_colptr_off, err));
  TRY(upload(P, Rrows, &D.Rrows, err));
  TRY(upload(P, tiles, &D.tiles, err));
  TRY(upload(P, steps, &D.steps, err));
  TRY(upload(P, reach, &D.reach, err));
  TRY(upload(P, binit, &D.binit, err));
  TRY(upload(P, pairs, &D.pairs, err));
  TRY(upload(P, segs, &D.segs, err));
  TRY(upload(P, P.sub_cls, &D.sub_cls, err));
  TRY(upload(P, P.sub_X_base, &D.sub_X_base, err));
  TRY(upload(P, P.sub_F_base, &D.sub_F_base, err));
  TRY(upload(P, P.sub_m, &D.sub_m, err));
  TRY(upload(P, P.trsm_tasks, &D.trsm_tasks, err));
  TRY(upload(P, P.syrk_tasks, &D.syrk_tasks, err));
  TRY(upload(P, P.apply_tasks, &D.apply_tasks, err));
  TRY(upload(P, P.sub_slm_off, &D.sub_slm_off, err));
  TRY(upload(P, P.slm, &D.slm, err));
  TRY(upload(P, P.sub_part_off, &D.sub_part_off, err));
  TRY(upload(P, P.qg_ptr, &D.qg_ptr, err));
  TRY(upload(P, P.qg_sub_a, &D.qg_sub_a, err));
  TRY(alloc_zero(P, P.X_doubles, &D.X, err));
  TRY(alloc_zero(P, P.F_doubles, &D.F, err));
  TRY(alloc_zero(P, P.part_doubles, &D.part, err));
  TRY(alloc_zero(P, 1, &D.err, err));
  double** dl = nullptr;
  TRY(alloc_zero(P, std::max(P.nsub, 1), &dl, err));
  P.d_Lptr = dl;
  D.Lptr = dl;
  void* hp = nullptr;
  CUDA_TRY(cudaMallocHost(&hp, sizeof(double*) * (size_t)std::max(P.nsub, 1)));
  P.h_Lptr_pinned = static_cast<const double**>(hp);
  cudaEvent_t ev;
  CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  P.lptr_event = ev;
  D.nsub = P.nsub;
  D.max_n = P.max_n;
  P.smem_trsm = trsm_smem_bytes(P.T, P.max_n);
  if (P.smem_trsm > 227 * 1024) {
    err = "TRSM shared memory exceeds 227 KB";
    return SC_ERR_INVALID_ARG;
  }
  switch (P.T) {
    case 16: CUDA_TRY(cudaFuncSetAttribute(trsm_tile_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_trsm)); break;
    case 32: CUDA_TRY(cudaFuncSetAttribute(trsm_tile_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_trsm)); break;
    default: CUDA_TRY(cudaFuncSetAttribute(trsm_tile_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.smem_trsm)); break;
  }
  double total = 0;
  total += 8.0 * (P.X_doubles + P.F_doubles + P.part_doubles);
  total += colptr.size() * 8.0 + Rrows.size() * 4.0 + tiles.size() * sizeof(Tile) + steps.size() * sizeof(Step) +
           reach.size() * sizeof(Reach) + binit.size() * sizeof(BInit) + pairs.size() * sizeof(Pair) +
           segs.size() * sizeof(Seg) + P.slm.size() * 8.0 + P.qg_sub_a.size() * 8.0 + P.qg_ptr.size() * 8.0;
  P.stats.device_bytes = total;
  P.on_device = true;
  return SC_OK;
}

void free_plan_device(Plan& P) {
  if (!P.on_device) return;
  cudaSetDevice(P.opt.device);
  cudaDeviceSynchronize();
  for (void* p : P.allocations) cudaFree(p);
  P.allocations.clear();
  if (P.h_Lptr_pinned) cudaFreeHost((void*)P.h_Lptr_pinned);
  P.h_Lptr_pinned = nullptr;
  if (P.lptr_event) cudaEventDestroy((cudaEvent_t)P.lptr_event);
  P.lptr_event = nullptr;
  if (P.d_Lstage) cudaFree(P.d_Lstage);
  P.d_Lstage = nullptr;
  P.on_device = false;
}

sc_status launch_assemble(Plan& P, const double* const* Lptr_host, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  bool same = (int32_t)P.last_Lptr.size() == P.nsub;
  for (int32_t i = 0; same && i < P.nsub; i++) same = (P.last_Lptr[(size_t)i] == Lptr_host[i]);
  if (!same) {
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
  }
  P.last_stream = stream_v;
  const int ntr = (int)P.trsm_tasks.size(), nsy = (int)P.syrk_tasks.size();
  if (P.tev[0]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[0], stream));
  if (ntr > 0) {
    switch (P.T) {
      case 16: trsm_tile_kernel<16><<<ntr, kThreads, P.smem_trsm, stream>>>(P.dev); break;
      case 32: trsm_tile_kernel<32><<<ntr, kThreads, P.smem_trsm, stream>>>(P.dev); break;
      default: trsm_tile_kernel<64><<<ntr, kThreads, P.smem_trsm, stream>>>(P.dev); break;
    }
    CUDA_TRY(cudaGetLastError());
  }
  if (P.tev[1]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[1], stream));
  if (nsy > 0) {
    switch (P.T) {
      case 16: syrk_pair_kernel<16><<<nsy, kThreads, 0, stream>>>(P.dev); break;
      case 32: syrk_pair_kernel<32><<<nsy, kThreads, 0, stream>>>(P.dev); break;
      default: syrk_pair_kernel<64><<<nsy, kThreads, 0, stream>>>(P.dev); break;
    }
    CUDA_TRY(cudaGetLastError());
  }
  if (P.tev[2]) CUDA_TRY(cudaEventRecord((cudaEvent_t)P.tev[2], stream));
  return SC_OK;
}

sc_status stage_host_L(Plan& P, const double* const* Lhost, void* stream_v, std::vector<const double*>& dptrs,
                       std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  if (!P.d_Lstage) {
    P.Lstage_off.assign((size_t)P.nsub + 1, 0);
    for (int32_t i = 0; i < P.nsub; i++) P.Lstage_off[(size_t)i + 1] = P.Lstage_off[(size_t)i] + P.sub_nnz[(size_t)i];
    void* d = nullptr;
    CUDA_TRY(cudaMalloc(&d, std::max<size_t>(8 * (size_t)P.Lstage_off.back(), 16)));
    P.d_Lstage = static_cast<double*>(d);
  }
  dptrs.resize((size_t)P.nsub);
  for (int32_t i = 0; i < P.nsub; i++) {
    double* dst = P.d_Lstage + P.Lstage_off[(size_t)i];
    if (P.sub_nnz[(size_t)i] > 0) {
      if (!Lhost[i]) {
        err = "L_values_host[" + std::to_string(i) + "] is NULL";
        return SC_ERR_INVALID_ARG;
      }
      CUDA_TRY(cudaMemcpyAsync(dst, Lhost[i], 8 * (size_t)P.sub_nnz[(size_t)i], cudaMemcpyHostToDevice, stream));
    }
    dptrs[(size_t)i] = dst;
  }
  return SC_OK;
}

sc_status launch_apply(Plan& P, const double* lambda, double* q, void* stream_v, std::string& err) {
  cudaStream_t stream = static_cast<cudaStream_t>(stream_v);
  CUDA_TRY(cudaSetDevice(P.opt.device));
  P.last_stream = stream_v;
  const int na = (int)P.apply_tasks.size();
  if (na > 0) {
    apply_partial_kernel<<<na, kThreads, 0, stream>>>(P.dev, lambda);
    CUDA_TRY(cudaGetLastError());
  }
  if (P.n_lambda > 0) {
    const int64_t nb = (P.n_lambda + kThreads - 1) / kThreads;
    apply_scatter_kernel<<<(unsigned)nb, kThreads, 0, stream>>>(P.dev, q, P.n_lambda);
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

sc_status copy_F_lower(Plan& P, int32_t i, std::vector<double>& out, std::string& err) {
  TRY(device_check(P, err));
  int64_t m = P.sub_m[(size_t)i];
  out.resize((size_t)(m * m));
  if (m > 0)
    CUDA_TRY(cudaMemcpy(out.data(), P.dev.F + P.sub_F_base[(size_t)i], 8 * (size_t)(m * m), cudaMemcpyDeviceToHost));
  return SC_OK;
}

sc_status copy_X_strips(Plan& P, int32_t i, std::vector<double>& out, std::string& err) {
  TRY(device_check(P, err));
  const ClassPlan& C = P.classes[(size_t)P.sub_cls[(size_t)i]];
  out.resize((size_t)C.x_doubles);
  if (C.x_doubles > 0)
    CUDA_TRY(cudaMemcpy(out.data(), P.dev.X + P.sub_X_base[(size_t)i], 8 * (size_t)C.x_doubles, cudaMemcpyDeviceToHost));
  return SC_OK;
}

}  // namespace sc
