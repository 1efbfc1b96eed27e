// pcpg.cu — the solution stage on the GPU: the projected conjugate gradient loop
// that drives sc_apply (+ the caller's all-reduce over ranks) for the FETI dual problem
//
//     [ F    -G ] [ lambda ]   [  d ]
//     [ -G^T  O ] [ alpha  ] = [ -e ]          PAPER.md P:250-254, eq. tfetidualproblem
//
// "solved, e.g., by the preconditioned conjugate projected gradient method (PCPG) ... In each
// iteration, the operator F is applied".  Here with the identity preconditioner (projected
// CG): lambda_0 = G (G^T G)^{-1} e, P = I - G (G^T G)^{-1} G^T, r = d - F lambda, w = P r, and the CG
// recurrences on w; alpha = (G^T G)^{-1} G^T (F lambda - d) at the end.  G = B R is applied per
// subdomain from B~_i R_i (m_i x k_i, supplied by the caller), (G^T G)^{-1} as a dense matrix.
//
// Every vector operation is a kernel of this file: deterministic dot products (fixed-order block
// partials + fixed-order final sum), axpy, G^T x per subdomain, G y per global multiplier in the
// fixed (subdomain, multiplier) order of the plan's CSR, (G^T G)^{-1} b as a warp-per-row GEMV.
// Dual vectors are replicated on every rank; only the partial results of F p, G^T x and G y are
// summed over ranks through the caller's all-reduce callback (NCCL via torch.distributed).
#include <cuda_runtime.h>

#include <cmath>
#include <vector>

#include "sc_internal.h"

namespace sc {

#define PC_TRY(expr)                                                          \
  do {                                                                        \
    cudaError_t e_ = (expr);                                                  \
    if (e_ != cudaSuccess) {                                                  \
      err = std::string(#expr) + ": " + cudaGetErrorString(e_);               \
      return e_ == cudaErrorMemoryAllocation ? SC_ERR_OOM : SC_ERR_CUDA;      \
    }                                                                         \
  } while (0)

namespace {

constexpr int kDotBlocks = 296;  // 2 x 148 SMs, fixed so the summation order never changes
constexpr int kVT = 256;

__global__ void __launch_bounds__(kVT) dot_partial_kernel(const double* __restrict__ x, const double* __restrict__ y,
                                                          int64_t n, double* __restrict__ part) {
  __shared__ double red[kVT / 32];
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVT + threadIdx.x; i < n; i += (int64_t)gridDim.x * kVT) s = fma(x[i], y[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < kVT / 32; w++) t += red[w];
    part[blockIdx.x] = t;
  }
}

__global__ void dot_final_kernel(const double* __restrict__ part, int nb, double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    double t = 0.0;
    for (int b = 0; b < nb; b++) t += part[b];
    *out = t;
  }
}

// y += a x
__global__ void axpy_kernel(double* __restrict__ y, const double* __restrict__ x, double a, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * kVT + threadIdx.x;
  if (i < n) y[i] = fma(a, x[i], y[i]);
}
// p = w + b p
__global__ void xpby_kernel(double* __restrict__ p, const double* __restrict__ w, double b, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * kVT + threadIdx.x;
  if (i < n) p[i] = fma(b, p[i], w[i]);
}
// z = x - y
__global__ void sub_kernel(double* __restrict__ z, const double* __restrict__ x, const double* __restrict__ y, int64_t n) {
  const int64_t i = (int64_t)blockIdx.x * kVT + threadIdx.x;
  if (i < n) z[i] = x[i] - y[i];
}

// out[coff_i + k] = sum_a (B~_i R_i)[a, k] x[lambda_map_i(a)]   (one CTA per subdomain of this plan)
__global__ void __launch_bounds__(kVT) gt_kernel(DevPlan P, const double* __restrict__ x,
                                                 const double* const* __restrict__ Rt, const int32_t* __restrict__ ck,
                                                 const int64_t* __restrict__ coff, double* __restrict__ out) {
  __shared__ double red[kVT / 32];
  const int sub = blockIdx.x;
  const int m = P.sub_m[sub], k_i = ck[sub];
  const int64_t* __restrict__ slm = P.slm + P.sub_slm_off[sub];
  const int32_t* __restrict__ sig = P.ssig + P.sub_slm_off[sub];
  const double* __restrict__ R = Rt[sub];
  for (int k = 0; k < k_i; k++) {
    double s = 0.0;
    for (int a = threadIdx.x; a < m; a += kVT) s = fma(R[(int64_t)k * m + sig[a]], x[slm[a]], s);  // stepped a
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
      double t = 0.0;
      for (int w = 0; w < kVT / 32; w++) t += red[w];
      out[coff[sub] + k] = t;
    }
    __syncthreads();
  }
}

// out[g] = sum over (sub, a) with lambda_map_sub(a) = g, in the plan's fixed CSR order, of
//          sum_k (B~_sub R_sub)[a, k] y[coff_sub + k]
__global__ void __launch_bounds__(kVT) gy_kernel(DevPlan P, const double* const* __restrict__ Rt,
                                                 const int32_t* __restrict__ ck, const int64_t* __restrict__ coff,
                                                 const double* __restrict__ y, double* __restrict__ out, int64_t nl) {
  const int64_t gidx = (int64_t)blockIdx.x * kVT + threadIdx.x;
  if (gidx >= nl) return;
  double s = 0.0;
  for (int64_t p = P.qg_ptr[gidx]; p < P.qg_ptr[gidx + 1]; p++) {
    const int64_t sa = P.qg_sub_a[p];
    const int sub = (int)(sa >> 32), a = (int)(sa & 0xffffffff);
    const int m = P.sub_m[sub];
    const int ao = P.ssig[P.sub_slm_off[sub] + a];
    const double* R = Rt[sub];
    for (int k = 0; k < ck[sub]; k++) s = fma(R[(int64_t)k * m + ao], y[coff[sub] + k], s);
  }
  out[gidx] = s;
}

// y = A b (A dense nc x nc, column-major, symmetric): one warp per output row, fixed-order sums
__global__ void __launch_bounds__(kVT) gemv_kernel(const double* __restrict__ A, int nc, const double* __restrict__ b,
                                                   double* __restrict__ y) {
  const int row = blockIdx.x * (kVT / 32) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (row >= nc) return;
  double s = 0.0;
  for (int c = lane; c < nc; c += 32) s = fma(A[(int64_t)row * nc + c], b[c], s);  // symmetric: row of A = column
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) y[row] = s;
}

inline unsigned nblk(int64_t n) { return (unsigned)((n + kVT - 1) / kVT); }

}  // namespace

sc_status pcpg_solve(Plan& P, const double* d, const double* e_host, double* lambda, const sc_coarse* cs,
                     const sc_pcpg_opts& o, sc_allreduce_fn allreduce, void* ctx, sc_pcpg_result* res, void* stream_v,
                     std::string& err) {
  cudaStream_t st = static_cast<cudaStream_t>(stream_v);
  PC_TRY(cudaSetDevice(P.opt.device));
  const int64_t n = P.n_lambda;
  const int nc = cs ? cs->nc : 0;
  std::vector<void*> allocs;
  auto dalloc = [&](size_t bytes) -> double* {
    void* ptr = nullptr;
    if (cudaMalloc(&ptr, std::max<size_t>(bytes, 16)) != cudaSuccess) return nullptr;
    allocs.push_back(ptr);
    return static_cast<double*>(ptr);
  };
  struct Free {
    std::vector<void*>& a;
    ~Free() {
      for (void* p : a) cudaFree(p);
    }
  } guard{allocs};
  double* r = dalloc(8 * n);
  double* w = dalloc(8 * n);
  double* p = dalloc(8 * n);
  double* q = dalloc(8 * n);
  double* t = dalloc(8 * n);
  double* part = dalloc(8 * kDotBlocks);
  double* sc = dalloc(8 * 4);
  double* cv = dalloc(8 * (size_t)std::max(nc, 1));
  double* cy = dalloc(8 * (size_t)std::max(nc, 1));
  const double** dRt = nullptr;
  int32_t* dck = nullptr;
  int64_t* dcoff = nullptr;
  if (!r || !w || !p || !q || !t || !part || !sc || !cv || !cy) {
    err = "pcpg: device allocation failed";
    return SC_ERR_OOM;
  }
  if (nc > 0) {
    void *a1, *a2, *a3;
    PC_TRY(cudaMalloc(&a1, sizeof(double*) * (size_t)std::max(P.nsub, 1)));
    allocs.push_back(a1);
    PC_TRY(cudaMalloc(&a2, sizeof(int32_t) * (size_t)std::max(P.nsub, 1)));
    allocs.push_back(a2);
    PC_TRY(cudaMalloc(&a3, sizeof(int64_t) * (size_t)std::max(P.nsub, 1)));
    allocs.push_back(a3);
    dRt = static_cast<const double**>(a1);
    dck = static_cast<int32_t*>(a2);
    dcoff = static_cast<int64_t*>(a3);
    PC_TRY(cudaMemcpyAsync(a1, cs->Rt, sizeof(double*) * (size_t)P.nsub, cudaMemcpyHostToDevice, st));
    PC_TRY(cudaMemcpyAsync(a2, cs->k, sizeof(int32_t) * (size_t)P.nsub, cudaMemcpyHostToDevice, st));
    PC_TRY(cudaMemcpyAsync(a3, cs->off, sizeof(int64_t) * (size_t)P.nsub, cudaMemcpyHostToDevice, st));
  }
  auto reduce = [&](double* buf, int64_t len) -> sc_status {
    if (!allreduce || len == 0) return SC_OK;
    PC_TRY(cudaStreamSynchronize(st));
    allreduce(buf, len, ctx);
    return SC_OK;
  };
  auto dot = [&](const double* x, const double* y, double* out_host) -> sc_status {
    dot_partial_kernel<<<kDotBlocks, kVT, 0, st>>>(x, y, n, part);
    dot_final_kernel<<<1, 32, 0, st>>>(part, kDotBlocks, sc);
    PC_TRY(cudaGetLastError());
    PC_TRY(cudaMemcpyAsync(out_host, sc, sizeof(double), cudaMemcpyDeviceToHost, st));
    PC_TRY(cudaStreamSynchronize(st));
    return SC_OK;
  };
  auto applyF = [&](const double* x, double* y) -> sc_status {  // y = F x (all ranks)
    sc_status s2 = launch_apply(P, x, y, st, err);
    if (s2 != SC_OK) return s2;
    return reduce(y, n);
  };
  // y_dual = G (G^T G)^{-1} b_coarse  (b_coarse in cv, already summed over ranks)
  auto coarse_back = [&](double* out) -> sc_status {
    gemv_kernel<<<(nc + kVT / 32 - 1) / (kVT / 32), kVT, 0, st>>>(cs->GtG_inv, nc, cv, cy);
    gy_kernel<<<nblk(n), kVT, 0, st>>>(P.dev, dRt, dck, dcoff, cy, out, n);
    PC_TRY(cudaGetLastError());
    return reduce(out, n);
  };
  // out = P x = x - G (G^T G)^{-1} G^T x
  auto project = [&](const double* x, double* out) -> sc_status {
    if (nc == 0) {
      PC_TRY(cudaMemcpyAsync(out, x, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
      return SC_OK;
    }
    PC_TRY(cudaMemsetAsync(cv, 0, 8 * (size_t)nc, st));
    if (P.nsub > 0) gt_kernel<<<P.nsub, kVT, 0, st>>>(P.dev, x, dRt, dck, dcoff, cv);
    PC_TRY(cudaGetLastError());
    sc_status s2 = reduce(cv, nc);
    if (s2 != SC_OK) return s2;
    s2 = coarse_back(t);
    if (s2 != SC_OK) return s2;
    sub_kernel<<<nblk(n), kVT, 0, st>>>(out, x, t, n);
    PC_TRY(cudaGetLastError());
    return SC_OK;
  };
#define PC_STEP(x)               \
  do {                           \
    sc_status s_ = (x);          \
    if (s_ != SC_OK) return s_;  \
  } while (0)
  // lambda_0 = G (G^T G)^{-1} e   (or the caller's lambda when there is no coarse space)
  if (nc > 0) {
    PC_TRY(cudaMemcpyAsync(cv, e_host, 8 * (size_t)nc, cudaMemcpyHostToDevice, st));
    PC_STEP(coarse_back(lambda));
  }
  // r = d - F lambda, w = P r, p = w
  PC_STEP(applyF(lambda, q));
  sub_kernel<<<nblk(n), kVT, 0, st>>>(r, d, q, n);
  PC_STEP(project(r, w));
  PC_TRY(cudaMemcpyAsync(p, w, 8 * (size_t)n, cudaMemcpyDeviceToDevice, st));
  double ww = 0.0, pd = 0.0;
  PC_STEP(dot(w, w, &ww));
  PC_STEP(project(d, t));  // reference norm ||P d||
  PC_STEP(dot(t, t, &pd));
  const double ref = std::sqrt(pd) > 0 ? std::sqrt(pd) : 1.0;
  int it = 0;
  double rel = std::sqrt(ww) / ref;
  if (res && res->history && res->history_len > 0) res->history[0] = rel;
  while (rel > o.rtol && it < o.max_it) {
    PC_STEP(applyF(p, q));
    double pq = 0.0;
    PC_STEP(dot(p, q, &pq));
    if (!(pq > 0.0)) break;  // F is SPD on ker(G^T); a non-positive curvature means breakdown
    const double a = ww / pq;
    axpy_kernel<<<nblk(n), kVT, 0, st>>>(lambda, p, a, n);
    axpy_kernel<<<nblk(n), kVT, 0, st>>>(r, q, -a, n);
    PC_STEP(project(r, w));
    double ww2 = 0.0;
    PC_STEP(dot(w, w, &ww2));
    xpby_kernel<<<nblk(n), kVT, 0, st>>>(p, w, ww2 / ww, n);
    PC_TRY(cudaGetLastError());
    ww = ww2;
    it++;
    rel = std::sqrt(ww) / ref;
    if (res && res->history && it < res->history_len) res->history[it] = rel;
  }
  // alpha = (G^T G)^{-1} G^T (F lambda - d) = -(G^T G)^{-1} G^T r   (r = d - F lambda, recomputed)
  if (nc > 0 && o.alpha) {
    PC_STEP(applyF(lambda, q));
    sub_kernel<<<nblk(n), kVT, 0, st>>>(r, q, d, n);  // F lambda - d
    PC_TRY(cudaMemsetAsync(cv, 0, 8 * (size_t)nc, st));
    if (P.nsub > 0) gt_kernel<<<P.nsub, kVT, 0, st>>>(P.dev, r, dRt, dck, dcoff, cv);
    PC_STEP(reduce(cv, nc));
    gemv_kernel<<<(nc + kVT / 32 - 1) / (kVT / 32), kVT, 0, st>>>(cs->GtG_inv, nc, cv, o.alpha);
    PC_TRY(cudaGetLastError());
  }
  PC_TRY(cudaStreamSynchronize(st));
  if (res) {
    res->iterations = it;
    res->rel_residual = rel;
  }
  P.last_stream = stream_v;
  return SC_OK;
#undef PC_STEP
}

}  // namespace sc
