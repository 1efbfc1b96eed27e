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
constexpr int kSLd = kFW + 1;           // per-warp frame buffer: 32 x 33 doubles (column 32: 1 / l_jj)
constexpr int kFSmem = kFWarps * kFW * kSLd * 8;

__device__ __forceinline__ void fdmma(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c0), "+d"(c1)
               : "d"(a), "d"(b));
}
__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// index of v in the ascending R[lo, hi), or -1
__device__ __forceinline__ int find_row(const int32_t* R, int lo, int hi, int v) {
  int h = hi;
  while (lo < h) {
    const int mid = (lo + h) >> 1;
    if (__ldg(R + mid) < v) lo = mid + 1;
    else h = mid;
  }
  return (lo < hi && __ldg(R + lo) == v) ? lo : -1;
}

__global__ void __launch_bounds__(32 * kFWarps, 4) factor_kernel(DevFactor F, int64_t t0, int64_t t1, int slot) {
  extern __shared__ double fsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  double* S = fsm + warp * kFW * kSLd;
  for (;;) {
    int64_t task = 0;
    if (lane == 0) task = t0 + atomicAdd(F.queue + slot, 1);
    task = __shfl_sync(~0u, task, 0);
    if (task >= t1) break;
    const FTask tk = F.tasks[task];
    const FFrame fr = F.frames[tk.frame];
    const FPanel pn = F.panels[fr.panel];
    const int sub = tk.sub;
    int* flags = F.flags + (F.sub_flag_base[sub] - F.cls_panel0[F.sub_cls[sub]]);  // indexed by global panel
    double* W = F.W + F.sub_W_base[sub];
    const bool diag = fr.r0 < 0;
    const int kw = pn.kw, nI = (fr.nrow + 7) >> 3, nJ = pn.kw8 >> 3;
    const int rv = lane < fr.nrow ? (diag ? pn.a + lane : __ldg(F.Rrows + pn.R_off + fr.r0 + lane)) : -1;
    double acc[4][4][2];
#pragma unroll
    for (int I = 0; I < 4; I++)
#pragma unroll
      for (int J = 0; J < 4; J++) acc[I][J][0] = acc[I][J][1] = 0.0;

    // ---- updates from the finished descendant panels (left-looking)
    for (int u = pn.upd_begin; u < pn.upd_end; u++) {
      const FUpd U = F.upd[u];
      const FPanel dn = F.panels[U.d];
      if (lane == 0) {
        const int* fl = flags + U.d;
        while ((ld_acquire(fl) & 0xFFFF) < dn.nframe) __nanosleep(100);
      }
      __syncwarp();
      const int32_t* Rd = F.Rrows + dn.R_off;
      const int lo = diag ? U.s0 : U.s1, hi = diag ? U.s1 : dn.nR;
      const int ridx = (rv >= 0 && lo < hi) ? find_row(Rd, lo, hi, rv) : -1;
      const int cidx = lane < kw ? find_row(Rd, U.s0, U.s1, pn.a + lane) : -1;
      const unsigned rm = __ballot_sync(~0u, ridx >= 0), cm = __ballot_sync(~0u, cidx >= 0);
      if (!rm || !cm) continue;
      const double* Wd = W + dn.w_off;
      const int ldd = dn.nR;
      int ri[4], ci[4];
#pragma unroll
      for (int I = 0; I < 4; I++) ri[I] = __shfl_sync(~0u, ridx, 8 * I + g);
#pragma unroll
      for (int J = 0; J < 4; J++) ci[J] = __shfl_sync(~0u, cidx, 8 * J + g);
      bool ra[4], ca[4];
#pragma unroll
      for (int I = 0; I < 4; I++) ra[I] = I < nI && ((rm >> (8 * I)) & 0xFFu);
#pragma unroll
      for (int J = 0; J < 4; J++) ca[J] = J < nJ && ((cm >> (8 * J)) & 0xFFu);
      for (int k0 = 0; k0 < dn.kw; k0 += 4) {
        const int kk = k0 + t;
        const bool kv = kk < dn.kw;
        const double* col = Wd + (int64_t)kk * ldd;
        double a[4], b[4];
#pragma unroll
        for (int I = 0; I < 4; I++) a[I] = (ra[I] && kv && ri[I] >= 0) ? __ldcg(col + ri[I]) : 0.0;
#pragma unroll
        for (int J = 0; J < 4; J++) b[J] = (ca[J] && kv && ci[J] >= 0) ? __ldcg(col + ci[J]) : 0.0;
#pragma unroll
        for (int I = 0; I < 4; I++)
#pragma unroll
          for (int J = 0; J < 4; J++)
            if (ra[I] && ca[J] && (!diag || J <= I)) fdmma(acc[I][J][0], acc[I][J][1], a[I], b[J]);
      }
    }

    // ---- S = K entries - updates (frame layout, row-major in the warp's shared buffer)
    __syncwarp();
#pragma unroll
    for (int I = 0; I < 4; I++)
#pragma unroll
      for (int J = 0; J < 4; J++)
        if (I < nI && J < nJ) {
          S[(8 * I + g) * kSLd + 8 * J + 2 * t] = -acc[I][J][0];
          S[(8 * I + g) * kSLd + 8 * J + 2 * t + 1] = -acc[I][J][1];
        }
    __syncwarp();
    {
      const double* Kv = static_cast<const double*>(F.Kptr[sub]);
      for (int e = fr.k_begin + lane; e < fr.k_end; e += 32) {
        const FEnt en = F.kent[e];
        S[(en.pos >> 5) * kSLd + (en.pos & 31)] += __ldg(Kv + en.q);
      }
    }
    __syncwarp();

    if (diag) {
      // ---- Cholesky of the diagonal block (right-looking, lane = row)
      for (int j = 0; j < kw; j++) {
        double djj = S[j * kSLd + j];
        if (!(djj > 0.0) || !isfinite(djj)) {
          if (lane == 0) {
            atomicCAS(F.err, 0ull, ((unsigned long long)(sub + 1) << 32) | (unsigned long long)(pn.a + j));
            atomicCAS(F.err + 1 + sub, 0ull, (unsigned long long)(pn.a + j) + 1ull);
          }
          djj = 1.0;
        }
        const double l = sqrt(djj), rl = 1.0 / l;
        __syncwarp();
        if (lane == j) {
          S[j * kSLd + j] = l;
          S[j * kSLd + kFW] = rl;
        }
        if (lane > j && lane < kw) S[lane * kSLd + j] *= rl;
        __syncwarp();
        if (lane > j && lane < kw) {
          const double lij = S[lane * kSLd + j];
          for (int c = j + 1; c <= lane; c++) S[lane * kSLd + c] -= lij * S[c * kSLd + j];
        }
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
    } else {
      // ---- wait for the panel's own diagonal frame, then X = S inv(L_pp)^T
      if (lane == 0) {
        const int* fl = flags + fr.panel;
        while (!(ld_acquire(fl) & 0x10000)) __nanosleep(100);
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
            if (r < fr.nrow) {
              if (c < kw) Wp[(int64_t)c * pn.nR + fr.r0 + r] = acc[I][J][0];
              if (c + 1 < kw) Wp[(int64_t)(c + 1) * pn.nR + fr.r0 + r] = acc[I][J][1];
            }
          }
    }
    __syncwarp();
    // ---- L values of this frame into the caller's CSC array
    if (F.fp32) {
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
      __threadfence();
      atomicAdd(flags + fr.panel, diag ? 0x10001 : 1);
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

sc_status factor_range(Plan& P, int64_t t0, int64_t t1, int slot, cudaStream_t stream, std::string& err) {
  if (t1 <= t0) return SC_OK;
  factor_kernel<<<factor_grid(t1 - t0), 32 * kFWarps, kFSmem, stream>>>(P.fac.dev, t0, t1, slot);
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
  F.d_ptrs = nullptr;
  F.ready = false;
}

sc_status upload_factor_plan(Plan& P, std::string& err) {
  FactorPlan& F = P.fac;
  FCUDA(cudaSetDevice(P.opt.device));
  DevFactor D{};
  FTRY(fupload(F, F.panels, &D.panels, err));
  FTRY(fupload(F, F.Rrows, &D.Rrows, err));
  FTRY(fupload(F, F.upd, &D.upd, err));
  FTRY(fupload(F, F.frames, &D.frames, err));
  FTRY(fupload(F, F.kent, &D.kent, err));
  FTRY(fupload(F, F.lent, &D.lent, err));
  FTRY(fupload(F, F.tasks, &D.tasks, err));
  FTRY(fupload(F, P.sub_cls, &D.sub_cls, err));
  FTRY(fupload(F, F.sub_W_base, &D.sub_W_base, err));
  FTRY(fupload(F, F.sub_flag_base, &D.sub_flag_base, err));
  FTRY(fupload(F, F.cls_panel0, &D.cls_panel0, err));
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
  FCUDA(cudaMemsetAsync(P.dev.err, 0, sizeof(unsigned long long) * (1 + (size_t)P.nsub), stream));
  FCUDA(cudaMemsetAsync(F.dev.flags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nflags, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  return factor_range(P, 0, (int64_t)F.tasks.size(), 0, stream, err);
}

// Host-fed pipeline: per chunk of subdomains, H2D of its K values on the copy stream, then on `stream`
// the factorization of the chunk into the plan's L staging buffer and the chunk's assembly.
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
  FCUDA(cudaMemsetAsync(F.dev.flags, 0, sizeof(int32_t) * (size_t)std::max<int64_t>(F.nflags, 1), stream));
  FCUDA(cudaMemsetAsync(F.dev.queue, 0, sizeof(int32_t) * kQueueSlots, stream));
  cudaStream_t cs = static_cast<cudaStream_t>(P.copy_stream);
  FCUDA(cudaEventRecord(static_cast<cudaEvent_t>(P.ev_start), stream));
  FCUDA(cudaStreamWaitEvent(cs, static_cast<cudaEvent_t>(P.ev_start), 0));
  const int32_t nchunk = (int32_t)F.chunk_sub.size() - 1;
  while ((int32_t)P.ev_chunk.size() < nchunk) {
    cudaEvent_t e;
    FCUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    P.ev_chunk.push_back(e);
  }
  for (int32_t k = 0; k < nchunk; k++) {
    const int32_t s0 = F.chunk_sub[(size_t)k], s1 = F.chunk_sub[(size_t)k + 1];
    int32_t i = s0;
    while (i < s1) {  // one copy per run of host-contiguous subdomains
      if (F.sub_nnzK[(size_t)i] == 0) {
        i++;
        continue;
      }
      const char* src = static_cast<const char*>(Khost[i]);
      size_t bytes = 8 * (size_t)F.sub_nnzK[(size_t)i];
      int32_t j = i + 1;
      while (j < s1 && F.sub_nnzK[(size_t)j] > 0 && static_cast<const char*>(Khost[j]) == src + bytes) {
        bytes += 8 * (size_t)F.sub_nnzK[(size_t)j];
        j++;
      }
      FCUDA(cudaMemcpyAsync(static_cast<char*>(F.d_Kstage) + 8 * F.Kstage_off[(size_t)i], src, bytes,
                            cudaMemcpyHostToDevice, cs));
      i = j;
    }
    cudaEvent_t e = static_cast<cudaEvent_t>(P.ev_chunk[(size_t)k]);
    FCUDA(cudaEventRecord(e, cs));
    FCUDA(cudaStreamWaitEvent(stream, e, 0));
    FTRY(factor_range(P, F.task_chunk[(size_t)k], F.task_chunk[(size_t)k + 1], k % kQueueSlots, stream, err));
    FTRY(assemble_range(P, s0, s1, stream_v, err));
  }
  return SC_OK;
}

}  // namespace sc
