// sc_internal.h — plan data structures shared by the host planner (plan.cpp), the device kernels
// (kernels.cu) and the C-ABI shim (api.cpp).  Not part of the public ABI (include/sc_b200.h).
#pragma once
#include <stdint.h>

#include <string>
#include <vector>

#include "sc_b200.h"

namespace sc {

constexpr int kThreads = 256;   // every kernel uses 8 warps
constexpr int kMaxPanel = 64;   // max factor panel width (factor-splitting block)
constexpr int kChunk = 64;      // rows per update / GEMM chunk

// One RHS column tile of one pattern class: stepped columns [col0, col0+width) (P:473-480 RHS
// splitting at tile granularity).  Its X strip holds only the rows of its reach, row-major with
// T doubles per row, at offset x_off inside the subdomain's X region.
struct Tile {
  int32_t col0, width, strip_rows, pad;
  int32_t step_begin, step_end;    // TRSM panel steps (global indices into steps[])
  int32_t reach_begin, reach_end;  // reach entries (global indices into reach[])
  int32_t binit_begin, binit_end;  // B~^T scatter entries (global indices into binit[])
  int64_t x_off;                   // doubles from the subdomain's X base
};

// One factor panel of a supernode as a TRSM step of one tile (diagonal-block TRSM
// then GEMM update of the pruned sub-diagonal rows).  Panel columns [e, e+kw) of the supernode
// whose last column is c1-1 and whose pruned row structure is R_s = Rrows[R_off .. R_off+nR).
struct Step {
  int32_t e, kw, c1, nR;
  int32_t R_off, strip_row;        // strip row of factor row e in the tile's X strip
};

// The rows [e, c1) of supernode s held by a tile's strip, starting at strip row `off`.
struct Reach {
  int32_t s, e, c1, off;
};

// One structural non-zero of B~^T placed in a tile strip (P:399-405 stepped column permutation).
struct BInit {
  int32_t strip_row, col;
  double val;
};

// SYRK output tile (I >= J) of a class: F'[I,J] = sum over segments of X_I[seg]^T X_J[seg]
// (P:534-540 output splitting with per-block k range; segments = rows both strips hold).
struct Pair {
  int32_t I, J;                    // global tile indices
  int32_t seg_begin, seg_end;      // global indices into segs[]
};

struct Seg {
  int32_t offI, offJ, len, pad;
};

struct I2 {
  int32_t x, y;
};

struct ApplyTask {
  int32_t sub, b0;                 // columns [b0, b0+32) of subdomain sub
};

// Symbolic plan of one pattern class (subdomains with identical L pattern, perm and B~^T).
struct ClassPlan {
  int32_t n = 0, m = 0, nsup = 0;
  uint64_t hash = 0;
  std::vector<int64_t> colptr;     // copy of L_colptr (n+1)
  std::vector<int32_t> rowidx;     // copy of L_rowidx (host: X export + checks)
  std::vector<int32_t> perm;       // perm[new] = old
  std::vector<int32_t> sn_c0, sn_c1, sn_nR;  // supernodes
  std::vector<int32_t> sn_Roff;    // offset into Rrows (class-local)
  std::vector<int32_t> Rrows;      // concatenated R_s
  std::vector<int32_t> sigma;      // stepped position -> original local column
  std::vector<int32_t> pivot;      // per stepped position (permuted row), n for empty columns
  std::vector<Tile> tiles;         // class-local indices in the *_begin/_end fields
  std::vector<Step> steps;
  std::vector<Reach> reach;
  std::vector<BInit> binit;
  std::vector<Pair> pairs;
  std::vector<Seg> segs;
  int64_t x_doubles = 0;           // X region size per subdomain
  // counters (per subdomain of this class)
  double fl_trsm_useful = 0, fl_syrk_useful = 0, fl_trsm_env = 0, fl_syrk_env = 0;
  double fl_trsm_dense = 0, fl_syrk_dense = 0, fl_trsm_sparse = 0;
  double fl_trsm_exec = 0, fl_syrk_exec = 0;
};

// Device-side view passed by value to every kernel.
struct DevPlan {
  const int64_t* colptr;           // concatenated class colptrs
  const int64_t* cls_colptr_off;   // per class
  const int32_t* Rrows;            // concatenated (global offsets baked into Step.R_off)
  const Tile* tiles;
  const Step* steps;
  const Reach* reach;
  const BInit* binit;
  const Pair* pairs;
  const Seg* segs;
  const int32_t* sub_cls;          // per subdomain
  const int64_t* sub_X_base;       // per subdomain, doubles
  const int64_t* sub_F_base;       // per subdomain, doubles (F' lower, column-major, ld = m)
  const int32_t* sub_m;
  const double* const* Lptr;       // per subdomain L values (device)
  const I2* trsm_tasks;            // (sub, global tile)
  const I2* syrk_tasks;            // (sub, global pair)
  const ApplyTask* apply_tasks;
  const int64_t* sub_slm_off;      // per subdomain offset into slm (stepped lambda map)
  const int64_t* slm;              // lambda_map[sigma[a]] per subdomain, concatenated
  const int64_t* sub_part_off;     // per subdomain offset into apply partial buffer
  const int64_t* qg_ptr;           // CSR over global multipliers: contributions
  const int64_t* qg_sub_a;         // (sub << 32) | a
  double* X;
  double* F;
  double* part;
  unsigned long long* err;         // sticky device error: ((sub+1) << 32) | col
  int32_t nsub, max_n;
};

struct Plan {
  sc_options opt{};
  int32_t T = 64, PW = 64;
  int32_t nsub = 0;
  std::vector<ClassPlan> classes;
  std::vector<int32_t> sub_cls;
  std::vector<int32_t> sub_m, sub_n;
  std::vector<int64_t> sub_nnz;
  std::vector<std::vector<int64_t>> lambda_map;  // per subdomain (original local order)
  // global (concatenated) arrays
  std::vector<int32_t> cls_tile_begin, cls_pair_begin;
  std::vector<I2> trsm_tasks, syrk_tasks;
  std::vector<ApplyTask> apply_tasks;
  std::vector<int64_t> sub_X_base, sub_F_base, sub_part_off, sub_slm_off;
  std::vector<int64_t> slm, qg_ptr, qg_sub_a;
  int64_t X_doubles = 0, F_doubles = 0, part_doubles = 0;
  int32_t max_n = 0;
  sc_stats stats{};
  // device state
  bool on_device = false;
  DevPlan dev{};
  std::vector<void*> allocations;
  const double** h_Lptr_pinned = nullptr;   // pinned staging for the per-call pointer array
  double** d_Lptr = nullptr;
  std::vector<const double*> last_Lptr;
  void* lptr_event = nullptr;              // cudaEvent_t of the last pointer upload
  double* d_Lstage = nullptr;              // staging for sc_assemble_batch_host
  std::vector<int64_t> Lstage_off;
  void* last_stream = nullptr;
  void* tev[3] = {nullptr, nullptr, nullptr};  // optional timing events (sc_set_timing_events)
  int64_t n_lambda = 0;
  size_t smem_trsm = 0, smem_syrk = 0;
};

// plan.cpp
sc_status build_plan(const sc_subdomain_desc* sd, int32_t nsub, const sc_options& opt, Plan& P, std::string& err);

// kernels.cu
sc_status upload_plan(Plan& P, std::string& err);
void free_plan_device(Plan& P);
sc_status launch_assemble(Plan& P, const double* const* Lptr_host, void* stream, std::string& err);
sc_status launch_apply(Plan& P, const double* lambda, double* q, void* stream, std::string& err);
sc_status device_check(Plan& P, std::string& err);
sc_status copy_F_lower(Plan& P, int32_t i, std::vector<double>& out, std::string& err);
sc_status copy_X_strips(Plan& P, int32_t i, std::vector<double>& out, std::string& err);
sc_status stage_host_L(Plan& P, const double* const* Lhost, void* stream, std::vector<const double*>& dptrs,
                       std::string& err);

}  // namespace sc
