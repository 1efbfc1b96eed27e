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
constexpr int kChunk = 64;      // below-diagonal rows per L block
constexpr int kSmallPanel = 32; // panels up to this width are prepared by one warp each

#ifdef __CUDACC__
#define SC_HD __host__ __device__
#else
#define SC_HD
#endif

// Leading dimension (in doubles) of a staged block holding `rows` rows: the smallest value
// >= rows that is == 4 (mod 16), so DMMA fragment loads (4 consecutive k x 8 consecutive rows)
// hit 16 distinct 8-byte bank pairs.
// (ld == 4 (mod 8) suffices: for t = 0..3 and 4 consecutive rows, ld*t + row covers 16 banks.)
SC_HD constexpr int block_ld(int rows) { return rows <= 4 ? 4 : 4 + 8 * ((rows - 4 + 7) / 8); }

constexpr int kLdC = 68;                        // block_ld(kChunk): ld of a full 64-row chunk
constexpr size_t kSmemBudget = 232448;          // B200 max dynamic shared memory per block (227 KB)
constexpr int64_t kSmemPerSM = 233472;          // B200 shared memory per SM (228 KB)
constexpr int kSlots = 16;                      // TRSM L-block pipeline depth (mbarrier pairs)
constexpr int kRingMaxBytes = 163840;           // TRSM L-block ring: at most 160 KB ...
constexpr int kBlockMaxBytes = kLdC * kMaxPanel * 8;  // ... and at least 2 of the largest blocks

// Byte offsets of the TRSM kernel's dynamic shared memory: full/empty mbarriers and ring offsets
// of the L-block pipeline, per-slot strip rows of a chunk's R_p rows (uint16, copied with the
// block), the byte ring of L blocks (ring_bytes, sized by the planner from what the strip leaves
// free), the solved panel Y (64 x ld) and the X strip ((strip_cap + 4) rows of ld doubles).
struct TrsmSmem {
  size_t full, empty, off, srow, ring, ys, strip, total;
};
// Row stride of the shared-memory strip: T (column-swizzled) for T >= 16, T + 4 for T = 8.
SC_HD constexpr int strip_ld(int T) { return T >= 16 ? T : T + 4; }
SC_HD inline TrsmSmem trsm_smem_layout(int T, int ring_bytes, int strip_cap, bool global_strip, bool ybuf) {
  TrsmSmem s{};
  s.full = 0;
  s.empty = 8 * kSlots;
  s.off = 16 * kSlots;            // per-slot records (48 B each, kernels.cu SlotRec)
  s.srow = s.off + 48 * kSlots;
  s.ring = s.srow + sizeof(uint16_t) * kSlots * kChunk;
  // 512 B guard after the ring: a warp's 8-row fragment loads of a block whose ld is below 64 may
  // read up to 60 doubles past its end (rows that are never used)
  s.ys = s.ring + (size_t)ring_bytes + 512;
  // Y buffer (Y mode: 64 x strip_ld(T)); in W mode the solved panel stays in registers
  s.strip = s.ys + (ybuf ? sizeof(double) * (size_t)kMaxPanel * (size_t)strip_ld(T) : 0);
  s.total = s.strip + (global_strip ? 0 : sizeof(double) * (size_t)(strip_cap + 4) * (size_t)strip_ld(T));
  return s;
}

// A factor panel (P:482-494 factor splitting; relaxed: several small supernodes may be merged
// into one dense panel, zeros stored explicitly).  Columns [a, a+kw); below-diagonal row set
// R_p = Rrows[R_off .. R_off+nR) (ascending, all >= a+kw: the pruned rows).  In the
// per-subdomain panel buffer (written by the prep kernel) it occupies, from buf_off: the inverse
// of its diagonal block (ldD x kw4, column-major) then ceil(nR/64) row chunks of L[R_p, panel]
// (chunk c: ld = block_ld(rows_c) x kw4, column-major).
struct Panel {
  int32_t a, kw, kw4, nR;
  int32_t R_off, nchunk, ldD, ldLast;   // ldLast = ld of the last chunk
  int64_t buf_off;                      // doubles from the subdomain's panel-buffer base
  int64_t csc_begin, csc_end;           // L entries of columns [a, a+kw) in CSC order
  int32_t relaxed, pad;                 // relaxed: merged supernodes (structural zeros inside)
  int64_t gx_off;                       // warp TRSM: first entry of the panel's fragment gather map
};

// Warp TRSM (narrow panels, kw <= 32): per panel a gather map from DMMA fragment positions to CSC
// positions of L (int32 relative to the subdomain's L values, -1 = structural zero), so a warp
// loads its m8n8k4 A fragments straight from the caller's CSC values (L crosses HBM once):
//   triangle: 8x8 blocks (I >= K) in the order K = 0.., I = K..kw8-1; per block [lane][s] (s = 0,1)
//             -> L[a + 8I + g][a + 8K + 4s + t]   (lane = 4g + t)
//   R rows:   per row block RB of R_p, [s/2][lane][s%2] (s < KS = 2 kw8) -> L[R_p[8RB + g]][a + 4s + t]
//             (one int2 per lane and pair of k steps: lane-contiguous, bank-conflict free once staged)
SC_HD inline int64_t warp_tri_block(int K, int I, int kw8) { return (int64_t)(K * kw8 - K * (K - 1) / 2 + (I - K)); }
SC_HD inline int64_t warp_gx_size(int kw, int nR) {
  const int kw8 = (kw + 7) / 8, nRB = (nR + 7) / 8;
  return 64 * (int64_t)(kw8 * (kw8 + 1) / 2) + (int64_t)nRB * 32 * (2 * kw8);
}

// One RHS column tile of TRSM width T of one pattern class: stepped columns [col0, col0+width)
// (P:473-480 RHS splitting at tile granularity).  Its X strip holds the rows of the panels of
// its reach (whole panels), in panel order.
struct Tile {
  int32_t col0, width, strip_rows, group;
  int32_t step_begin, step_end;    // panels visited (global indices into steps[])
  int32_t binit_begin, binit_end;  // B~^T scatter entries (global indices into binit[])
  int32_t col_in_group, pad;
};

// TRSM step: tile visits panel `panel` (global index) whose rows start at `strip_row` (tile strip in
// shared memory, or the group strip itself for global strips).
// srow_off: offset (uint16 units, 64 per chunk) of the strip rows of R_p for this tile in srows[]
// (0xFFFF = row outside the tile's reach, whose update is exactly zero).
struct Step {
  int32_t panel, strip_row;
  int32_t grow, pad;               // row of the panel in the tile's group strip (solved rows go there)
  int64_t srow_off;
};
// Warp TRSM step descriptor: the Step and Panel fields one step of trsm_warp_kernel reads, in one
// 32-byte sector (one dependent load per step instead of Step -> Panel)
struct WStep {
  int32_t strip_row, a, kw, nR;    // strip row of the panel, its first column, width, pruned rows
  int64_t gx_off, srow_off;        // fragment gather map (global), strip rows of R_p (global)
};
static_assert(sizeof(WStep) == 32, "WStep is one sector");


// SYRK column group (width kGroup, a union of TRSM tiles): its X strip in global memory holds
// the union of the member tiles' panels; reach entries (panel, off) in panel order.
struct Group {
  int32_t col0, width, strip_rows, pad;
  int32_t reach_begin, reach_end;
  int64_t x_off;                   // doubles from the subdomain's X base (row-major, kGroup wide)
};

struct Reach {
  int32_t panel, off;              // global panel index, first strip row
};

// One structural non-zero of B~^T placed in a tile strip (P:399-405 stepped column permutation).
struct BInit {
  int32_t strip_row, col;
  double val;
};

// SYRK output tile (I >= J) of a class over groups: F'[I,J] = sum_seg X_I[seg]^T X_J[seg]
// (P:534-540 output splitting with per-block k range; segments = rows both strips hold).
struct Pair {
  int32_t I, J;                    // global group indices
  int32_t seg_begin, seg_end;      // global indices into segs[]
};

struct Seg {
  int32_t offI, offJ, len, pad;
};

struct I2 {
  int32_t x, y;
};
// Input-split SYRK (f3 ablation, SC_SYRK_SPLIT=input): one warp per (subdomain, pair, common-row
// segment, 16 x 16 sub-tile (ib, jb) of the pair's G x G output tile)
struct SplitTask {
  int32_t sub, pair, seg, ij;      // ij = ib * 4 + jb
};

// Apply: one 64 x 64 tile (row block rb >= column block cb) of the lower F' of subdomain sub.
constexpr int kApplyTile = 64;
// F' storage (SURVEY §8.1 a4/a5 "lower tiles"): per subdomain only the lower 64 x 64 tiles (rb >= cb),
// tile (rb, cb) at position rb (rb + 1) / 2 + cb, each column-major with ld 64 (the diagonal tiles'
// upper halves stay unused); about half of an m x m square.
SC_HD inline int64_t f_tiles(int m) {
  const int64_t nab = (m + kApplyTile - 1) / kApplyTile;
  return nab * (nab + 1) / 2;
}
SC_HD inline int64_t f_index(int r, int c) {  // r >= c
  const int rb = r / kApplyTile, cb = c / kApplyTile;
  return ((int64_t)rb * (rb + 1) / 2 + cb) * (kApplyTile * kApplyTile) + (int64_t)(c % kApplyTile) * kApplyTile +
         (r % kApplyTile);
}
struct ApplyTask {
  int32_t sub, rb, cb, pad;
};

// Symbolic plan of one pattern class (subdomains with identical L pattern, perm and B~^T).
struct ClassPlan {
  int32_t n = 0, m = 0, nsup = 0;
  uint64_t hash = 0;
  std::vector<int64_t> colptr;     // copy of L_colptr (n+1)
  std::vector<int32_t> rowidx;     // copy of L_rowidx (nnz(L)): the device factorization's symbolic input
  std::vector<int32_t> perm;       // perm[new] = old
  std::vector<int32_t> dest;       // per CSC entry: >= 0 panel-buffer offset (below rows),
                                   //   < 0: -1 - (col_in_panel * 64 + row_in_panel) (triangle)
  std::vector<Panel> panels;
  std::vector<int32_t> Rrows;      // concatenated R_p
  std::vector<int32_t> sigma;      // stepped position -> original local column
  std::vector<int32_t> pivot;      // per stepped position (permuted row), n for empty columns
  std::vector<Tile> tiles;         // *_begin/_end: class-local until build_plan globalises them
  std::vector<Step> steps;
  std::vector<uint16_t> srows;     // per step, per chunk: 64 strip rows of R_p (see Step)
  std::vector<Group> groups;
  std::vector<Reach> greach;
  std::vector<BInit> binit;
  std::vector<int32_t> ib_ptr, ib_row;  // B~^T by stepped column (m+1 pointers, permuted rows)
  std::vector<double> ib_val;
  std::vector<Pair> pairs;
  std::vector<Seg> segs;
  std::vector<int32_t> gidx;       // warp TRSM fragment gather maps (Panel::gx_off, class-local)
  int64_t x_doubles = 0;           // X region (group strips) per subdomain
  int64_t pb_doubles = 0;          // panel buffer per subdomain
  int32_t max_strip_rows = 0;      // over TRSM tiles
  bool too_big = false;            // analysis stopped: a strip exceeds the shared-memory limit
  // counters (per subdomain of this class)
  double fl_trsm_useful = 0, fl_syrk_useful = 0, fl_trsm_env = 0, fl_syrk_env = 0;
  double fl_trsm_dense = 0, fl_syrk_dense = 0, fl_trsm_sparse = 0;
  double fl_trsm_exec = 0, fl_syrk_exec = 0, fl_prep_exec = 0;
  double x_reach_doubles = 0;      // sum over tiles of own-reach rows x T
};

// ---- Numeric factorization on the device (§2.2 "two-stage
// factorization": symbolic once, numeric whenever K changes).  Left-looking supernodal Cholesky of
// P K_reg P^T over factor panels of <= 32 columns (a partition of its own, independent of the TRSM's).
constexpr int kFW = 32;         // factor panel width cap = frame rows = frame columns
// Factor panel: columns [a, a+kw), below-diagonal rows R = fRrows[R_off .. R_off+nR) (ascending).
// Workspace per subdomain (doubles from the subdomain's base): the finished L[R, panel] at w_off
// (nR x kw8, row-major: row r at w_off + r kw8, padding columns zero) and inv(L_pp) at inv_off
// (kw8 x kw8, column-major, zero padded).
struct FPanel {
  int32_t a, kw, nR, R_off;
  int32_t upd_begin, upd_end;      // descendant updates of this panel (class-local indices into FactorClass::upd)
  int32_t frame_begin, nframe;     // 1 diagonal frame + ceil(nR / 32) row frames (global indices)
  int64_t w_off, inv_off;
  int32_t level, kw8;              // level: 0 = no descendants, else 1 + max over its descendants
  int32_t anc_begin, anc_end;      // implicit apply (backward): the ancestor panels this panel updates
                                   //   (global indices into fanc: {a, s0, s1} = R_p[s0, s1) in a's columns)
};
// Descendant panel d updates panel p: rows R_d[s0, s1) lie in [a_p, a_p + kw_p) (the columns of p),
// rows R_d[s1, nR_d) below it (a subset of R_p by the closure of the fill pattern).
struct FUpd {
  int32_t d, s0, s1, pad;          // d: global factor-panel index
};
// Frame = one warp task: the diagonal block (r0 = -1, rows = the panel's columns) or 32 consecutive
// rows R_p[r0, r0 + nrow) of a panel.  K / L entries of the frame: (value index within the subdomain's
// CSC array, frame position row * 32 + col).  Frame updates [u_begin, u_end): the descendant panels
// that touch this frame (global indices into fupd).
struct FFrame {
  int32_t panel, r0, nrow, pad;
  int32_t k_begin, k_end, l_begin, l_end;
  int32_t u_begin, u_end;          // the frame task's own updates
  int32_t part_begin, part_end;    // its split-off partial update tasks (FPart, class-local index
                                   //   relative to the subdomain's partial slots; global list offset
                                   //   via cls_part0)
};
// Partial update task of a frame with many descendant updates (SC_FACTOR_SPLIT): accumulates the
// updates [u_begin, u_end) of `frame` into a partial 32 x 32 block (subdomain slot `slot`), summed
// by the frame task in slot order.
struct FPart {
  int32_t frame, u_begin, u_end, slot;
};
// Descendant panel d updates one frame of p: the frame's columns get d's rows R_d[s0, s1) (values in
// [a_p, a_p + kw_p)); its rows get R_d[k0, k1) (diagonal frame: k0 = s0, k1 = s1; row frame: the rows of
// R_d below p's columns whose values fall in the frame's row range -- contiguous in R_d; a row of a
// relaxed panel that is not in R_p contributes exact zeros and is skipped by the kernel).
struct FFUpd {
  int32_t d, s0, s1, k0, k1, pad;
};
struct FEnt {
  int32_t q, pos;
};
struct FTask {
  int32_t sub, frame;              // frame: global index
  int32_t nf, pad;                 // frames [frame, frame + nf) of one panel, processed in order by one warp
};

// Host symbolic data of the device factorization, per pattern class.
struct FactorClass {
  std::vector<FPanel> panels;      // class-local indices until globalised
  std::vector<int32_t> Rrows;
  std::vector<FUpd> upd;
  std::vector<FFrame> frames;
  std::vector<FFUpd> fupd;
  std::vector<FPart> parts;        // partial update tasks (class-local frame / update indices)
  std::vector<FEnt> kent, lent;
  std::vector<FUpd> anc;           // per panel (FPanel::anc_*): {ancestor a, s0, s1}
  std::vector<int32_t> bt_rp, bt_a; // B~^T by permuted row (CSR, n+1 / entries): stepped column, value
  std::vector<double> bt_v;
  int64_t nnzK = 0, w_doubles = 0;
  int32_t max_level = 0;
  double flops = 0;                // executed factorization flops per subdomain (updates + diag + TRSM)
  double flops_useful = 0;         // sum_k cc_k^2 (column counts of L): the textbook Cholesky count
};

// Device view of the factorization plan.
struct DevFactor {
  const FPanel* panels;
  const int32_t* Rrows;            // concatenated per class; FPanel::R_off globalised
  const FFUpd* fupd;
  const FFrame* frames;            // FFrame::k_* / l_* global indices into kent / lent
  const FEnt* kent;
  const FEnt* lent;
  const FTask* tasks;
  const int32_t* sub_cls;
  const int64_t* sub_W_base;       // doubles
  const int64_t* sub_flag_base;    // per subdomain: first flag (one per factor panel of its class)
  const int32_t* cls_panel0;       // per class first global factor panel
  const void* const* Kptr;         // per subdomain K values (device, double)
  void* const* Lout;               // per subdomain L values out (device; double, or float when fp32)
  double* W;
  int32_t* flags;                  // per (sub, panel): completed frames + 0x10000 once the diagonal is done
  int32_t* queue;                  // task counters (one per launch slot)
  unsigned long long* err;
  int32_t fp32, pad;
  // implicit apply on the factor workspace
  const FUpd* anc;
  const I2* ptasks;                // (sub, global panel) in forward (level) order; backward = reversed
  const int32_t* bt_rp;            // per class (offset cls_bt0) CSR of B~^T by permuted row
  const int32_t* bt_a;
  const double* bt_v;
  const int64_t* cls_bt0;          // per class: offset into bt_rp (n+1 entries); bt_rp values are global
  const int64_t* sub_x_base;       // per subdomain: offset of its work vector in xv (n doubles)
  double* xv;
  const void* const* Lin;          // stage mode: the plan's L table (DevPlan::Lptr)
  const int64_t* slm;              // = DevPlan::slm / sub_slm_off (stepped lambda map)
  const int64_t* sub_slm_off;
  // split frames (SC_FACTOR_SPLIT): partial update tasks, their per-subdomain slots and flags
  const FPart* parts;              // global list (FPart::frame / u_* global)
  const int32_t* cls_part0;        // per class: first entry of its parts in the global list
  const int64_t* sub_part_base;    // per subdomain: first partial slot
  int32_t* pflags;                 // per partial slot: 1 once its block is written
  double* pbuf;                    // per partial slot: 32 lanes x 32 accumulator values ([value][lane])
};

struct FactorPlan {
  bool ready = false;
  std::vector<FactorClass> classes;
  std::vector<FPanel> panels;      // global
  std::vector<int32_t> Rrows;
  std::vector<FFUpd> fupd;
  std::vector<FFrame> frames;
  std::vector<FEnt> kent, lent;
  std::vector<FTask> tasks;
  std::vector<FUpd> anc;
  std::vector<I2> ptasks;
  std::vector<FPart> parts;        // global
  std::vector<int32_t> cls_part0, cls_frame0;
  std::vector<int64_t> sub_part_base;
  int64_t nparts = 0;              // partial slots over all subdomains
  int32_t part_merge = 1;          // partials merged per slot to fit the budget (> 64: no split)
  int32_t part_min_updates = 0;    // only frames with more updates than this are split (budget)
  std::vector<int32_t> bt_rp, bt_a;
  std::vector<double> bt_v;
  std::vector<int64_t> cls_bt0, sub_x_base;
  bool has_K = false;              // built with a K pattern (factorize), else staging from L only
  bool w_ready = false;            // W holds the factor (last factorize or stage)
  std::vector<int64_t> task_chunk; // {number of tasks of the whole-batch order}
  std::vector<int64_t> sub_W_base, sub_flag_base, sub_nnzK;
  std::vector<int32_t> cls_panel0;
  int64_t W_doubles = 0, nflags = 0;
  double flops = 0, flops_useful = 0, bytes_K = 0;
  DevFactor dev{};
  std::vector<void*> allocations;
  void** h_ptrs = nullptr;         // pinned: nsub K pointers then nsub L pointers
  void** d_ptrs = nullptr;
  void* ptr_event = nullptr;
  void* d_Kstage = nullptr;        // host-fed path: K values staging
  void* d_hptrs = nullptr;         // host-fed path: device table of the mapped host K pointers
  int64_t* d_Kstage_off = nullptr; //   and the staging offsets (gather_host_kernel)
  const void** h_hptrs = nullptr;  //   pinned upload buffer of that table (guarded by hptr_event)
  void* hptr_event = nullptr;
  std::vector<int64_t> Kstage_off;
};

// Per-launch parameters of the TRSM kernel: first task, L-block ring bytes and shared strip capacity
// (rows) of this launch (tiles are split into a small-strip class at two CTAs per SM and the rest).
struct TrsmLaunch {
  int32_t task0, ring_bytes, strip_cap, pad;
};

// Device-side view passed by value to every kernel.
struct DevPlan {
  const Panel* panels;             // all classes, concatenated
  const int32_t* Rrows;
  const int32_t* dest;             // concatenated per class (offset cls_csc_off)
  const int64_t* cls_csc_off;
  const Tile* tiles;
  const Step* steps;
  const WStep* wsteps;             // warp TRSM: per step, Step + Panel fields (empty otherwise)
  const uint16_t* srows;           // concatenated per class (Step.srow_off globalised)
  const Group* groups;
  const Reach* greach;
  const BInit* binit;
  const Pair* pairs;
  const Seg* segs;
  const int32_t* sub_cls;          // per subdomain
  const int32_t* cls_panel0;       // per class: first global panel, then (next entry) the end
  const int64_t* cls_ib0;          // per class: offset into ib_ptr; ib_ptr values are global entry indices
  const int32_t* ib_ptr;
  const int32_t* ib_row;
  const double* ib_val;
  double* upart;                   // implicit apply: per (subdomain, stepped column) result, sub_slm_off
  double* xv;                      // implicit apply: per subdomain work vector (n doubles) if not in smem
  const int64_t* sub_X_base;       // per subdomain, doubles
  const int64_t* sub_F_base;       // per subdomain, elements (F' lower 64 x 64 tiles, f_index)
  const int64_t* sub_PB_base;      // per subdomain panel buffer, doubles
  const int32_t* sub_m;
  const void* const* Lptr;         // per subdomain L values (device; double, or float when fp32)
  const I2* prep_tasks;            // (sub, global panel), panels wider than kSmallPanel
  const I2* prep_small_tasks;      // (sub, global panel), panels of <= kSmallPanel columns, bucketed
                                   //   by padded width 8 / 16 / 32 (Plan::small_begin)
  const I2* trsm_tasks;            // (sub, global tile)
  const I2* syrk_tasks;            // (sub, global pair)
  const ApplyTask* apply_tasks;
  const int64_t* sub_slm_off;      // per subdomain offset into slm (stepped lambda map)
  const int64_t* slm;              // lambda_map[sigma[a]] per subdomain, concatenated
  const int32_t* ssig;             // sigma[a] (original local column of stepped a), same layout
  const int64_t* sub_part_off;     // per subdomain offset into apply partial buffer
  const int64_t* qg_ptr;           // CSR over global multipliers: contributions
  const int64_t* qg_sub_a;         // (sub << 32) | a
  void* X;                         // X group strips: double, or float when fp32
  void* F;                         // F' lower tiles: double, or float when fp32
  double* PB;                      // panel buffers
  double* part;
  unsigned long long* err;         // sticky device error: [0] = ((sub+1) << 32) | col, [1+sub] = col+1
  const int32_t* gidx;             // warp TRSM gather maps (all classes; Panel::gx_off is global)
  int32_t nsub, max_n, T, G;
  int32_t wmode;                         // 1: chunks hold W_p = L[R_p,p] inv(L_pp) (W mode), 0: L (Y mode)
  int32_t fp32;                          // precision 32: L, X and F' stored in FP32 (FP64 arithmetic)
};

struct Plan {
  sc_options opt{};
  int32_t T = 32, G = 64, PW = 64, ring_bytes = 0;
  bool gstrip = false;             // X strips solved in place in the group strips (global memory)
  int32_t gs2 = 0;                 // global strips at T = 16 with this many CTAs per SM (2; 3 via SC_GS2=3)
  bool wmode = true;               // TRSM update operand W_p = L[R_p,p] inv(L_pp) (wide panels) or L (Y mode)
  bool warp_trsm = false;          // fused warp-per-tile TRSM straight from the CSC values (no prep)
  bool syrk_input = false;         // SC_SYRK_SPLIT=input: input-split SYRK (f3 ablation) instead of output split
  const SplitTask* d_split = nullptr;
  std::vector<int64_t> split_sub_begin;  // first split task of each subdomain (nsub + 1)
  int32_t warp_ctas = 4;           // warps (tiles) per CTA of the warp TRSM
  int32_t nsub = 0;
  std::vector<ClassPlan> classes;
  std::vector<int32_t> sub_cls;
  std::vector<int32_t> sub_m, sub_n;
  std::vector<int64_t> sub_nnz;
  // global (concatenated) arrays
  std::vector<int32_t> cls_tile_begin, cls_pair_begin, cls_panel_begin, cls_group_begin;
  std::vector<I2> prep_tasks, prep_small_tasks, trsm_tasks, syrk_tasks;
  int32_t small_begin[4] = {0, 0, 0, 0};  // prep_small_tasks buckets: npad 8 | 16 | 32
  std::vector<ApplyTask> apply_tasks;
  std::vector<int64_t> sub_X_base, sub_F_base, sub_PB_base, sub_part_off, sub_slm_off;
  std::vector<int64_t> slm, qg_ptr, qg_sub_a;
  std::vector<int32_t> ssig;
  int64_t X_doubles = 0, F_doubles = 0, PB_doubles = 0, part_doubles = 0;
  int32_t max_n = 0, max_strip_rows = 0;
  sc_stats stats{};
  // device state
  bool on_device = false;
  DevPlan dev{};
  std::vector<void*> allocations;
  const void** h_Lptr_pinned = nullptr;     // pinned staging for the per-call pointer array
  double** d_Lptr = nullptr;
  std::vector<const void*> last_Lptr;
  int32_t esz = 8;                         // bytes per stored element of L / X / F' (8, or 4 when fp32)
  void* lptr_event = nullptr;              // cudaEvent_t of the last pointer upload
  void* d_Lstage = nullptr;                // staging for sc_assemble_batch_host
  std::vector<int64_t> Lstage_off;
  void* last_stream = nullptr;
  void* tev[4] = {nullptr, nullptr, nullptr, nullptr};  // optional timing events (sc_set_timing_events)
  int64_t n_lambda = 0;
  size_t smem_trsm = 0;
  // small-strip TRSM tile class: trsm_tasks[0, ntrsm_small) at two CTAs per SM
  int32_t ntrsm_small = 0, ring_small = 0, strip_small = 0;
  size_t smem_trsm_small = 0;
  void* side_stream = nullptr;   // cudaStream_t for the large-strip launch
  void* ev_fork = nullptr;       // cudaEvent_t
  void* ev_join = nullptr;
  int32_t overlap = 0;           // >1: phase-overlapped assembly over this many subdomain chunks
  void* ov_stream[2] = {nullptr, nullptr};
  std::vector<void*> ev_ov;
  void* copy_stream = nullptr;   // host-fed pipeline (sc_assemble_batch_host): H2D copies
  void* d_hsrc = nullptr;        // host-fed pipeline: device table of the mapped host L pointers
  int64_t* d_Lstage_off = nullptr;
  const void** h_hsrc = nullptr; //   its pinned upload buffer (guarded by ev_hsrc)
  void* ev_hsrc = nullptr;
  void* ev_start = nullptr;
  std::vector<void*> ev_chunk;
  FactorPlan fac;                // device numeric factorization (sc_factor_attach)
};

// plan.cpp
struct PanelPart {
  int32_t a = -1, b = -1, merged = 0;  // columns [a, b); merged: relaxed (several supernodes)
  std::vector<int32_t> R;              // rows below the panel, ascending
};
// zmax / wsmall < 0: the TRSM defaults (SC_RELAX_ZMAX / SC_RELAX_WSMALL)
int32_t partition_panels(int32_t n, const int64_t* cp, const int32_t* ri, const std::vector<int32_t>& parent, int PW,
                         std::vector<PanelPart>& out, double zmax = -1.0, int wsmall = -1);
sc_status build_plan(const sc_subdomain_desc* sd, int32_t nsub, const sc_options& opt, Plan& P, std::string& err);

// kernels.cu
sc_status upload_plan(Plan& P, std::string& err);
void free_plan_device(Plan& P);
sc_status launch_assemble(Plan& P, const void* const* Lptr_host, void* stream, std::string& err);
sc_status launch_apply(Plan& P, const double* lambda, double* q, void* stream, std::string& err);
sc_status launch_prepare(Plan& P, const void* const* Lptr_host, void* stream, std::string& err);
sc_status launch_apply_implicit(Plan& P, const double* lambda, double* q, void* stream, std::string& err);
sc_status device_check(Plan& P, std::string& err);
sc_status copy_F_lower(Plan& P, int32_t i, std::vector<double>& out, std::string& err);
sc_status copy_X_strips(Plan& P, int32_t i, std::vector<double>& out, std::string& err);
sc_status export_F_device(Plan& P, int32_t i, double* F, int64_t ld, void* stream, std::string& err);
sc_status assemble_host_pipelined(Plan& P, const void* const* Lhost, void* stream, std::string& err);
sc_status assemble_stage_begin(Plan& P, std::vector<void*>& dptrs, void* stream, std::string& err);
sc_status assemble_range(Plan& P, int32_t s0, int32_t s1, void* stream, std::string& err);

// factor_plan.cpp / factor.cu (device numeric factorization)
sc_status build_factor_plan(Plan& P, const sc_K_pattern* kp, int32_t nsub, std::string& err);
sc_status upload_factor_plan(Plan& P, std::string& err);
void free_factor_device(Plan& P);
sc_status launch_factorize(Plan& P, const void* const* Kptr, void* const* Lout, void* stream, std::string& err);
sc_status factorize_assemble_host(Plan& P, const void* const* Khost, void* stream, std::string& err);
sc_status launch_stage(Plan& P, void* stream, std::string& err);
sc_status launch_implicit_solve(Plan& P, const double* lambda, void* stream, std::string& err);
sc_status ensure_factor_plan(Plan& P, std::string& err);  // K-less factor plan for the implicit apply
sc_status gather_host_range(const void* const* d_src, const int64_t* d_off, void* d_dst, int32_t s0, int32_t s1,
                            int esz, void* stream, std::string& err);

// pcpg.cu
sc_status pcpg_solve(Plan& P, const double* d, const double* e_host, double* lambda, const sc_coarse* cs,
                     const sc_pcpg_opts& o, sc_allreduce_fn allreduce, void* ctx, sc_pcpg_result* res, void* stream,
                     std::string& err);

}  // namespace sc
