// plan.cpp — "initialization" stage: host-only integer symbolic analysis.
//
// Per pattern class (subdomains with identical L pattern, perm and B~^T):
//   1. validate L (lower CSC, diagonal first, rows ascending) and that its pattern is a Cholesky fill
//      pattern (closed under the elimination tree), B~^T rows, perm;
//   2. elimination tree parent(j) = first sub-diagonal row of column j, maximal supernodes (chains
//      j -> j+1 with equal row structure below); factor panels of <= 64 columns: wide supernodes
//      split, runs of small consecutive supernodes merged into one dense panel while it stays mostly
//      non-zero (relaxed amalgamation); each panel's pruned below-diagonal row set R_p (P:494
//      "extract only the non-empty rows", CHOLMOD-like) and the CSC -> panel-buffer scatter map;
//   3. row-permute B~^T by perm, column pivots p_j (first non-zero), stepped order sigma =
//      stable sort by (p_j, j) (ties: SURVEY §8.3 reading 7);
//   4. RHS column tiles of width T and, per tile, the panels its X strip must hold:
//        exact    : panels met by the elimination-tree reach of the tile's B~^T non-zeros (zeros
//                   above the pivots and off the etree paths are preserved),
//        envelope : every panel ending below the tile's highest pivot (the paper's stepped envelope),
//        none     : every panel (the original algorithm);
//   5. per tile the ordered factor panels ("factor splitting") it must apply;
//   6. SYRK column groups of 64 and output tiles I >= J with the row segments both group strips
//      hold (output splitting with the k range restricted to non-zero rows);
//   7. work counters and memory layout.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <iterator>
#include <numeric>
#include <atomic>
#include <thread>
#include <unordered_map>

#include "sc_internal.h"

namespace sc {

namespace {

uint64_t fnv(uint64_t h, const void* data, size_t bytes) {
  const unsigned char* p = static_cast<const unsigned char*>(data);
  for (size_t i = 0; i < bytes; i++) {
    h ^= p[i];
    h *= 1099511628211ull;
  }
  return h;
}

uint64_t desc_hash(const sc_subdomain_desc& d) {
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, &d.n, sizeof(d.n));
  h = fnv(h, &d.m, sizeof(d.m));
  h = fnv(h, d.L_colptr, sizeof(int64_t) * (size_t)(d.n + 1));
  h = fnv(h, d.L_rowidx, sizeof(int32_t) * (size_t)d.L_colptr[d.n]);
  if (d.perm) h = fnv(h, d.perm, sizeof(int32_t) * (size_t)d.n);
  h = fnv(h, d.Bt_colptr, sizeof(int32_t) * (size_t)(d.m + 1));
  int64_t nb = d.Bt_colptr[d.m];
  h = fnv(h, d.Bt_rowidx, sizeof(int32_t) * (size_t)nb);
  h = fnv(h, d.Bt_values, sizeof(double) * (size_t)nb);
  return h;
}

bool same_pattern(const sc_subdomain_desc& a, const sc_subdomain_desc& b) {
  if (a.n != b.n || a.m != b.m) return false;
  if (a.L_colptr[a.n] != b.L_colptr[b.n]) return false;
  auto eq = [](const void* x, const void* y, size_t bytes) { return x == y || std::memcmp(x, y, bytes) == 0; };
  if (!eq(a.L_colptr, b.L_colptr, sizeof(int64_t) * (size_t)(a.n + 1))) return false;
  if (!eq(a.L_rowidx, b.L_rowidx, sizeof(int32_t) * (size_t)a.L_colptr[a.n])) return false;
  if ((a.perm == nullptr) != (b.perm == nullptr)) return false;
  if (a.perm && !eq(a.perm, b.perm, sizeof(int32_t) * (size_t)a.n)) return false;
  if (!eq(a.Bt_colptr, b.Bt_colptr, sizeof(int32_t) * (size_t)(a.m + 1))) return false;
  int64_t nb = a.Bt_colptr[a.m];
  if (!eq(a.Bt_rowidx, b.Bt_rowidx, sizeof(int32_t) * (size_t)nb)) return false;
  if (!eq(a.Bt_values, b.Bt_values, sizeof(double) * (size_t)nb)) return false;
  return true;
}

#define FAIL(code, msg)   \
  do {                    \
    err = (msg);          \
    return (code);        \
  } while (0)

sc_status validate_desc(const sc_subdomain_desc& d, int32_t i, std::string& err) {
  std::string who = "subdomain " + std::to_string(i) + ": ";
  if (d.n < 0 || d.m < 0) FAIL(SC_ERR_INVALID_ARG, who + "negative n or m");
  if (d.n > 65535) FAIL(SC_ERR_INVALID_ARG, who + "n > 65535 not supported (16-bit strip row map)");
  if (!d.L_colptr || (d.n > 0 && !d.L_rowidx)) FAIL(SC_ERR_INVALID_ARG, who + "NULL L pattern");
  if (!d.Bt_colptr || (d.m > 0 && d.Bt_colptr[d.m] > 0 && (!d.Bt_rowidx || !d.Bt_values)))
    FAIL(SC_ERR_INVALID_ARG, who + "NULL B^T arrays");
  if (d.L_colptr[0] != 0) FAIL(SC_ERR_PATTERN, who + "L_colptr[0] != 0");
  for (int32_t c = 0; c < d.n; c++) {
    int64_t a = d.L_colptr[c], b = d.L_colptr[c + 1];
    if (b <= a) FAIL(SC_ERR_PATTERN, who + "L column " + std::to_string(c) + " is empty (no diagonal)");
    if (d.L_rowidx[a] != c) FAIL(SC_ERR_PATTERN, who + "L column " + std::to_string(c) + ": diagonal not first");
    for (int64_t p = a + 1; p < b; p++)
      if (d.L_rowidx[p] <= d.L_rowidx[p - 1] || d.L_rowidx[p] >= d.n)
        FAIL(SC_ERR_PATTERN, who + "L column " + std::to_string(c) + ": rows not strictly ascending / out of range");
  }
  if (d.perm) {
    std::vector<char> seen((size_t)d.n, 0);
    for (int32_t k = 0; k < d.n; k++) {
      int32_t v = d.perm[k];
      if (v < 0 || v >= d.n || seen[(size_t)v]) FAIL(SC_ERR_PATTERN, who + "perm is not a bijection");
      seen[(size_t)v] = 1;
    }
  }
  if (d.Bt_colptr[0] != 0) FAIL(SC_ERR_PATTERN, who + "Bt_colptr[0] != 0");
  for (int32_t j = 0; j < d.m; j++) {
    if (d.Bt_colptr[j + 1] < d.Bt_colptr[j]) FAIL(SC_ERR_PATTERN, who + "Bt_colptr not monotone");
    for (int32_t p = d.Bt_colptr[j]; p < d.Bt_colptr[j + 1]; p++)
      if (d.Bt_rowidx[p] < 0 || d.Bt_rowidx[p] >= d.n) FAIL(SC_ERR_PATTERN, who + "B^T row out of range");
  }
  return SC_OK;
}

// Steps 2-7 for one class.
// Relaxation thresholds for merging consecutive small supernodes into one dense panel (the GPU
// analogue of relaxed supernode amalgamation; zeros are stored explicitly).  Overridable with the
// environment variables SC_RELAX_ZMAX / SC_RELAX_WSMALL for tuning experiments.
double relax_zmax() {
  const char* e = std::getenv("SC_RELAX_ZMAX");
  return e ? std::atof(e) : 0.2;
}
int relax_wsmall() {
  const char* e = std::getenv("SC_RELAX_WSMALL");
  return e ? std::atoi(e) : 16;
}

}  // namespace

// Maximal supernodes (chains j -> j+1 with equal row structure below) cut into factor panels of <= PW
// columns: wide supernodes split evenly, runs of small consecutive supernodes merged into one dense
// panel while the merged trapezoid stays mostly non-zero (<= SC_RELAX_ZMAX explicit zeros) or tiny
// (<= SC_RELAX_WSMALL columns) -- relaxed amalgamation.  R = the panel's pruned below-diagonal rows
// (P:494), the union of its columns' rows below the panel.  Returns the number of supernodes.
int32_t partition_panels(int32_t n, const int64_t* cp, const int32_t* ri, const std::vector<int32_t>& parent, int PW,
                         std::vector<PanelPart>& out, double zmax, int wsmall) {
  auto cc = [&](int32_t c) { return (int32_t)(cp[c + 1] - cp[c]); };
  std::vector<int32_t> sn_c0, sn_c1;
  for (int32_t c = 0; c < n;) {
    int32_t c0 = c;
    c++;
    while (c < n && parent[(size_t)(c - 1)] == c && cc(c - 1) == cc(c) + 1) c++;
    sn_c0.push_back(c0);
    sn_c1.push_back(c);
  }
  const int32_t nsup = (int32_t)sn_c0.size();
  if (zmax < 0) zmax = relax_zmax();
  if (wsmall < 0) wsmall = relax_wsmall();
  PanelPart open;
  double open_nnz = 0;
  auto close_open = [&]() {
    if (open.a < 0) return;
    out.push_back(open);
    open = PanelPart();
    open_nnz = 0;
  };
  for (int32_t s = 0; s < nsup; s++) {
    const int32_t c0 = sn_c0[(size_t)s], c1 = sn_c1[(size_t)s], w = c1 - c0;
    std::vector<int32_t> Rs(ri + cp[c1 - 1] + 1, ri + cp[c1]);  // rows of the supernode below c1
    double nnz_s = 0;
    for (int32_t c = c0; c < c1; c++) nnz_s += cc(c);
    if (w > PW) {
      close_open();
      const int32_t np = (w + PW - 1) / PW;
      for (int32_t k = 0; k < np; k++) {
        int32_t pa = c0 + (int32_t)((int64_t)w * k / np), pb = c0 + (int32_t)((int64_t)w * (k + 1) / np);
        open.a = pa;
        open.b = pb;
        open.R.clear();
        for (int32_t r = pb; r < c1; r++) open.R.push_back(r);
        open.R.insert(open.R.end(), Rs.begin(), Rs.end());
        close_open();
      }
      continue;
    }
    if (open.a >= 0) {
      // candidate merge of [open.a, open.b) with [c0, c1)
      std::vector<int32_t> R2;
      R2.reserve(open.R.size() + Rs.size());
      std::vector<int32_t> tail;
      for (int32_t r : open.R)
        if (r >= c1) tail.push_back(r);
      std::set_union(tail.begin(), tail.end(), Rs.begin(), Rs.end(), std::back_inserter(R2));
      const double w2 = (double)(c1 - open.a);
      const double dense = w2 * (w2 + 1) / 2 + w2 * (double)R2.size();
      const double nnz2 = open_nnz + nnz_s;
      const double zf = 1.0 - nnz2 / dense;
      if (w2 <= PW && (zf <= zmax || w2 <= wsmall)) {
        open.b = c1;
        open.R.swap(R2);
        open_nnz = nnz2;
        open.merged = 1;
        continue;
      }
      close_open();
    }
    open.a = c0;
    open.b = c1;
    open.R = Rs;
    open_nnz = nnz_s;
  }
  close_open();
  return nsup;
}

namespace {

// Steps 2-7 for one class.
sc_status analyse_class(const sc_subdomain_desc& d, int T, int kGroup, int PW, int skip, bool gstrip,
                        int32_t strip_limit, bool warp, ClassPlan& C, std::string& err) {
  const int32_t n = d.n, m = d.m;
  C.n = n;
  C.m = m;
  C.colptr.assign(d.L_colptr, d.L_colptr + n + 1);
  C.rowidx.assign(d.L_rowidx, d.L_rowidx + d.L_colptr[n]);
  C.perm.resize((size_t)n);
  for (int32_t k = 0; k < n; k++) C.perm[(size_t)k] = d.perm ? d.perm[k] : k;
  const int64_t* cp = d.L_colptr;
  const int32_t* ri = d.L_rowidx;
  auto cc = [&](int32_t c) { return (int32_t)(cp[c + 1] - cp[c]); };

  // --- 2. etree + closure check + maximal supernodes
  std::vector<int32_t> parent((size_t)n, -1);
  for (int32_t c = 0; c < n; c++)
    if (cc(c) > 1) parent[(size_t)c] = ri[cp[c] + 1];
  {
    // struct(c) \ {c, parent(c)} must be a subset of struct(parent(c)) (Cholesky fill pattern)
    std::vector<int32_t> mark((size_t)n, -1);
    for (int32_t c = 0; c < n; c++) {
      int32_t p = parent[(size_t)c];
      if (p < 0) continue;
      for (int64_t q = cp[p]; q < cp[p + 1]; q++) mark[(size_t)ri[q]] = c;
      for (int64_t q = cp[c] + 2; q < cp[c + 1]; q++)
        if (mark[(size_t)ri[q]] != c)
          FAIL(SC_ERR_PATTERN, "L pattern is not a Cholesky fill pattern (column " + std::to_string(c) +
                                   " row " + std::to_string(ri[q]) + " not in the structure of its etree parent)");
    }
  }
  std::vector<PanelPart> parts;
  C.nsup = partition_panels(n, cp, ri, parent, PW, parts);
  for (auto& pp : parts) {
    Panel p{};
    p.a = pp.a;
    p.kw = pp.b - pp.a;
    p.relaxed = pp.merged;
    p.nR = (int32_t)pp.R.size();
    p.R_off = (int32_t)C.Rrows.size();
    C.Rrows.insert(C.Rrows.end(), pp.R.begin(), pp.R.end());
    C.panels.push_back(p);
  }
  std::vector<int32_t> panel_of_col((size_t)n, -1);
  for (size_t k = 0; k < C.panels.size(); k++)
    for (int32_t c = C.panels[k].a; c < C.panels[k].a + C.panels[k].kw; c++) panel_of_col[(size_t)c] = (int32_t)k;

  // --- panel-buffer layout and the CSC -> panel-buffer scatter map
  int64_t pb = 0;
  C.dest.assign((size_t)cp[n], 0);
  for (auto& p : C.panels) {
    p.kw4 = (p.kw + 3) & ~3;
    p.ldD = block_ld(p.kw);
    p.nchunk = (p.nR + kChunk - 1) / kChunk;
    p.ldLast = p.nchunk ? block_ld(p.nR - (p.nchunk - 1) * kChunk) : 4;
    p.buf_off = pb;
    p.csc_begin = cp[p.a];
    p.csc_end = cp[p.a + p.kw];
    const int64_t chunk0 = pb + (int64_t)p.ldD * p.kw4;
    const int32_t b = p.a + p.kw;
    const int32_t* R = C.Rrows.data() + p.R_off;
    for (int32_t c = p.a; c < b; c++)
      for (int64_t q = cp[c]; q < cp[c + 1]; q++) {
        const int32_t r = ri[q];
        if (r < b) {
          C.dest[(size_t)q] = -1 - ((c - p.a) * kMaxPanel + (r - p.a));
        } else {
          const int32_t k = (int32_t)(std::lower_bound(R, R + p.nR, r) - R);
          const int32_t ch = k / kChunk, kr = k % kChunk;
          const int64_t off = chunk0 + (int64_t)ch * block_ld(kChunk) * p.kw4 +
                              (int64_t)(c - p.a) * (ch == p.nchunk - 1 ? p.ldLast : block_ld(kChunk)) + kr;
          if (off > INT32_MAX) FAIL(SC_ERR_INVALID_ARG, "panel buffer exceeds 2^31 doubles per subdomain");
          C.dest[(size_t)q] = (int32_t)off;
        }
      }
    pb = chunk0 + (int64_t)(p.nchunk > 0 ? (p.nchunk - 1) : 0) * block_ld(kChunk) * p.kw4 +
         (p.nchunk > 0 ? (int64_t)p.ldLast * p.kw4 : 0);
    C.fl_prep_exec += (double)p.kw * p.kw * p.kw / 3.0;
  }
  C.pb_doubles = pb;
  // warp TRSM: fragment gather maps (sc_internal.h) from the same CSC walk
  if (warp) {
    int64_t gx = 0;
    for (auto& p : C.panels) {
      if (p.kw > 32) FAIL(SC_ERR_INVALID_ARG, "warp TRSM needs factor panels of <= 32 columns");
      p.gx_off = gx;
      gx += warp_gx_size(p.kw, p.nR);
    }
    if (cp[n] > INT32_MAX) FAIL(SC_ERR_INVALID_ARG, "warp TRSM: nnz(L) exceeds 2^31");
    C.gidx.assign((size_t)gx, -1);
    for (auto& p : C.panels) {
      const int kw8 = (p.kw + 7) / 8, KS = 2 * kw8;
      const int64_t roff = p.gx_off + 64 * (int64_t)(kw8 * (kw8 + 1) / 2);
      const int32_t* R = C.Rrows.data() + p.R_off;
      const int32_t b = p.a + p.kw;
      for (int32_t c = p.a; c < b; c++)
        for (int64_t q = cp[c]; q < cp[c + 1]; q++) {
          const int32_t r = ri[q], cc = c - p.a;
          const int s = (cc & 7) >> 2, t = cc & 3;
          if (r < b) {
            const int rr = r - p.a, lane = 4 * (rr & 7) + t;
            C.gidx[(size_t)(p.gx_off + 64 * warp_tri_block(cc >> 3, rr >> 3, kw8) + 2 * lane + s)] = (int32_t)q;
          } else {
            const int32_t k = (int32_t)(std::lower_bound(R, R + p.nR, r) - R);
            const int lane = 4 * (k & 7) + t;
            const int ks = cc >> 2;  // k step; R maps are [row block][k step pair][lane] int2
            C.gidx[(size_t)(roff + (((int64_t)(k >> 3) * (KS / 2) + (ks >> 1)) * 32 + lane) * 2 + (ks & 1))] = (int32_t)q;
          }
        }
    }
  }
  if (std::getenv("SC_DEBUG_PB")) {
    double inv = 0, chunk = 0, useful = 0, nsmall = 0, nbig = 0;
    std::vector<int> hist(9, 0);
    for (auto& p : C.panels) {
      inv += (double)p.ldD * p.kw4;
      chunk += (p.nchunk > 0 ? (double)(p.nchunk - 1) * kLdC * p.kw4 + (double)p.ldLast * p.kw4 : 0);
      useful += (double)p.kw * (p.kw + 1) / 2 + (double)p.kw * p.nR;
      (p.kw > kSmallPanel ? nbig : nsmall) += 1;
      hist[std::min(8, (p.kw + 7) / 8)]++;
    }
    fprintf(stderr, "PB: panels %zu (small %g big %g) inv %g chunk %g useful-trapezoid %g nnzL %lld pb %lld | kw/8 hist", C.panels.size(), nsmall, nbig, inv, chunk, useful, (long long)cp[n], (long long)pb);
    for (int h : hist) fprintf(stderr, " %d", h);
    fprintf(stderr, "\n");
  }

  // --- 3. permuted B~^T, pivots, stepped order
  std::vector<int32_t> iperm((size_t)n);
  for (int32_t k = 0; k < n; k++) iperm[(size_t)C.perm[(size_t)k]] = k;
  std::vector<std::vector<std::pair<int32_t, double>>> bcol((size_t)m);
  std::vector<int32_t> piv((size_t)m, n);
  for (int32_t j = 0; j < m; j++) {
    auto& v = bcol[(size_t)j];
    for (int32_t p = d.Bt_colptr[j]; p < d.Bt_colptr[j + 1]; p++) v.push_back({iperm[(size_t)d.Bt_rowidx[p]], d.Bt_values[p]});
    std::sort(v.begin(), v.end(), [](auto& a, auto& b) { return a.first < b.first; });
    std::vector<std::pair<int32_t, double>> u;  // sum duplicates
    for (auto& e : v) {
      if (!u.empty() && u.back().first == e.first)
        u.back().second += e.second;
      else
        u.push_back(e);
    }
    v.swap(u);
    if (!v.empty()) piv[(size_t)j] = v.front().first;
  }
  C.sigma.resize((size_t)m);
  std::iota(C.sigma.begin(), C.sigma.end(), 0);
  std::stable_sort(C.sigma.begin(), C.sigma.end(), [&](int32_t a, int32_t b) { return piv[(size_t)a] < piv[(size_t)b]; });
  C.pivot.resize((size_t)m);
  for (int32_t a = 0; a < m; a++) C.pivot[(size_t)a] = piv[(size_t)C.sigma[(size_t)a]];
  // B~^T by stepped column, rows permuted (for the implicit apply)
  C.ib_ptr.assign((size_t)m + 1, 0);
  for (int32_t a = 0; a < m; a++) {
    for (auto& e : bcol[(size_t)C.sigma[(size_t)a]]) {
      C.ib_row.push_back(e.first);
      C.ib_val.push_back(e.second);
    }
    C.ib_ptr[(size_t)a + 1] = (int32_t)C.ib_row.size();
  }

  // --- work counters: c_k = #columns whose X(k,:) is structurally non-zero
  {
    std::vector<double> ck((size_t)n, 0.0);
    std::vector<int32_t> stamp((size_t)n, -1);
    for (int32_t j = 0; j < m; j++)
      for (auto& e : bcol[(size_t)j])
        for (int32_t k = e.first; k >= 0 && stamp[(size_t)k] != j; k = parent[(size_t)k]) {
          stamp[(size_t)k] = j;
          ck[(size_t)k] += 1.0;
        }
    std::vector<double> wk((size_t)n + 1, 0.0);
    for (int32_t j = 0; j < m; j++)
      if (piv[(size_t)j] < n) wk[(size_t)piv[(size_t)j]] += 1.0;
    for (int32_t k = 1; k < n; k++) wk[(size_t)k] += wk[(size_t)(k - 1)];
    for (int32_t k = 0; k < n; k++) {
      double c2 = 2.0 * cc(k) - 1.0;
      C.fl_trsm_useful += ck[(size_t)k] * c2;
      C.fl_trsm_env += wk[(size_t)k] * c2;
      C.fl_syrk_useful += ck[(size_t)k] * (ck[(size_t)k] + 1.0);
      C.fl_syrk_env += wk[(size_t)k] * (wk[(size_t)k] + 1.0);
    }
    C.fl_trsm_dense = (double)m * (double)n * (double)n;
    C.fl_syrk_dense = (double)n * (double)m * (double)(m + 1);
    C.fl_trsm_sparse = (double)m * (2.0 * (double)cp[n] - (double)n);
  }

  // --- 4. TRSM tiles and their reach at panel granularity
  const int32_t np = (int32_t)C.panels.size();
  const int32_t ntiles = (m + T - 1) / T;
  std::vector<int32_t> inreach((size_t)np, -1), stamp((size_t)n, -1), strip_base((size_t)np, -1),
      in_tile((size_t)np, -1);
  std::vector<std::vector<int32_t>> tile_panels((size_t)ntiles);
  // exact mode: row-level reach of each SYRK group (the rows its columns' etree paths pass through);
  // the SYRK's k ranges skip the rows of a common panel that are structurally zero for one side
  // (e.g. the rows of a supernode above the column's entry point)
  const int32_t ngroups_r = (m + kGroup - 1) / kGroup;
  const bool row_reach = skip == SC_SKIP_EXACT && !std::getenv("SC_SYRK_PANEL_REACH");
  std::vector<std::vector<char>> grow_reach(row_reach ? (size_t)ngroups_r : 0);
  for (auto& v : grow_reach) v.assign((size_t)n, 0);
  for (int32_t J = 0; J < ntiles; J++) {
    Tile t{};
    t.col0 = J * T;
    t.width = std::min(T, m - J * T);
    t.group = t.col0 / kGroup;
    t.col_in_group = t.col0 - t.group * kGroup;
    int32_t pmin = n;
    for (int32_t a = t.col0; a < t.col0 + t.width; a++) pmin = std::min(pmin, C.pivot[(size_t)a]);
    auto& tp = tile_panels[(size_t)J];
    if (skip == SC_SKIP_EXACT) {
      for (int32_t a = t.col0; a < t.col0 + t.width; a++)
        for (auto& e : bcol[(size_t)C.sigma[(size_t)a]])
          for (int32_t c = e.first; c >= 0 && stamp[(size_t)c] != J; c = parent[(size_t)c]) {
            stamp[(size_t)c] = J;
            inreach[(size_t)panel_of_col[(size_t)c]] = J;
            if (row_reach) grow_reach[(size_t)t.group][(size_t)c] = 1;
          }
      for (int32_t p = 0; p < np; p++)
        if (inreach[(size_t)p] == J) tp.push_back(p);
    } else if (pmin < n) {
      const int32_t from = (skip == SC_SKIP_ENVELOPE) ? pmin : 0;
      for (int32_t p = 0; p < np; p++)
        if (C.panels[(size_t)p].a + C.panels[(size_t)p].kw > from) tp.push_back(p);
    }
    int32_t rows = 0;
    for (int32_t p : tp) rows += C.panels[(size_t)p].kw;
    C.max_strip_rows = std::max(C.max_strip_rows, rows);
    C.tiles.push_back(t);
  }
  // a shared-memory strip that cannot fit: stop here (the planner picks another tile width or
  // the global strip; the rest of the analysis would be discarded)
  if (strip_limit >= 0 && C.max_strip_rows > strip_limit) {
    C.too_big = true;
    return SC_OK;
  }

  // --- 5/6. SYRK groups (kGroup columns: union of the member tiles' panels), and per tile the
  // ordered factor panels it applies (steps), the strip rows of their pruned rows and the B~^T
  // scatter.  Strip rows are tile-local (shared-memory strip, written out into the group strip at
  // the end) or, for global strips, the rows of the group strip itself (solved in place).
  const int32_t ngroups = (m + kGroup - 1) / kGroup;
  int64_t xoff = 0;
  int32_t J0 = 0;
  std::vector<int32_t> gmark((size_t)np, -1);
  std::vector<int64_t> gsrow_off((size_t)np, -1);
  for (int32_t g = 0; g < ngroups; g++) {
    Group G{};
    G.col0 = g * kGroup;
    G.width = std::min(kGroup, m - g * kGroup);
    int32_t J1 = J0;
    while (J1 < ntiles && C.tiles[(size_t)J1].group == g) J1++;
    std::vector<int32_t> gp;
    for (int32_t J = J0; J < J1; J++) {
      std::vector<int32_t> u;
      std::set_union(gp.begin(), gp.end(), tile_panels[(size_t)J].begin(), tile_panels[(size_t)J].end(),
                     std::back_inserter(u));
      gp.swap(u);
    }
    G.reach_begin = (int32_t)C.greach.size();
    int32_t grows = 0;
    for (int32_t p : gp) {
      C.greach.push_back({p, grows});
      gmark[(size_t)p] = g;
      grows += C.panels[(size_t)p].kw;
    }
    G.reach_end = (int32_t)C.greach.size();
    G.strip_rows = grows;
    // global strip: one row map per (group, panel), shared by the group's tiles.  R_p rows outside
    // a tile's own reach but inside the group's receive exact-zero updates (Y vanishes on columns
    // outside the reach, whose L rows hit only reach rows), so mapping them is harmless.
    if (gstrip) {
      for (int32_t q = G.reach_begin; q < G.reach_end; q++) strip_base[(size_t)C.greach[(size_t)q].panel] = C.greach[(size_t)q].off;
      for (int32_t q = G.reach_begin; q < G.reach_end; q++) {
        const Panel& P = C.panels[(size_t)C.greach[(size_t)q].panel];
        gsrow_off[(size_t)C.greach[(size_t)q].panel] = (int64_t)C.srows.size();
        for (int32_t k = 0; k < P.nchunk * kChunk; k++) {
          uint16_t v = 0xFFFF;
          if (k < P.nR) {
            const int32_t r = C.Rrows[(size_t)(P.R_off + k)];
            const int32_t qq = panel_of_col[(size_t)r];
            if (gmark[(size_t)qq] == g) v = (uint16_t)(strip_base[(size_t)qq] + (r - C.panels[(size_t)qq].a));
          }
          C.srows.push_back(v);
        }
      }
    }
    G.x_off = xoff;
    xoff += (int64_t)grows * kGroup;
    for (int32_t J = J0; J < J1; J++) {
      Tile& t = C.tiles[(size_t)J];
      const auto& tp = tile_panels[(size_t)J];
      t.step_begin = (int32_t)C.steps.size();
      int32_t rows = 0;
      size_t q = (size_t)G.reach_begin;
      for (int32_t p : tp) {
        while (C.greach[q].panel != p) q++;
        strip_base[(size_t)p] = gstrip ? C.greach[q].off : rows;
        in_tile[(size_t)p] = J;
        C.steps.push_back({p, strip_base[(size_t)p], C.greach[q].off, 0, 0});
        const Panel& P = C.panels[(size_t)p];
        C.x_reach_doubles += (double)P.kw * T;
        if (warp) {  // 8x8 triangle blocks (I >= K) + 8-row blocks of R_p, k padded to 8
          const double kw8 = (P.kw + 7) / 8, nRB = (P.nR + 7) / 8;
          C.fl_trsm_exec += 2.0 * T * (32.0 * kw8 * (kw8 + 1) + 64.0 * nRB * kw8);
        } else {  // GEMM1 skips the zero blocks above the diagonal of inv(L_pp)
          C.fl_trsm_exec += 2.0 * T * P.kw4 * (0.5 * (double)P.kw4 + 4.0 + (double)P.nR);
        }
        rows += P.kw;
      }
      t.step_end = (int32_t)C.steps.size();
      // strip rows of each step's pruned rows R_p, 64 per chunk (0xFFFF: not in this tile's strip)
      for (int32_t s = t.step_begin; s < t.step_end; s++) {
        Step& st = C.steps[(size_t)s];
        const Panel& P = C.panels[(size_t)st.panel];
        if (gstrip) {
          st.srow_off = gsrow_off[(size_t)st.panel];
          continue;
        }
        st.srow_off = (int64_t)C.srows.size();
        for (int32_t k = 0; k < P.nchunk * kChunk; k++) {
          uint16_t v = 0xFFFF;
          if (k < P.nR) {
            const int32_t r = C.Rrows[(size_t)(P.R_off + k)];
            const int32_t qq = panel_of_col[(size_t)r];
            if (in_tile[(size_t)qq] == J) v = (uint16_t)(strip_base[(size_t)qq] + (r - C.panels[(size_t)qq].a));
          }
          C.srows.push_back(v);
        }
      }
      // global strips are zeroed over all rows of the group strip (rows outside this tile's reach
      // stay exactly zero in its columns)
      t.strip_rows = gstrip ? grows : rows;
      t.binit_begin = (int32_t)C.binit.size();
      for (int32_t a = t.col0; a < t.col0 + t.width; a++)
        for (auto& e : bcol[(size_t)C.sigma[(size_t)a]]) {
          const int32_t p = panel_of_col[(size_t)e.first];
          C.binit.push_back({strip_base[(size_t)p] + (e.first - C.panels[(size_t)p].a), a - t.col0, e.second});
        }
      t.binit_end = (int32_t)C.binit.size();
    }
    C.groups.push_back(G);
    J0 = J1;
  }
  C.x_doubles = xoff;
  if (std::getenv("SC_DEBUG_LIVE") && !gstrip) {
    // frontal-stack experiment: max rows live at once per tile, B injected upfront / at own step
    std::vector<int32_t> first((size_t)np), ownstep((size_t)np);
    double sum_up = 0, sum_own = 0, sum_all = 0;
    int mx_up = 0, mx_own = 0;
    for (auto& t : C.tiles) {
      if (t.step_end <= t.step_begin) continue;
      for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
        first[(size_t)C.steps[(size_t)s2].panel] = s2;
        ownstep[(size_t)C.steps[(size_t)s2].panel] = s2;
      }
      std::vector<int32_t> firstB = first;
      for (int32_t q = t.binit_begin; q < t.binit_end; q++) {
        // B entry row -> panel: find the step whose strip rows contain it
        const int32_t sr = C.binit[(size_t)q].strip_row;
        for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
          const Step& st = C.steps[(size_t)s2];
          if (sr >= st.strip_row && sr < st.strip_row + C.panels[(size_t)st.panel].kw) firstB[(size_t)st.panel] = t.step_begin;
        }
      }
      for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
        const Step& st = C.steps[(size_t)s2];
        const Panel& P = C.panels[(size_t)st.panel];
        for (int32_t k = 0; k < P.nR; k++) {
          const uint16_t v = C.srows[(size_t)(st.srow_off + k)];
          if (v == 0xFFFF) continue;
          for (int32_t s3 = s2; s3 < t.step_end; s3++) {
            const Step& st3 = C.steps[(size_t)s3];
            if (v >= st3.strip_row && v < st3.strip_row + C.panels[(size_t)st3.panel].kw) {
              first[(size_t)st3.panel] = std::min(first[(size_t)st3.panel], s2);
              firstB[(size_t)st3.panel] = std::min(firstB[(size_t)st3.panel], s2);
              break;
            }
          }
        }
      }
      int m_up = 0, m_own = 0;
      for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
        int l_up = 0, l_own = 0;
        for (int32_t s3 = t.step_begin; s3 < t.step_end; s3++) {
          const int32_t q = C.steps[(size_t)s3].panel;
          const int kw = C.panels[(size_t)q].kw;
          if (firstB[(size_t)q] <= s2 && s2 <= ownstep[(size_t)q]) l_up += kw;
          if (first[(size_t)q] <= s2 && s2 <= ownstep[(size_t)q]) l_own += kw;
        }
        m_up = std::max(m_up, l_up);
        m_own = std::max(m_own, l_own);
      }
      sum_up += m_up; sum_own += m_own; sum_all += t.strip_rows;
      mx_up = std::max(mx_up, m_up); mx_own = std::max(mx_own, m_own);
    }
    fprintf(stderr, "live rows: strip mean %.0f max %d | live(B upfront) mean %.0f max %d | live(B at own step) mean %.0f max %d\n",
            sum_all / C.tiles.size(), C.max_strip_rows, sum_up / C.tiles.size(), mx_up, sum_own / C.tiles.size(), mx_own);
  }
  if (std::getenv("SC_DEBUG_TILES")) {
    double st = 0, rows = 0, bytes = 0, flops = 0, nch = 0;
    int mxs = 0, mxr = 0;
    std::vector<int> kwh(9, 0);
    for (auto& t : C.tiles) {
      st += t.step_end - t.step_begin;
      mxs = std::max(mxs, t.step_end - t.step_begin);
      rows += t.strip_rows;
      mxr = std::max(mxr, t.strip_rows);
      for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
        const Panel& P = C.panels[(size_t)C.steps[(size_t)s2].panel];
        bytes += 8.0 * (P.ldD * P.kw4 + (P.nchunk ? ((P.nchunk - 1) * kLdC + P.ldLast) * P.kw4 : 0));
        flops += 2.0 * T * P.kw * (P.kw + P.nR);
        nch += P.nchunk;
        kwh[std::min(8, (P.kw + 7) / 8)]++;
      }
    }
    double pbytes = 0;
    for (auto& P : C.panels) pbytes += 8.0 * (P.ldD * P.kw4 + (P.nchunk ? ((P.nchunk - 1) * kLdC + P.ldLast) * P.kw4 : 0));
    const double nt = (double)C.tiles.size();
    fprintf(stderr, "tiles n=%d m=%d T=%d: %zu tiles, steps/tile %.1f (max %d), chunks/tile %.1f, strip rows %.0f (max %d), "
            "L block bytes/tile %.0f (panel buffer %.0f, reuse %.1f), flops/tile %.3g, kw/8 hist of steps",
            n, m, T, C.tiles.size(), st / nt, mxs, nch / nt, rows / nt, mxr, bytes / nt, pbytes, bytes / pbytes, flops / nt);
    for (int h : kwh) fprintf(stderr, " %d", h);
    fprintf(stderr, "\n");
    std::vector<int> vh(12, 0), rh(20, 0);
    for (auto& t : C.tiles)
      for (int32_t s2 = t.step_begin; s2 < t.step_end; s2++) {
        const Panel& P = C.panels[(size_t)C.steps[(size_t)s2].panel];
        const int kw8 = (P.kw + 7) / 8, nRB = (P.nR + 7) / 8;
        vh[std::min(11, (kw8 * (kw8 + 1) + nRB * 2 * kw8) / 8)]++;
        rh[std::min(19, nRB)]++;
      }
    fprintf(stderr, "  values/lane per step (x8) hist:");
    for (int h : vh) fprintf(stderr, " %d", h);
    fprintf(stderr, "\n  nRB hist:");
    for (int h : rh) fprintf(stderr, " %d", h);
    fprintf(stderr, "\n");
  }
  if (std::getenv("SC_DEBUG_PLAN"))
    fprintf(stderr, "class n=%d m=%d T=%d gstrip=%d: panels %d tiles %zu steps %zu srows %zu Rrows %zu greach %zu binit %zu\n",
            n, m, T, (int)gstrip, np, C.tiles.size(), C.steps.size(), C.srows.size(), C.Rrows.size(), C.greach.size(),
            C.binit.size());

  // --- 6. SYRK output tiles I >= J over groups with their common-row segments
  for (int32_t I = 0; I < ngroups; I++)
    for (int32_t J = 0; J <= I; J++) {
      const Group &gi = C.groups[(size_t)I], &gj = C.groups[(size_t)J];
      Pair pr{I, J, (int32_t)C.segs.size(), 0};
      int32_t qi = gi.reach_begin, qj = gj.reach_begin;
      int64_t K = 0;
      while (qi < gi.reach_end && qj < gj.reach_end) {
        const Reach &a = C.greach[(size_t)qi], &b = C.greach[(size_t)qj];
        if (a.panel < b.panel) {
          qi++;
          continue;
        }
        if (b.panel < a.panel) {
          qj++;
          continue;
        }
        const Panel& Pp = C.panels[(size_t)a.panel];
        // runs of rows reached by both groups (whole panel without row-level reach)
        for (int32_t r = 0; r < Pp.kw;) {
          if (row_reach && !(grow_reach[(size_t)I][(size_t)(Pp.a + r)] && grow_reach[(size_t)J][(size_t)(Pp.a + r)])) {
            r++;
            continue;
          }
          int32_t e = r + 1;
          while (e < Pp.kw && (!row_reach || (grow_reach[(size_t)I][(size_t)(Pp.a + e)] &&
                                              grow_reach[(size_t)J][(size_t)(Pp.a + e)])))
            e++;
          const int32_t len = e - r, oi = a.off + r, oj = b.off + r;
          K += len;
          Seg* last = (int32_t)C.segs.size() > pr.seg_begin ? &C.segs.back() : nullptr;
          if (last && last->offI + last->len == oi && last->offJ + last->len == oj)
            last->len += len;
          else
            C.segs.push_back({oi, oj, len, 0});
          r = e;
        }
        qi++;
        qj++;
      }
      pr.seg_end = (int32_t)C.segs.size();
      if (pr.seg_end > pr.seg_begin) {
        C.pairs.push_back(pr);
        C.fl_syrk_exec += 2.0 * kGroup * kGroup * (double)K;
      }
    }
  return SC_OK;
}

}  // namespace

sc_status build_plan(const sc_subdomain_desc* sd, int32_t nsub, const sc_options& opt, Plan& P, std::string& err) {
  if (nsub < 0 || (nsub > 0 && !sd)) FAIL(SC_ERR_INVALID_ARG, "sd is NULL or nsub < 0");
  if (opt.precision != 64 && opt.precision != 32) FAIL(SC_ERR_INVALID_ARG, "precision must be 64 or 32");
  P.esz = opt.precision == 32 ? 4 : 8;
  if (opt.skip < 0 || opt.skip > 2) FAIL(SC_ERR_INVALID_ARG, "skip must be 0, 1 or 2");
  if (!(opt.tile_cols == 0 || opt.tile_cols == 8 || opt.tile_cols == 16 || opt.tile_cols == 32 || opt.tile_cols == 64))
    FAIL(SC_ERR_INVALID_ARG, "tile_cols must be 0, 8, 16, 32 or 64");
  if (opt.panel_cols < 0 || opt.panel_cols > kMaxPanel) FAIL(SC_ERR_INVALID_ARG, "panel_cols must be in [0, 64]");
  if (opt.x_strip < 0 || opt.x_strip > 2) FAIL(SC_ERR_INVALID_ARG, "x_strip must be 0, 1 or 2");
  for (int k = 0; k < 5; k++)
    if (opt.reserved[k] != 0) FAIL(SC_ERR_INVALID_ARG, "reserved options must be zero");
  P.opt = opt;
  P.nsub = nsub;
  P.n_lambda = opt.n_lambda_global;
  for (int32_t i = 0; i < nsub; i++) {
    sc_status st = validate_desc(sd[i], i, err);
    if (st != SC_OK) return st;
    if (sd[i].lambda_map)
      for (int32_t a = 0; a < sd[i].m; a++)
        if (sd[i].lambda_map[a] < 0 || sd[i].lambda_map[a] >= opt.n_lambda_global)
          FAIL(SC_ERR_INVALID_ARG, "subdomain " + std::to_string(i) + ": lambda_map entry outside [0, n_lambda_global)");
  }

  // --- classes (dedup identical patterns); the TRSM tile width is chosen so the largest X strip
  // fits in shared memory (T = 32 when possible, else 16; tile_cols forces a width)
  std::unordered_map<uint64_t, std::vector<int32_t>> by_hash;
  std::vector<int32_t> rep;  // representative subdomain of each class
  P.sub_cls.assign((size_t)nsub, -1);
  for (int32_t i = 0; i < nsub; i++) {
    uint64_t h = desc_hash(sd[i]);
    auto& cands = by_hash[h];
    int32_t cls = -1;
    for (int32_t c : cands)
      if (same_pattern(sd[rep[(size_t)c]], sd[i])) {
        cls = c;
        break;
      }
    if (cls < 0) {
      cls = (int32_t)P.classes.size();
      P.classes.emplace_back();
      P.classes.back().hash = h;
      rep.push_back(i);
      cands.push_back(cls);
    }
    P.sub_cls[(size_t)i] = cls;
  }
  // SYRK output tile (group) width: 64 for large local operators (CTA per 64 x 64 tile); 16 for small
  // ones (warp per 16 x 16 tile: the k range of each tile restricted at 16-column granularity, 1.35x
  // instead of 1.94x the useful flops on cfg2, tile-exact X strips); never below T
  int32_t max_m = 0;
  for (int32_t i = 0; i < nsub; i++) max_m = std::max(max_m, sd[i].m);
  int32_t G0 = max_m > 512 ? 64 : 16;
  // factor panel width: 64 for large operators (3D: wide separators, DMMA-bound); 32 for small ones
  // (2D: narrow supernodes, latency-bound; narrower L blocks leave shared memory for T = 32 strips)
  P.PW = opt.panel_cols ? opt.panel_cols : (max_m > 512 ? kMaxPanel : 32);
  // TRSM update operand: Y mode (default: L[R_p,p] times the solved panel Y, exchanged through
  // shared memory within each column-block group) or W mode (W_p = L[R_p,p] inv(L_pp) prepared once
  // per subdomain in prep: no intra-step barrier, but the prep transform costs more than the
  // barrier saves: cfg2-5 measured equal or slower in total, e.g. cfg4 3649 vs 3730 subdomains/s)
  P.wmode = false;
  if (const char* e = std::getenv("SC_OVERLAP")) P.overlap = std::atoi(e);
  if (const char* e = std::getenv("SC_TRSM_MODE")) P.wmode = e[0] == 'W';
  if (const char* e = std::getenv("SC_SYRK_SPLIT")) P.syrk_input = e[0] == 'i';
  if (P.esz == 4 && P.wmode) FAIL(SC_ERR_INVALID_ARG, "precision 32 supports the Y-mode TRSM only");
  if (const char* e = std::getenv("SC_GROUP")) G0 = std::atoi(e);
  if (!(G0 == 16 || G0 == 32 || G0 == 64)) FAIL(SC_ERR_INVALID_ARG, "SC_GROUP must be 16, 32 or 64");
  // classes are independent: analysed on all host cores
  bool warp = false;  // analyse for the warp TRSM (fragment gather maps)
  auto analyse_all = [&](int T, bool gstrip, int32_t strip_limit) -> sc_status {
    P.T = T;
    P.G = std::max(G0, T);
    P.gstrip = gstrip;
    const size_t nc = P.classes.size();
    std::vector<sc_status> st(nc, SC_OK);
    std::vector<std::string> errs(nc);
    std::atomic<size_t> next{0};
    auto work = [&]() {
      for (size_t c = next++; c < nc; c = next++) {
        uint64_t h = P.classes[c].hash;
        P.classes[c] = ClassPlan();
        P.classes[c].hash = h;
        st[c] = analyse_class(sd[rep[c]], T, P.G, P.PW, opt.skip, gstrip, strip_limit, warp, P.classes[c], errs[c]);
      }
    };
    const size_t nthr = std::min<size_t>(nc, std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (size_t k = 1; k < nthr; k++) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (size_t c = 0; c < nc; c++)
      if (st[c] != SC_OK) {
        err = "subdomain " + std::to_string(rep[c]) + ": " + errs[c];
        return st[c];
      }
    return SC_OK;
  };
  auto too_big = [&]() {
    for (auto& C : P.classes)
      if (C.too_big) return true;
    return false;
  };
  // largest shared-memory strip (rows) that fits next to a ring of two of the largest L blocks a
  // panel width of PW can produce
  auto strip_limit_for = [&](int T) -> int32_t {
    const int64_t kw4 = (P.PW + 3) & ~3;
    const int64_t maxblk = std::max<int64_t>(block_ld(P.PW), kLdC) * kw4 * 8;
    const int64_t fixed = (int64_t)trsm_smem_layout(T, (int)(2 * maxblk), 0, false, !P.wmode).total;
    return (int32_t)std::max<int64_t>(-1, ((int64_t)kSmemBudget - fixed) / (8 * strip_ld(T)));
  };
  // TRSM tile width: the widest of 32 / 16 / 8 whose largest X strip fits in shared memory next to
  // an L-block ring of at least two of the plan's largest blocks; the ring gets what is left (up
  // to 160 KB) so the producer can run ahead.  A global strip (solved in place in the group strip,
  // through L2) needs no strip space: the ring gets up to 160 KB.
  auto ring_for = [&](int T) -> int64_t {
    int32_t mx = 0;
    int64_t maxblk = 16;
    for (auto& C : P.classes) {
      mx = std::max(mx, C.max_strip_rows);
      for (auto& p : C.panels) {
        maxblk = std::max<int64_t>(maxblk, (int64_t)p.ldD * p.kw4 * 8);
        if (p.nchunk > 0) maxblk = std::max<int64_t>(maxblk, (int64_t)(p.nchunk > 1 ? kLdC : p.ldLast) * p.kw4 * 8);
      }
    }
    const int64_t fixed = (int64_t)trsm_smem_layout(T, 0, mx, P.gstrip, !P.wmode).total;
    int64_t ring = std::min<int64_t>(kRingMaxBytes, (int64_t)kSmemBudget - fixed) & ~(int64_t)127;
    return ring >= 2 * maxblk ? ring : -1;
  };
  // two-CTAs-per-SM budget for tile width T (after an analysis at T): strip rows that fit next to a
  // ring of max(2 largest L blocks, 32 KB) in half an SM, and how many tiles qualify
  struct TwoCta {
    int32_t rmax = 0, fit_max = 0;
    int64_t n_all = 0, n_fit = 0, half = 0;
  };
  auto two_cta = [&](int T) -> TwoCta {
    TwoCta r;
    int64_t maxblk = 16;
    for (auto& C : P.classes)
      for (auto& p : C.panels) {
        maxblk = std::max<int64_t>(maxblk, (int64_t)p.ldD * p.kw4 * 8);
        if (p.nchunk > 0) maxblk = std::max<int64_t>(maxblk, (int64_t)(p.nchunk > 1 ? kLdC : p.ldLast) * p.kw4 * 8);
      }
    const int64_t ring_min = (std::max<int64_t>(2 * maxblk, 32768) + 127) & ~(int64_t)127;
    r.half = kSmemPerSM / 2 - 1024;  // per-CTA reservation
    const int64_t fixed = (int64_t)trsm_smem_layout(T, (int)ring_min, 0, false, !P.wmode).total;
    r.rmax = (int32_t)((r.half - fixed) / (8 * strip_ld(T)));
    for (auto& C : P.classes)
      for (auto& t : C.tiles)
        if (t.width > 0) {
          r.n_all++;
          if (t.strip_rows <= r.rmax) {
            r.n_fit++;
            r.fit_max = std::max(r.fit_max, t.strip_rows);
          }
        }
    return r;
  };
  // global-strip tile width: 32 (measured on cfg4 / cfg5: 16 and 64 are slower)
  const int Tg = opt.tile_cols ? opt.tile_cols : 32;
  // warp TRSM (one warp per tile, fragments straight from the CSC values, no prep): small operators
  // (2D) with narrow panels; tiles of 8 or 16 columns solved in place in the group strips
  if (opt.trsm_kernel < 0 || opt.trsm_kernel > 2) FAIL(SC_ERR_INVALID_ARG, "trsm_kernel must be 0, 1 or 2");
  warp = opt.trsm_kernel == SC_TRSM_WARP ||
         (opt.trsm_kernel == SC_TRSM_AUTO && max_m <= 512 && P.PW <= 32 && !P.wmode &&
          (opt.tile_cols == 0 || opt.tile_cols <= 16) && opt.x_strip != SC_STRIP_SHARED && !std::getenv("SC_NO_WARP"));
  if (warp) {
    if (P.PW > 32) FAIL(SC_ERR_INVALID_ARG, "warp TRSM needs panel_cols <= 32");
    if (opt.x_strip == SC_STRIP_SHARED) FAIL(SC_ERR_INVALID_ARG, "warp TRSM solves in the global strips");
    int Tw = opt.tile_cols;
    if (!Tw) {
      const char* e = std::getenv("SC_WARP_T");
      Tw = e ? std::atoi(e) : 16;
    }
    if (!(Tw == 8 || Tw == 16)) FAIL(SC_ERR_INVALID_ARG, "warp TRSM needs tile_cols 8 or 16");
    P.wmode = false;
    sc_status st = analyse_all(Tw, true, -1);
    if (st != SC_OK) return st;
    P.warp_trsm = true;
  } else if (opt.x_strip == SC_STRIP_GLOBAL) {
    sc_status st = analyse_all(Tg, true, -1);
    if (st != SC_OK) return st;
  } else {
    // automatic: a shared-memory strip of 32 or 16 columns if it fits, else (AUTO) the global strip
    // at T = 32, which beats a shared strip of only 8 columns (cfg4: TRSM 67 vs 81 ms); an explicit
    // SC_STRIP_SHARED request still falls back to T = 8
    const int cand_auto[3] = {32, 16, 8};
    const int* cand = opt.tile_cols ? &opt.tile_cols : cand_auto;
    const int ncand = opt.tile_cols ? 1 : (opt.x_strip == SC_STRIP_SHARED ? 3 : 2);
    bool fits = false;
    // large operators (3D): global strips at T = 16, two CTAs per SM (see gs2 below)
    if (!opt.tile_cols && max_m > 512 && opt.x_strip == SC_STRIP_AUTO) {
      sc_status st = analyse_all(16, true, -1);
      if (st != SC_OK) return st;
      fits = true;
      P.gstrip = true;
    }
    // small operators (2D): T = 16 at two CTAs per SM beats T = 32 at one when most tiles' strips
    // fit in half an SM (cfg2 TRSM 1.72 vs 2.01 ms)
    if (!fits && !opt.tile_cols && max_m <= 512) {
      sc_status st = analyse_all(16, false, strip_limit_for(16));
      if (st != SC_OK) return st;
      if (!too_big() && ring_for(16) > 0) {
        const TwoCta tc = two_cta(16);
        fits = tc.rmax > 0 && tc.n_fit * 2 >= tc.n_all;
      }
    }
    for (int k = 0; k < ncand && !fits; k++) {
      // SC_STRIP_SHARED with an explicit tile width analyses fully and reports the misfit below
      const bool force = opt.x_strip == SC_STRIP_SHARED && opt.tile_cols;
      sc_status st = analyse_all(cand[k], false, force ? -1 : strip_limit_for(cand[k]));
      if (st != SC_OK) return st;
      fits = !too_big() && ring_for(cand[k]) > 0;
    }
    if (!fits && opt.x_strip == SC_STRIP_AUTO) {
      sc_status st = analyse_all(Tg, true, -1);
      if (st != SC_OK) return st;
    } else if (!fits) {
      sc_status st = analyse_all(cand[ncand - 1], false, -1);  // full analysis for the error report
      if (st != SC_OK) return st;
    }
  }
  for (auto& C : P.classes) P.max_strip_rows = std::max(P.max_strip_rows, C.max_strip_rows);
  P.ring_bytes = (int32_t)std::max<int64_t>(ring_for(P.T), 0);
  // global strips at T = 16 run two CTAs per SM (4 consumer warps each; measured: cfg3 TRSM 12.6 vs
  // 13.7 ms with shared strips, cfg4 51.8 vs 54.5 ms at T = 32, cfg5 324 vs 339 ms); SC_GS2=0 disables
  const char* gs2_env = std::getenv("SC_GS2");
  if (P.warp_trsm) P.ring_bytes = 0;
  if (P.gstrip && !P.warp_trsm && P.T == 16 && !(gs2_env && gs2_env[0] == '0')) {  // ring within 1/ctas of an SM
    int64_t maxblk = 16;
    for (auto& C : P.classes)
      for (auto& p : C.panels) {
        maxblk = std::max<int64_t>(maxblk, (int64_t)p.ldD * p.kw4 * 8);
        if (p.nchunk > 0) maxblk = std::max<int64_t>(maxblk, (int64_t)(p.nchunk > 1 ? kLdC : p.ldLast) * p.kw4 * 8);
      }
    const int64_t fixed = (int64_t)trsm_smem_layout(16, 0, 0, true, !P.wmode).total;
    // 3 CTAs per SM only when the ring still holds two of the largest L blocks (double buffering)
    const int want = (gs2_env && gs2_env[0] == '3') ? 3 : 2;
    P.gs2 = 2;
    if (want == 3 && ((kSmemPerSM / 3 - 1024 - fixed) & ~(int64_t)127) >= 2 * maxblk) P.gs2 = 3;
    const int64_t share = kSmemPerSM / P.gs2 - 1024;
    P.ring_bytes = (int32_t)(std::min<int64_t>(P.ring_bytes, share - fixed) & ~(int64_t)127);
  }
  // small-strip tile class (shared strips): tiles whose strip fits next to a ring of >= 2 of the
  // largest L blocks (and >= 32 KB) within half of the SM's shared memory run two CTAs per SM
  // (T <= 16 only: the register cap of two 288-thread CTAs per SM makes wider tiles spill)
  int32_t split_rows = 0;
  bool want_split = true;
  if (const char* e = std::getenv("SC_TRSM_SPLIT")) want_split = std::atoi(e) != 0;
  if (!P.gstrip && !P.warp_trsm && want_split && P.T <= 16) {
    TwoCta tc = two_cta(P.T);
    if (const char* e = std::getenv("SC_TRSM_SPLIT_ROWS")) {  // test hook: force the class boundary
      const int32_t r = std::min(tc.rmax, (int32_t)std::atoi(e));
      tc.n_fit = 0;
      tc.fit_max = 0;
      for (auto& C : P.classes)
        for (auto& t : C.tiles)
          if (t.width > 0 && t.strip_rows <= r) {
            tc.n_fit++;
            tc.fit_max = std::max(tc.fit_max, t.strip_rows);
          }
      tc.n_all = 2 * tc.n_fit;  // accept
      if (tc.n_fit == 0) tc.rmax = 0;
    }
    if (tc.rmax > 0 && tc.n_fit * 2 >= tc.n_all) {  // (all tiles fitting: one launch at two CTAs per SM)
      split_rows = tc.fit_max;
      P.strip_small = tc.fit_max;
      P.ring_small =
          (int32_t)((tc.half - (int64_t)trsm_smem_layout(P.T, 0, tc.fit_max, false, !P.wmode).total) & ~(int64_t)127);
    }
  }

  // --- global concatenation: class-local indices -> global
  int64_t srow_base = 0;
  int32_t tile_base = 0, step_base = 0, binit_base = 0, seg_base = 0, R_base = 0, pair_base = 0, panel_base = 0,
          group_base = 0, greach_base = 0;
  for (auto& C : P.classes) {
    P.cls_tile_begin.push_back(tile_base);
    P.cls_pair_begin.push_back(pair_base);
    P.cls_panel_begin.push_back(panel_base);
    P.cls_group_begin.push_back(group_base);
    for (auto& p : C.panels) p.R_off += R_base;
    for (auto& s : C.steps) {
      s.panel += panel_base;
      s.srow_off += srow_base;
    }
    for (auto& r : C.greach) r.panel += panel_base;
    for (auto& t : C.tiles) {
      t.step_begin += step_base;
      t.step_end += step_base;
      t.binit_begin += binit_base;
      t.binit_end += binit_base;
      t.group += group_base;
    }
    for (auto& g : C.groups) {
      g.reach_begin += greach_base;
      g.reach_end += greach_base;
    }
    for (auto& p : C.pairs) {
      p.I += group_base;
      p.J += group_base;
      p.seg_begin += seg_base;
      p.seg_end += seg_base;
    }
    tile_base += (int32_t)C.tiles.size();
    step_base += (int32_t)C.steps.size();
    binit_base += (int32_t)C.binit.size();
    seg_base += (int32_t)C.segs.size();
    R_base += (int32_t)C.Rrows.size();
    pair_base += (int32_t)C.pairs.size();
    panel_base += (int32_t)C.panels.size();
    group_base += (int32_t)C.groups.size();
    greach_base += (int32_t)C.greach.size();
    srow_base += (int64_t)C.srows.size();
  }

  // --- per subdomain layout + task lists
  P.sub_m.resize((size_t)nsub);
  P.sub_n.resize((size_t)nsub);
  P.sub_nnz.resize((size_t)nsub);
  sc_stats& S = P.stats;
  std::memset(&S, 0, sizeof(S));
  S.nsub = nsub;
  S.n_classes = (int32_t)P.classes.size();
  S.tile_cols = P.T;
  S.panel_cols = P.PW;
  std::vector<int64_t> qcount((size_t)std::max<int64_t>(opt.n_lambda_global, 0) + 1, 0);
  std::vector<I2> small_bkt[3];
  std::vector<I2> trsm_small;
  for (int32_t i = 0; i < nsub; i++) {
    const int32_t cls = P.sub_cls[(size_t)i];
    const ClassPlan& C = P.classes[(size_t)cls];
    P.sub_m[(size_t)i] = C.m;
    P.sub_n[(size_t)i] = C.n;
    P.sub_nnz[(size_t)i] = C.colptr[(size_t)C.n];
    P.max_n = std::max(P.max_n, C.n);
    P.sub_X_base.push_back(P.X_doubles);
    P.X_doubles += C.x_doubles;
    P.sub_F_base.push_back(P.F_doubles);
    P.F_doubles += f_tiles(C.m) * kApplyTile * kApplyTile;
    P.sub_PB_base.push_back(P.PB_doubles);
    P.PB_doubles += C.pb_doubles;
    P.sub_part_off.push_back(P.part_doubles);
    const int32_t nab = (C.m + kApplyTile - 1) / kApplyTile;  // apply tiles: nab (nab + 1) / 2
    P.part_doubles += (int64_t)nab * (nab + 1) / 2 * 2 * kApplyTile;
    for (size_t q = 0; q < C.panels.size(); q++) {
      const I2 tk{i, P.cls_panel_begin[(size_t)cls] + (int32_t)q};
      const int32_t kw = C.panels[q].kw;
      if (kw > kSmallPanel) P.prep_tasks.push_back(tk);
      else small_bkt[kw <= 8 ? 0 : (kw <= 16 ? 1 : 2)].push_back(tk);
    }
    for (size_t t = 0; t < C.tiles.size(); t++)
      if (C.tiles[t].width > 0)
        (split_rows > 0 && C.tiles[t].strip_rows <= split_rows ? trsm_small : P.trsm_tasks)
            .push_back({i, P.cls_tile_begin[(size_t)cls] + (int32_t)t});
    for (size_t q = 0; q < C.pairs.size(); q++) P.syrk_tasks.push_back({i, P.cls_pair_begin[(size_t)cls] + (int32_t)q});
    for (int32_t rb = 0; rb < nab; rb++)
      for (int32_t cb = 0; cb <= rb; cb++) P.apply_tasks.push_back({i, rb, cb, 0});
    P.sub_slm_off.push_back((int64_t)P.slm.size());
    P.ssig.insert(P.ssig.end(), C.sigma.begin(), C.sigma.end());
    if (sd[i].lambda_map) {
      for (int32_t a = 0; a < C.m; a++) {
        int64_t g = sd[i].lambda_map[C.sigma[(size_t)a]];
        P.slm.push_back(g);
        qcount[(size_t)g]++;
      }
    } else {
      for (int32_t a = 0; a < C.m; a++) P.slm.push_back(0);
    }
    S.sum_n += C.n;
    S.sum_m += C.m;
    S.max_m = std::max<int64_t>(S.max_m, C.m);
    S.sum_nnz_L += C.colptr[(size_t)C.n];
    S.flops_trsm_useful += C.fl_trsm_useful;
    S.flops_syrk_useful += C.fl_syrk_useful;
    S.flops_trsm_envelope += C.fl_trsm_env;
    S.flops_syrk_envelope += C.fl_syrk_env;
    S.flops_trsm_dense += C.fl_trsm_dense;
    S.flops_syrk_dense += C.fl_syrk_dense;
    S.flops_trsm_sparse_orig += C.fl_trsm_sparse;
    S.flops_trsm_executed += C.fl_trsm_exec;
    S.flops_syrk_executed += C.fl_syrk_exec;
    S.bytes_L_values += 8.0 * (double)C.colptr[(size_t)C.n];
    S.bytes_F_lower += 8.0 * (double)C.m * (C.m + 1) / 2.0;
    S.trsm_steps += (int64_t)C.steps.size();
    S.syrk_segments += (int64_t)C.segs.size();
    S.bytes_apply += 8.0 * (double)C.m * (C.m + 1) / 2.0 + 8.0 * 3.0 * C.m;
    S.bytes_panels += 8.0 * (double)C.pb_doubles;
    S.bytes_X_reach += 8.0 * C.x_reach_doubles;
    S.panels += (int64_t)C.panels.size();
  }
  P.ntrsm_small = (int32_t)trsm_small.size();
  P.trsm_tasks.insert(P.trsm_tasks.begin(), trsm_small.begin(), trsm_small.end());
  for (int b = 0; b < 3; b++) {
    P.small_begin[b] = (int32_t)P.prep_small_tasks.size();
    P.prep_small_tasks.insert(P.prep_small_tasks.end(), small_bkt[b].begin(), small_bkt[b].end());
  }
  P.small_begin[3] = (int32_t)P.prep_small_tasks.size();
  S.group_cols = P.G;
  S.x_strip = P.gstrip ? SC_STRIP_GLOBAL : SC_STRIP_SHARED;
  S.trsm_tasks = (int64_t)P.trsm_tasks.size();
  S.trsm_tasks_2cta = P.ntrsm_small;
  S.trsm_kernel = P.warp_trsm ? SC_TRSM_WARP : SC_TRSM_CTA;
  S.syrk_tasks = (int64_t)P.syrk_tasks.size();
  S.bytes_X = 8.0 * (double)P.X_doubles;
  // CSR over global multipliers of the (sub, stepped position) contributions, in (sub, a) order
  const int64_t NL = std::max<int64_t>(opt.n_lambda_global, 0);
  P.qg_ptr.assign((size_t)NL + 1, 0);
  for (int64_t g = 0; g < NL; g++) P.qg_ptr[(size_t)g + 1] = P.qg_ptr[(size_t)g] + qcount[(size_t)g];
  P.qg_sub_a.assign((size_t)P.qg_ptr[(size_t)NL], 0);
  std::vector<int64_t> fillpos(P.qg_ptr.begin(), P.qg_ptr.begin() + NL);
  for (int32_t i = 0; i < nsub; i++) {
    if (!sd[i].lambda_map) continue;
    const ClassPlan& C = P.classes[(size_t)P.sub_cls[(size_t)i]];
    for (int32_t a = 0; a < C.m; a++) {
      int64_t g = P.slm[(size_t)(P.sub_slm_off[(size_t)i] + a)];
      P.qg_sub_a[(size_t)fillpos[(size_t)g]++] = ((int64_t)i << 32) | (int64_t)a;
    }
  }
  return SC_OK;
}

}  // namespace sc
