// plan.cpp — "initialization" stage: host-only integer symbolic analysis.
//
// Per pattern class (subdomains with identical L pattern, perm and B~^T):
//   1. validate L (lower CSC, diagonal first, rows ascending) and that its pattern is a Cholesky fill
//      pattern (closed under the elimination tree), B~^T rows, perm;
//   2. elimination tree parent(j) = first sub-diagonal row of column j, maximal supernodes (chains
//      j -> j+1 with equal row structure below), their pruned row structures R_s ("extract
//      only the non-empty rows", CHOLMOD-like);
//   3. row-permute B~^T by perm, column pivots p_j (first non-zero), stepped order sigma =
//      stable sort by (p_j, j) (ties: SURVEY §8.3 reading 7);
//   4. RHS column tiles of width T and, per tile, the rows its X strip must hold:
//        exact    : elimination-tree reach of the tile's B~^T non-zeros (zeros above the pivots and
//                   off the etree paths are preserved),
//        envelope : every row >= the tile's highest (smallest) pivot (the paper's stepped envelope),
//        none     : every row (the original algorithm);
//   5. per tile the ordered factor panels ("factor splitting") it must apply;
//   6. SYRK output tiles I >= J with the row segments both strips hold (output splitting with the
//      k range restricted to non-zero rows);
//   7. work counters and memory layout.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <numeric>
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
sc_status analyse_class(const sc_subdomain_desc& d, int T, int PW, int skip, ClassPlan& C, std::string& err) {
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

  // --- 2. etree + closure check + supernodes
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
  std::vector<int32_t> snode_of((size_t)n);
  for (int32_t c = 0; c < n;) {
    int32_t c0 = c;
    c++;
    while (c < n && parent[(size_t)(c - 1)] == c && cc(c - 1) == cc(c) + 1) c++;
    int32_t s = (int32_t)C.sn_c0.size();
    C.sn_c0.push_back(c0);
    C.sn_c1.push_back(c);
    int32_t last = c - 1;
    int32_t nR = cc(last) - 1;
    C.sn_nR.push_back(nR);
    C.sn_Roff.push_back((int32_t)C.Rrows.size());
    for (int64_t q = cp[last] + 1; q < cp[last + 1]; q++) C.Rrows.push_back(ri[q]);
    for (int32_t k = c0; k < c; k++) snode_of[(size_t)k] = s;
  }
  C.nsup = (int32_t)C.sn_c0.size();

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

  // --- 4/5. tiles, reach, panel steps, B scatter
  const int32_t ntiles = (m + T - 1) / T;
  std::vector<int32_t> entry((size_t)C.nsup, INT32_MAX);
  std::vector<int32_t> strip_base((size_t)C.nsup, -1);
  int64_t xoff = 0;
  for (int32_t J = 0; J < ntiles; J++) {
    Tile t{};
    t.col0 = J * T;
    t.width = std::min(T, m - J * T);
    std::fill(entry.begin(), entry.end(), INT32_MAX);
    int32_t pmin = n;
    for (int32_t a = t.col0; a < t.col0 + t.width; a++) pmin = std::min(pmin, C.pivot[(size_t)a]);
    if (skip == SC_SKIP_EXACT) {
      for (int32_t a = t.col0; a < t.col0 + t.width; a++)
        for (auto& e : bcol[(size_t)C.sigma[(size_t)a]]) {
          int32_t cur = e.first;
          while (true) {
            int32_t s = snode_of[(size_t)cur];
            if (entry[(size_t)s] <= cur) break;
            entry[(size_t)s] = cur;
            if (C.sn_nR[(size_t)s] == 0) break;
            cur = C.Rrows[(size_t)C.sn_Roff[(size_t)s]];
          }
        }
    } else if (pmin < n) {
      int32_t from = (skip == SC_SKIP_ENVELOPE) ? pmin : 0;
      for (int32_t s = 0; s < C.nsup; s++)
        if (C.sn_c1[(size_t)s] > from) entry[(size_t)s] = std::max(C.sn_c0[(size_t)s], from);
    }
    t.reach_begin = (int32_t)C.reach.size();
    t.step_begin = (int32_t)C.steps.size();
    int32_t rows = 0;
    for (int32_t s = 0; s < C.nsup; s++) {
      if (entry[(size_t)s] == INT32_MAX) {
        strip_base[(size_t)s] = -1;
        continue;
      }
      int32_t e = entry[(size_t)s], c1 = C.sn_c1[(size_t)s];
      C.reach.push_back({s, e, c1, rows});
      strip_base[(size_t)s] = rows;
      for (int32_t a = e; a < c1; a += PW) {
        Step st{};
        st.e = a;
        st.kw = std::min(PW, c1 - a);
        st.c1 = c1;
        st.nR = C.sn_nR[(size_t)s];
        st.R_off = C.sn_Roff[(size_t)s];
        st.strip_row = rows + (a - e);
        C.steps.push_back(st);
        int64_t M = (int64_t)(c1 - a - st.kw) + st.nR;
        C.fl_trsm_exec += (double)T * st.kw * ((double)st.kw + 2.0 * (double)M);
      }
      rows += c1 - e;
    }
    t.reach_end = (int32_t)C.reach.size();
    t.step_end = (int32_t)C.steps.size();
    t.strip_rows = rows;
    t.binit_begin = (int32_t)C.binit.size();
    for (int32_t a = t.col0; a < t.col0 + t.width; a++)
      for (auto& e : bcol[(size_t)C.sigma[(size_t)a]]) {
        int32_t s = snode_of[(size_t)e.first];
        int32_t sr = strip_base[(size_t)s] + (e.first - entry[(size_t)s]);
        C.binit.push_back({sr, a - t.col0, e.second});
      }
    t.binit_end = (int32_t)C.binit.size();
    t.x_off = xoff;
    xoff += (int64_t)rows * T;
    C.tiles.push_back(t);
  }
  C.x_doubles = xoff;

  // --- 6. SYRK output tiles I >= J with their common-row segments
  for (int32_t I = 0; I < ntiles; I++)
    for (int32_t J = 0; J <= I; J++) {
      const Tile &ti = C.tiles[(size_t)I], &tj = C.tiles[(size_t)J];
      Pair pr{I, J, (int32_t)C.segs.size(), 0};
      int32_t qi = ti.reach_begin, qj = tj.reach_begin;
      int64_t K = 0;
      while (qi < ti.reach_end && qj < tj.reach_end) {
        const Reach &ri_ = C.reach[(size_t)qi], &rj = C.reach[(size_t)qj];
        if (ri_.s < rj.s) {
          qi++;
          continue;
        }
        if (rj.s < ri_.s) {
          qj++;
          continue;
        }
        int32_t start = std::max(ri_.e, rj.e);
        int32_t len = ri_.c1 - start;
        int32_t oi = ri_.off + (start - ri_.e), oj = rj.off + (start - rj.e);
        if (len > 0) {
          if ((int32_t)C.segs.size() > pr.seg_begin) {
            Seg& last = C.segs.back();
            if (last.offI + last.len == oi && last.offJ + last.len == oj) {
              last.len += len;
              K += len;
              qi++;
              qj++;
              continue;
            }
          }
          C.segs.push_back({oi, oj, len, 0});
          K += len;
        }
        qi++;
        qj++;
      }
      pr.seg_end = (int32_t)C.segs.size();
      if (pr.seg_end > pr.seg_begin) {
        C.pairs.push_back(pr);
        C.fl_syrk_exec += 2.0 * T * T * (double)K;
      }
    }
  return SC_OK;
}

}  // namespace

sc_status build_plan(const sc_subdomain_desc* sd, int32_t nsub, const sc_options& opt, Plan& P, std::string& err) {
  if (nsub < 0 || (nsub > 0 && !sd)) FAIL(SC_ERR_INVALID_ARG, "sd is NULL or nsub < 0");
  if (opt.precision != 64) FAIL(SC_ERR_INVALID_ARG, "only precision = 64 (FP64) is supported");
  if (opt.skip < 0 || opt.skip > 2) FAIL(SC_ERR_INVALID_ARG, "skip must be 0, 1 or 2");
  if (!(opt.tile_cols == 0 || opt.tile_cols == 16 || opt.tile_cols == 32 || opt.tile_cols == 64))
    FAIL(SC_ERR_INVALID_ARG, "tile_cols must be 0, 16, 32 or 64");
  if (opt.panel_cols < 0 || opt.panel_cols > kMaxPanel) FAIL(SC_ERR_INVALID_ARG, "panel_cols must be in [0, 64]");
  for (int k = 0; k < 7; k++)
    if (opt.reserved[k] != 0) FAIL(SC_ERR_INVALID_ARG, "reserved options must be zero");
  P.opt = opt;
  P.nsub = nsub;
  P.n_lambda = opt.n_lambda_global;
  int32_t max_m = 0;
  for (int32_t i = 0; i < nsub; i++) {
    sc_status st = validate_desc(sd[i], i, err);
    if (st != SC_OK) return st;
    max_m = std::max(max_m, sd[i].m);
    if (sd[i].lambda_map)
      for (int32_t a = 0; a < sd[i].m; a++)
        if (sd[i].lambda_map[a] < 0 || sd[i].lambda_map[a] >= opt.n_lambda_global)
          FAIL(SC_ERR_INVALID_ARG, "subdomain " + std::to_string(i) + ": lambda_map entry outside [0, n_lambda_global)");
  }
  P.T = opt.tile_cols ? opt.tile_cols : (max_m <= 64 ? 16 : (max_m <= 512 ? 32 : 64));
  P.PW = opt.panel_cols ? opt.panel_cols : kMaxPanel;

  // --- classes (dedup identical patterns)
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
      sc_status st = analyse_class(sd[i], P.T, P.PW, opt.skip, P.classes.back(), err);
      if (st != SC_OK) {
        err = "subdomain " + std::to_string(i) + ": " + err;
        return st;
      }
    }
    P.sub_cls[(size_t)i] = cls;
  }

  // --- global concatenation: class-local indices -> global
  int32_t tile_base = 0, step_base = 0, reach_base = 0, binit_base = 0, seg_base = 0, R_base = 0, pair_base = 0;
  for (auto& C : P.classes) {
    P.cls_tile_begin.push_back(tile_base);
    P.cls_pair_begin.push_back(pair_base);
    for (auto& t : C.tiles) {
      t.step_begin += step_base;
      t.step_end += step_base;
      t.reach_begin += reach_base;
      t.reach_end += reach_base;
      t.binit_begin += binit_base;
      t.binit_end += binit_base;
    }
    for (auto& s : C.steps) s.R_off += R_base;
    for (auto& p : C.pairs) {
      p.I += tile_base;
      p.J += tile_base;
      p.seg_begin += seg_base;
      p.seg_end += seg_base;
    }
    tile_base += (int32_t)C.tiles.size();
    step_base += (int32_t)C.steps.size();
    reach_base += (int32_t)C.reach.size();
    binit_base += (int32_t)C.binit.size();
    seg_base += (int32_t)C.segs.size();
    R_base += (int32_t)C.Rrows.size();
    pair_base += (int32_t)C.pairs.size();
  }

  // --- per subdomain layout + task lists
  P.sub_m.resize((size_t)nsub);
  P.sub_n.resize((size_t)nsub);
  P.sub_nnz.resize((size_t)nsub);
  P.lambda_map.resize((size_t)nsub);
  sc_stats& S = P.stats;
  std::memset(&S, 0, sizeof(S));
  S.nsub = nsub;
  S.n_classes = (int32_t)P.classes.size();
  S.tile_cols = P.T;
  S.panel_cols = P.PW;
  std::vector<std::vector<std::pair<int64_t, int64_t>>> contrib;  // unused placeholder
  std::vector<int64_t> qcount((size_t)std::max<int64_t>(opt.n_lambda_global, 0) + 1, 0);
  for (int32_t i = 0; i < nsub; i++) {
    const ClassPlan& C = P.classes[(size_t)P.sub_cls[(size_t)i]];
    int32_t cls = P.sub_cls[(size_t)i];
    P.sub_m[(size_t)i] = C.m;
    P.sub_n[(size_t)i] = C.n;
    P.sub_nnz[(size_t)i] = C.colptr[(size_t)C.n];
    P.max_n = std::max(P.max_n, C.n);
    P.sub_X_base.push_back(P.X_doubles);
    P.X_doubles += C.x_doubles;
    P.sub_F_base.push_back(P.F_doubles);
    P.F_doubles += (int64_t)C.m * C.m;
    P.sub_part_off.push_back(P.part_doubles);
    int32_t nblk = (C.m + 31) / 32;
    P.part_doubles += (int64_t)nblk * C.m;
    for (size_t t = 0; t < C.tiles.size(); t++)
      if (C.tiles[t].strip_rows > 0) P.trsm_tasks.push_back({i, P.cls_tile_begin[(size_t)cls] + (int32_t)t});
    for (size_t q = 0; q < C.pairs.size(); q++) P.syrk_tasks.push_back({i, P.cls_pair_begin[(size_t)cls] + (int32_t)q});
    for (int32_t b = 0; b < C.m; b += 32) P.apply_tasks.push_back({i, b});
    auto& lm = P.lambda_map[(size_t)i];
    lm.assign((size_t)C.m, -1);
    P.sub_slm_off.push_back((int64_t)P.slm.size());
    if (sd[i].lambda_map) {
      lm.assign(sd[i].lambda_map, sd[i].lambda_map + C.m);
      for (int32_t a = 0; a < C.m; a++) {
        int64_t g = lm[(size_t)C.sigma[(size_t)a]];
        P.slm.push_back(g);
        qcount[(size_t)g]++;
      }
    } else {
      for (int32_t a = 0; a < C.m; a++) P.slm.push_back(-1);
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
    S.trsm_steps += 0;
    for (auto& t : C.tiles) S.trsm_steps += t.step_end - t.step_begin;
    for (auto& p : C.pairs) S.syrk_segments += p.seg_end - p.seg_begin;
    S.bytes_apply += 8.0 * (double)C.m * (C.m + 1) / 2.0 + 8.0 * 3.0 * C.m;
  }
  (void)contrib;
  S.trsm_tasks = (int64_t)P.trsm_tasks.size();
  S.syrk_tasks = (int64_t)P.syrk_tasks.size();
  S.bytes_X = 8.0 * (double)P.X_doubles;
  // CSR over global multipliers of the (sub, stepped position) contributions, in (sub, a) order
  int64_t NL = std::max<int64_t>(opt.n_lambda_global, 0);
  P.qg_ptr.assign((size_t)NL + 1, 0);
  for (int64_t g = 0; g < NL; g++) P.qg_ptr[(size_t)g + 1] = P.qg_ptr[(size_t)g] + qcount[(size_t)g];
  P.qg_sub_a.assign((size_t)P.qg_ptr[(size_t)NL], 0);
  std::vector<int64_t> fillpos(P.qg_ptr.begin(), P.qg_ptr.end() - (NL >= 0 ? 1 : 0));
  for (int32_t i = 0; i < nsub; i++) {
    const ClassPlan& C = P.classes[(size_t)P.sub_cls[(size_t)i]];
    if (!sd[i].lambda_map) continue;
    for (int32_t a = 0; a < C.m; a++) {
      int64_t g = P.slm[(size_t)(P.sub_slm_off[(size_t)i] + a)];
      P.qg_sub_a[(size_t)fillpos[(size_t)g]++] = ((int64_t)i << 32) | (int64_t)a;
    }
  }
  return SC_OK;
}

}  // namespace sc
