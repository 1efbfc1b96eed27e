// factor_plan.cpp — symbolic stage of the device numeric factorization.
//
// PAPER.md P:326-328 (§2.2): "the factorization is done in two stages: the symbolic factorization
// ... performed only once ... and the numeric factorization" whenever the values change.  The
// pattern of L_i is already known (sc_plan_create validated it as a Cholesky fill pattern); this
// file derives, per pattern class, what the left-looking supernodal numeric factorization in
// factor.cu needs:
//   1. factor panels of <= 32 columns (partition_panels: maximal supernodes, wide ones split, small
//      consecutive ones merged; rows below each panel R_p);
//   2. per panel p the list of descendant panels d that update it (R_d meets the columns of p), with
//      the index ranges of R_d inside p's columns [s0, s1) and below them [s1, nR_d);
//   3. levels (0 = no descendant, else 1 + max over the descendants) and frames: the diagonal block
//      plus one frame per 32 rows of R_p -- one warp task each;
//   4. K entries -> frame positions (perm applied, each entry moved to the lower triangle of
//      P K P^T; an entry outside the pattern of L is a pattern error) and L entries -> frame
//      positions (the output scatter in the caller's CSC order);
//   5. the task order: chunks of subdomains, inside a chunk by (level, subdomain, panel, frame), so
//      every dependency precedes its dependants in the queue (the kernel's deadlock-freedom argument).
#include <algorithm>
#include <atomic>
#include <thread>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "sc_internal.h"

namespace sc {

namespace {

#define FFAIL(code, msg) \
  do {                   \
    err = (msg);         \
    return (code);       \
  } while (0)

sc_status analyse_factor_class(const ClassPlan& C, const sc_K_pattern* Kp, FactorClass& F, std::string& err) {
  const int32_t n = C.n;
  const int64_t* cp = C.colptr.data();
  const int32_t* ri = C.rowidx.data();
  std::vector<int32_t> parent((size_t)n, -1);
  for (int32_t c = 0; c < n; c++)
    if (cp[c + 1] - cp[c] > 1) parent[(size_t)c] = ri[cp[c] + 1];
  std::vector<PanelPart> parts;
  // relaxation of the factor panels (explicit zeros cost workspace bytes and update flops here, and
  // panels cost tasks): SC_FACTOR_ZMAX / SC_FACTOR_WSMALL, default the TRSM's rule
  const char* ez = std::getenv("SC_FACTOR_ZMAX");
  const char* ew = std::getenv("SC_FACTOR_WSMALL");
  partition_panels(n, cp, ri, parent, kFW, parts, ez ? std::atof(ez) : -1.0, ew ? std::atoi(ew) : -1);
  std::vector<int32_t> poc((size_t)n, -1);
  for (size_t k = 0; k < parts.size(); k++) {
    FPanel p{};
    p.a = parts[k].a;
    p.kw = parts[k].b - parts[k].a;
    p.kw8 = (p.kw + 7) & ~7;
    p.nR = (int32_t)parts[k].R.size();
    p.R_off = (int32_t)F.Rrows.size();
    F.Rrows.insert(F.Rrows.end(), parts[k].R.begin(), parts[k].R.end());
    for (int32_t c = p.a; c < parts[k].b; c++) poc[(size_t)c] = (int32_t)k;
    F.panels.push_back(p);
  }
  const int32_t np = (int32_t)F.panels.size();
  // 2. update lists: walk R_d and group its rows by the panel they fall in
  std::vector<std::vector<FUpd>> lists((size_t)np);
  for (int32_t d = 0; d < np; d++) {
    const FPanel& dn = F.panels[(size_t)d];
    const int32_t* R = F.Rrows.data() + dn.R_off;
    int32_t k = 0;
    while (k < dn.nR) {
      const int32_t p = poc[(size_t)R[k]];
      const int32_t b = F.panels[(size_t)p].a + F.panels[(size_t)p].kw;
      const int32_t s0 = k;
      while (k < dn.nR && R[k] < b) k++;
      lists[(size_t)p].push_back(FUpd{d, s0, k, 0});
    }
  }
  // 3. levels, frames, workspace layout, flop counts
  int64_t w = 0;
  for (int32_t p = 0; p < np; p++) {
    FPanel& pn = F.panels[(size_t)p];
    pn.upd_begin = (int32_t)F.upd.size();
    int32_t lev = 0;
    for (const FUpd& u : lists[(size_t)p]) {
      lev = std::max(lev, F.panels[(size_t)u.d].level + 1);
      F.upd.push_back(u);
      const FPanel& dn = F.panels[(size_t)u.d];
      // executed: rows of d in this panel and below x columns of d in this panel x 2 kw_d
      F.flops += 2.0 * dn.kw * (double)(dn.nR - u.s0) * (double)(u.s1 - u.s0);
    }
    pn.upd_end = (int32_t)F.upd.size();
    pn.level = lev;
    F.max_level = std::max(F.max_level, lev);
    pn.frame_begin = (int32_t)F.frames.size();
    pn.nframe = 1 + (pn.nR + kFW - 1) / kFW;
    for (int32_t f = 0; f < pn.nframe; f++) {
      FFrame fr{};
      fr.panel = p;
      fr.r0 = f == 0 ? -1 : (f - 1) * kFW;
      fr.nrow = f == 0 ? pn.kw : std::min(kFW, pn.nR - (f - 1) * kFW);
      F.frames.push_back(fr);
    }
    pn.w_off = w;
    w += (int64_t)pn.nR * pn.kw8;  // row-major rows, kw8 wide (16-byte aligned rows for cp.async)
    pn.inv_off = w;
    w += (int64_t)pn.kw8 * pn.kw8;
    F.flops += (double)pn.kw * pn.kw * pn.kw / 3.0 * 2.0 + 2.0 * pn.nR * (double)pn.kw * pn.kw;
  }
  F.w_doubles = w;
  for (int32_t c = 0; c < n; c++) {
    const double cc = (double)(cp[c + 1] - cp[c]);
    F.flops_useful += cc * cc;
  }
  // ancestors (implicit apply, backward): the reverse of the update lists
  {
    std::vector<std::vector<FUpd>> al((size_t)np);
    for (int32_t p = 0; p < np; p++)
      for (int32_t u = F.panels[(size_t)p].upd_begin; u < F.panels[(size_t)p].upd_end; u++) {
        const FUpd U = F.upd[(size_t)u];
        al[(size_t)U.d].push_back(FUpd{p, U.s0, U.s1, 0});
      }
    for (int32_t p = 0; p < np; p++) {
      F.panels[(size_t)p].anc_begin = (int32_t)F.anc.size();
      F.anc.insert(F.anc.end(), al[(size_t)p].begin(), al[(size_t)p].end());
      F.panels[(size_t)p].anc_end = (int32_t)F.anc.size();
    }
  }
  // B~^T by permuted row (implicit apply, forward gather): transpose of the plan's stepped columns
  {
    F.bt_rp.assign((size_t)n + 1, 0);
    for (int32_t r : C.ib_row) F.bt_rp[(size_t)r + 1]++;
    for (int32_t r = 0; r < n; r++) F.bt_rp[(size_t)r + 1] += F.bt_rp[(size_t)r];
    F.bt_a.assign(C.ib_row.size(), 0);
    F.bt_v.assign(C.ib_row.size(), 0.0);
    std::vector<int32_t> pos(F.bt_rp.begin(), F.bt_rp.end() - 1);
    for (int32_t a = 0; a < C.m; a++)  // ascending stepped column within each row: a fixed summation order
      for (int32_t e = C.ib_ptr[(size_t)a]; e < C.ib_ptr[(size_t)a + 1]; e++) {
        const int32_t r = C.ib_row[(size_t)e];
        F.bt_a[(size_t)pos[(size_t)r]] = a;
        F.bt_v[(size_t)pos[(size_t)r]++] = C.ib_val[(size_t)e];
      }
  }
  // frame update lists: for every update (d -> p) the diagonal frame gets (d, s0, s1, s0, s1); the
  // rows R_d[s1, nR_d) are grouped by the row frame of p they fall in (two-pointer walk over R_p)
  std::vector<std::vector<FFUpd>> fl(F.frames.size());
  for (int32_t p = 0; p < np; p++) {
    const FPanel& pn = F.panels[(size_t)p];
    const int32_t* Rp = F.Rrows.data() + pn.R_off;
    for (int32_t u = pn.upd_begin; u < pn.upd_end; u++) {
      const FUpd U = F.upd[(size_t)u];
      const FPanel& dn = F.panels[(size_t)U.d];
      const int32_t* Rd = F.Rrows.data() + dn.R_off;
      fl[(size_t)pn.frame_begin].push_back(FFUpd{U.d, U.s0, U.s1, U.s0, U.s1, 0});
      int32_t k = U.s1;
      int32_t ip = k < dn.nR ? (int32_t)(std::lower_bound(Rp, Rp + pn.nR, Rd[k]) - Rp) : pn.nR;
      while (k < dn.nR && ip < pn.nR) {
        const int32_t f = ip / kFW, fend = std::min(pn.nR, (f + 1) * kFW);
        const int32_t k0 = k;
        // rows of R_d up to the last row of this frame (rows of d missing from R_p are skipped later)
        while (k < dn.nR && Rd[k] <= Rp[fend - 1]) k++;
        if (k > k0) fl[(size_t)(pn.frame_begin + 1 + f)].push_back(FFUpd{U.d, U.s0, U.s1, k0, k, 0});
        if (k < dn.nR) ip = (int32_t)(std::lower_bound(Rp + fend, Rp + pn.nR, Rd[k]) - Rp);
      }
    }
  }
  if (std::getenv("SC_DEBUG_FACTOR")) {
    size_t nu = 0, rows = 0, maxu = 0;
    for (auto& v : fl) {
      nu += v.size();
      maxu = std::max(maxu, v.size());
      for (auto& u : v) rows += (size_t)(u.k1 - u.k0);
    }
    fprintf(stderr, "factor class: n %d panels %d frames %zu frame-updates %zu (max %zu per frame) update rows %zu levels %d\n",
            n, np, F.frames.size(), nu, maxu, rows, F.max_level);
  }
  // frames with more than `split` descendant updates keep the first `split` and hand the rest to
  // partial update tasks of at most `split` updates each (their blocks are summed by the frame)
  int split = 8;
  if (const char* e = std::getenv("SC_FACTOR_SPLIT")) split = std::atoi(e);
  F.parts.clear();
  for (size_t f = 0; f < F.frames.size(); f++) {
    F.frames[f].u_begin = (int32_t)F.fupd.size();
    F.fupd.insert(F.fupd.end(), fl[f].begin(), fl[f].end());
    F.frames[f].u_end = (int32_t)F.fupd.size();
    F.frames[f].part_begin = F.frames[f].part_end = (int32_t)F.parts.size();
    const int32_t nu = F.frames[f].u_end - F.frames[f].u_begin;
    if (split > 0 && nu > split) {
      for (int32_t u = F.frames[f].u_begin + split; u < F.frames[f].u_end; u += split)
        F.parts.push_back(FPart{(int32_t)f, u, std::min(u + split, F.frames[f].u_end), (int32_t)F.parts.size()});
      F.frames[f].u_end = F.frames[f].u_begin + split;
      F.frames[f].part_end = (int32_t)F.parts.size();
    }
  }
  // 4. entry maps
  std::vector<int32_t> iperm((size_t)n);
  for (int32_t k = 0; k < n; k++) iperm[(size_t)C.perm[(size_t)k]] = k;
  auto locate = [&](int32_t r, int32_t c, int32_t& frame, int32_t& pos) -> bool {  // r >= c, permuted
    const int32_t p = poc[(size_t)c];
    const FPanel& pn = F.panels[(size_t)p];
    if (r < pn.a + pn.kw) {
      frame = pn.frame_begin;
      pos = (r - pn.a) * kFW + (c - pn.a);
      return true;
    }
    const int32_t* R = F.Rrows.data() + pn.R_off;
    const int32_t k = (int32_t)(std::lower_bound(R, R + pn.nR, r) - R);
    if (k >= pn.nR || R[k] != r) return false;
    frame = pn.frame_begin + 1 + k / kFW;
    pos = (k % kFW) * kFW + (c - pn.a);
    return true;
  };
  std::vector<std::vector<FEnt>> kf(F.frames.size()), lf(F.frames.size());
  if (Kp) {
    const sc_K_pattern& K = *Kp;
    F.nnzK = K.K_colptr[n];
    for (int32_t j = 0; j < n; j++)
      for (int64_t q = K.K_colptr[j]; q < K.K_colptr[j + 1]; q++) {
        const int32_t i = K.K_rowidx[q];
        const int32_t pi = iperm[(size_t)i], pj = iperm[(size_t)j];
        const int32_t r = std::max(pi, pj), c = std::min(pi, pj);
        int32_t fr, pos;
        const bool inL = std::binary_search(ri + cp[c], ri + cp[c + 1], r);
        if (!inL || !locate(r, c, fr, pos))
          FFAIL(SC_ERR_PATTERN, "K entry (" + std::to_string(i) + ", " + std::to_string(j) +
                                    ") lies outside the pattern of L (permuted (" + std::to_string(r) + ", " +
                                    std::to_string(c) + "))");
        kf[(size_t)fr].push_back(FEnt{(int32_t)q, pos});
      }
  }
  for (int32_t c = 0; c < n; c++)
    for (int64_t q = cp[c]; q < cp[c + 1]; q++) {
      int32_t fr, pos;
      if (!locate(ri[q], c, fr, pos)) FFAIL(SC_ERR_PATTERN, "internal: L entry outside its factor panel");
      lf[(size_t)fr].push_back(FEnt{(int32_t)q, pos});
    }
  std::vector<int32_t> mark((size_t)kFW * kFW, -1);
  for (size_t f = 0; f < F.frames.size(); f++) {
    for (const FEnt& e : kf[f]) {  // each lower position of P K P^T at most once (no duplicate entries)
      if (mark[(size_t)e.pos] == (int32_t)f) FFAIL(SC_ERR_PATTERN, "K has a duplicate entry (after perm / transpose)");
      mark[(size_t)e.pos] = (int32_t)f;
    }
    F.frames[f].k_begin = (int32_t)F.kent.size();
    F.kent.insert(F.kent.end(), kf[f].begin(), kf[f].end());
    F.frames[f].k_end = (int32_t)F.kent.size();
    F.frames[f].l_begin = (int32_t)F.lent.size();
    F.lent.insert(F.lent.end(), lf[f].begin(), lf[f].end());
    F.frames[f].l_end = (int32_t)F.lent.size();
  }
  // every diagonal of P K P^T must be present (a missing one is a structurally singular K)
  if (Kp) {
    std::vector<char> hasd((size_t)n, 0);
    for (int32_t j = 0; j < n; j++)
      for (int64_t q = Kp->K_colptr[j]; q < Kp->K_colptr[j + 1]; q++)
        if (Kp->K_rowidx[q] == j) hasd[(size_t)j] = 1;
    for (int32_t j = 0; j < n; j++)
      if (!hasd[(size_t)j]) FFAIL(SC_ERR_PATTERN, "K diagonal entry " + std::to_string(j) + " missing");
  }
  return SC_OK;
}

sc_status validate_K(const sc_K_pattern& K, int32_t n, int32_t i, std::string& err) {
  const std::string who = "subdomain " + std::to_string(i) + ": ";
  if (!K.K_colptr || (n > 0 && !K.K_rowidx)) FFAIL(SC_ERR_INVALID_ARG, who + "NULL K pattern");
  if (K.K_colptr[0] != 0) FFAIL(SC_ERR_PATTERN, who + "K_colptr[0] != 0");
  if (K.K_colptr[n] > INT32_MAX) FFAIL(SC_ERR_INVALID_ARG, who + "nnz(K) exceeds 2^31");
  for (int32_t j = 0; j < n; j++) {
    if (K.K_colptr[j + 1] < K.K_colptr[j]) FFAIL(SC_ERR_PATTERN, who + "K_colptr not monotone");
    for (int64_t q = K.K_colptr[j]; q < K.K_colptr[j + 1]; q++) {
      const int32_t r = K.K_rowidx[q];
      if (r < j || r >= n) FFAIL(SC_ERR_PATTERN, who + "K entry not in the lower triangle / out of range");
      if (q > K.K_colptr[j] && r <= K.K_rowidx[q - 1]) FFAIL(SC_ERR_PATTERN, who + "K rows not strictly ascending");
    }
  }
  return SC_OK;
}

bool same_K(const sc_K_pattern& a, const sc_K_pattern& b, int32_t n) {
  if (a.K_colptr[n] != b.K_colptr[n]) return false;
  if (std::memcmp(a.K_colptr, b.K_colptr, sizeof(int64_t) * (size_t)(n + 1)) != 0) return false;
  return a.K_rowidx == b.K_rowidx ||
         std::memcmp(a.K_rowidx, b.K_rowidx, sizeof(int32_t) * (size_t)a.K_colptr[n]) == 0;
}

}  // namespace

sc_status build_factor_plan(Plan& P, const sc_K_pattern* kp, int32_t nsub, std::string& err) {
  if (nsub != P.nsub) FFAIL(SC_ERR_INVALID_ARG, "sc_factor_attach: nsub differs from the plan's");
  FactorPlan& F = P.fac;  // kp == NULL: symbolic from L only (staging for the implicit apply)
  F.has_K = kp != nullptr;
  const int32_t ncls = (int32_t)P.classes.size();
  std::vector<int32_t> rep((size_t)ncls, -1);
  for (int32_t i = 0; i < nsub; i++) {
    const int32_t c = P.sub_cls[(size_t)i];
    if (!kp) {
      if (rep[(size_t)c] < 0) rep[(size_t)c] = i;
      continue;
    }
    sc_status st = validate_K(kp[i], P.sub_n[(size_t)i], i, err);
    if (st != SC_OK) return st;
    if (rep[(size_t)c] < 0) {
      rep[(size_t)c] = i;
    } else if (!same_K(kp[rep[(size_t)c]], kp[i], P.sub_n[(size_t)i])) {
      FFAIL(SC_ERR_PATTERN, "subdomain " + std::to_string(i) + ": K pattern differs from subdomain " +
                                std::to_string(rep[(size_t)c]) + " of the same L/B pattern class");
    }
  }
  F.classes.assign((size_t)ncls, FactorClass());
  {  // classes are independent: analysed on all host threads (first error wins, by class order)
    std::vector<sc_status> cst((size_t)ncls, SC_OK);
    std::vector<std::string> cerr((size_t)ncls);
    std::atomic<int32_t> next{0};
    auto work = [&]() {
      for (int32_t c = next++; c < ncls; c = next++) {
        if (rep[(size_t)c] < 0) continue;
        cst[(size_t)c] = analyse_factor_class(P.classes[(size_t)c], kp ? &kp[rep[(size_t)c]] : nullptr,
                                              F.classes[(size_t)c], cerr[(size_t)c]);
      }
    };
    const int32_t nthr = std::min<int32_t>(ncls, (int32_t)std::max(1u, std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int32_t k = 1; k < nthr; k++) pool.emplace_back(work);
    work();
    for (auto& t : pool) t.join();
    for (int32_t c = 0; c < ncls; c++)
      if (cst[(size_t)c] != SC_OK) {
        err = "subdomain " + std::to_string(rep[(size_t)c]) + ": " + cerr[(size_t)c];
        return cst[(size_t)c];
      }
  }
  // globalise
  F.panels.clear();
  F.Rrows.clear();
  F.fupd.clear();
  F.anc.clear();
  F.bt_rp.clear();
  F.bt_a.clear();
  F.bt_v.clear();
  F.cls_bt0.assign((size_t)ncls, 0);
  F.frames.clear();
  F.kent.clear();
  F.lent.clear();
  F.parts.clear();
  F.cls_part0.assign((size_t)ncls + 1, 0);
  F.cls_frame0.assign((size_t)ncls + 1, 0);
  F.cls_panel0.assign((size_t)ncls + 1, 0);
  for (int32_t c = 0; c < ncls; c++) {
    const FactorClass& fc = F.classes[(size_t)c];
    const int32_t p0 = (int32_t)F.panels.size(), r0 = (int32_t)F.Rrows.size(), u0 = (int32_t)F.fupd.size();
    const int32_t f0 = (int32_t)F.frames.size(), k0 = (int32_t)F.kent.size(), l0 = (int32_t)F.lent.size();
    F.cls_panel0[(size_t)c] = p0;
    const int32_t a0 = (int32_t)F.anc.size();
    for (FPanel pn : fc.panels) {
      pn.R_off += r0;
      pn.frame_begin += f0;
      pn.anc_begin += a0;
      pn.anc_end += a0;
      F.panels.push_back(pn);
    }
    for (FUpd u : fc.anc) {
      u.d += p0;
      F.anc.push_back(u);
    }
    F.cls_bt0[(size_t)c] = (int64_t)F.bt_rp.size();
    const int32_t e0 = (int32_t)F.bt_a.size();
    for (int32_t v : fc.bt_rp) F.bt_rp.push_back(v + e0);
    F.bt_a.insert(F.bt_a.end(), fc.bt_a.begin(), fc.bt_a.end());
    F.bt_v.insert(F.bt_v.end(), fc.bt_v.begin(), fc.bt_v.end());
    F.Rrows.insert(F.Rrows.end(), fc.Rrows.begin(), fc.Rrows.end());
    for (FFUpd u : fc.fupd) {
      u.d += p0;
      F.fupd.push_back(u);
    }
    F.cls_part0[(size_t)c] = (int32_t)F.parts.size();
    F.cls_frame0[(size_t)c] = f0;
    for (FPart pt : fc.parts) {
      pt.frame += f0;
      pt.u_begin += u0;
      pt.u_end += u0;
      F.parts.push_back(pt);
    }
    for (FFrame fr : fc.frames) {
      fr.panel += p0;
      fr.u_begin += u0;
      fr.u_end += u0;
      fr.k_begin += k0;
      fr.k_end += k0;
      fr.l_begin += l0;
      fr.l_end += l0;
      F.frames.push_back(fr);
    }
    F.kent.insert(F.kent.end(), fc.kent.begin(), fc.kent.end());
    F.lent.insert(F.lent.end(), fc.lent.begin(), fc.lent.end());
  }
  F.cls_panel0[(size_t)ncls] = (int32_t)F.panels.size();
  F.cls_part0[(size_t)ncls] = (int32_t)F.parts.size();
  F.sub_part_base.assign((size_t)nsub + 1, 0);
  for (int32_t i = 0; i < nsub; i++)
    F.sub_part_base[(size_t)i + 1] = F.sub_part_base[(size_t)i] + (int64_t)F.classes[(size_t)P.sub_cls[(size_t)i]].parts.size();
  F.nparts = F.sub_part_base[(size_t)nsub];
  // per-subdomain workspace and flags
  F.sub_W_base.assign((size_t)nsub + 1, 0);
  F.sub_flag_base.assign((size_t)nsub + 1, 0);
  F.sub_nnzK.assign((size_t)nsub, 0);
  F.flops = F.flops_useful = F.bytes_K = 0;
  for (int32_t i = 0; i < nsub; i++) {
    const FactorClass& fc = F.classes[(size_t)P.sub_cls[(size_t)i]];
    F.sub_W_base[(size_t)i + 1] = F.sub_W_base[(size_t)i] + fc.w_doubles;
    F.sub_flag_base[(size_t)i + 1] = F.sub_flag_base[(size_t)i] + (int64_t)fc.panels.size();
    F.sub_nnzK[(size_t)i] = fc.nnzK;
    F.flops += fc.flops;
    F.flops_useful += fc.flops_useful;
    F.bytes_K += 8.0 * (double)fc.nnzK;
  }
  F.W_doubles = F.sub_W_base[(size_t)nsub];
  F.sub_x_base.assign((size_t)nsub + 1, 0);
  for (int32_t i = 0; i < nsub; i++) F.sub_x_base[(size_t)i + 1] = F.sub_x_base[(size_t)i] + P.sub_n[(size_t)i];
  F.nflags = F.sub_flag_base[(size_t)nsub];
  // 5. task order, by (level, subdomain, panel, frame) over the whole batch: the critical path is the
  // longest panel chain, every level of every subdomain is ready together (per-chunk orders would
  // serialise one chain per chunk: measured 2.6x slower for cfg2 with 16 chunks).
  const char* me = std::getenv("SC_FACTOR_MERGE");
  const int32_t merge = me ? std::atoi(me) : 6;  // panels with <= this many frames form one task
  const char* mst = std::getenv("SC_FACTOR_SUBTREE");
  const int32_t subtree = mst ? std::atoi(mst) : 24;  // self-contained panel ranges of <= this many frames
  // Per class: self-contained panel ranges [lo, hi] (every update of a panel in the range comes from
  // the range: a whole subtree when the ordering is a postorder, as nested dissection's is) of at
  // most `subtree` frames become ONE task -- its frames in panel order, processed by one warp with no
  // waits -- at level 0; the other panels are tasks of their own level.
  std::vector<std::vector<std::pair<int32_t, int32_t>>> cls_units((size_t)ncls);  // (first local panel, last)
  for (int32_t c = 0; c < ncls; c++) {
    const FactorClass& fc = F.classes[(size_t)c];
    const int32_t np = (int32_t)fc.panels.size();
    std::vector<int32_t> lo((size_t)np);
    for (int32_t p = 0; p < np; p++) {  // lowest panel of p's dependency closure
      int32_t l = p;
      for (int32_t u = fc.panels[(size_t)p].upd_begin; u < fc.panels[(size_t)p].upd_end; u++)
        l = std::min(l, lo[(size_t)fc.upd[(size_t)u].d]);
      lo[(size_t)p] = l;
    }
    auto& units = cls_units[(size_t)c];
    int32_t p = np - 1;
    while (p >= 0) {
      const int32_t l = lo[(size_t)p];
      int32_t frames = 0, minlo = l;
      for (int32_t q = l; q <= p; q++) {
        frames += fc.panels[(size_t)q].nframe;
        minlo = std::min(minlo, lo[(size_t)q]);
      }
      if (l < p && minlo >= l && frames <= subtree) {
        units.push_back({l, p});
        p = l - 1;
      } else {
        units.push_back({p, p});
        p--;
      }
    }
  }
  // frames inside multi-panel subtree units are processed in order by the unit's warp: their updates
  // are not split (a partial task placed before the unit would wait for frames of the unit itself)
  for (int32_t c = 0; c < ncls; c++)
    for (const auto& un : cls_units[(size_t)c])
      if (un.first < un.second)
        for (int32_t q = un.first; q <= un.second; q++) {
          const FPanel& pa = F.panels[(size_t)(F.cls_panel0[(size_t)c] + q)];
          for (int32_t f = 0; f < pa.nframe; f++) {
            FFrame& fr = F.frames[(size_t)(pa.frame_begin + f)];
            if (fr.part_end > fr.part_begin) {
              fr.u_end = F.parts[(size_t)(F.cls_part0[(size_t)c] + fr.part_end - 1)].u_end;
              fr.part_begin = fr.part_end;
            }
          }
        }
  // partial-update slots cost 8 KB each per subdomain.  Over the budget (SC_FACTOR_SPLIT_MB, default
  // 8192 MB) only the frames with more than t = 16, 32, ... updates stay split (the heaviest frames
  // are the ones on the critical path), then, if still over, consecutive partials of a frame are
  // merged 2, 4, ... at a time; past that nothing is split
  {
    double mb = 8192.0;
    if (const char* e = std::getenv("SC_FACTOR_SPLIT_MB")) mb = std::atof(e);
    std::vector<int64_t> ncls_sub((size_t)ncls, 0);
    for (int32_t i = 0; i < nsub; i++) ncls_sub[(size_t)P.sub_cls[(size_t)i]]++;
    auto nupd = [&](int32_t c, const FFrame& fr) {  // all updates of a (possibly split) frame
      return fr.part_end > fr.part_begin ? F.parts[(size_t)(F.cls_part0[(size_t)c] + fr.part_end - 1)].u_end - fr.u_begin
                                         : fr.u_end - fr.u_begin;
    };
    auto slots = [&](int t, int k) {  // slots over all subdomains: frames with > t updates, k merged
      double tot = 0;
      for (int32_t c = 0; c < ncls; c++)
        for (int32_t g = 0; g < (int32_t)F.classes[(size_t)c].frames.size(); g++) {
          const FFrame& fr = F.frames[(size_t)(F.cls_frame0[(size_t)c] + g)];
          if (fr.part_end > fr.part_begin && nupd(c, fr) > t)
            tot += (double)ncls_sub[(size_t)c] * (double)((fr.part_end - fr.part_begin + k - 1) / k);
        }
      return tot;
    };
    int t = 0, k = 1;
    while (t < 256 && 8192.0 * slots(t, 1) > mb * 1e6) t = t ? 2 * t : 16;
    if (t >= 256) {
      t = 128;
      while (k <= 64 && 8192.0 * slots(t, k) > mb * 1e6) k *= 2;
    }
    if (t > 0 || k > 1) {  // rebuild the partial lists
      std::vector<FPart> np;
      std::vector<int32_t> cp0((size_t)ncls + 1, 0);
      for (int32_t c = 0; c < ncls; c++) {
        cp0[(size_t)c] = (int32_t)np.size();
        int32_t local = 0;
        for (int32_t g = 0; g < (int32_t)F.classes[(size_t)c].frames.size(); g++) {
          FFrame& fr = F.frames[(size_t)(F.cls_frame0[(size_t)c] + g)];
          const int32_t pb = fr.part_begin, pe = fr.part_end, nu = nupd(c, fr);
          fr.part_begin = fr.part_end = local;
          if (pe <= pb) continue;
          if (nu <= t || k > 64) {  // not split
            fr.u_end = F.parts[(size_t)(F.cls_part0[(size_t)c] + pe - 1)].u_end;
            continue;
          }
          for (int32_t q = pb; q < pe; q += k) {
            FPart m = F.parts[(size_t)(F.cls_part0[(size_t)c] + q)];
            m.u_end = F.parts[(size_t)(F.cls_part0[(size_t)c] + std::min(pe, q + k) - 1)].u_end;
            m.slot = local++;
            np.push_back(m);
          }
          fr.part_end = local;
        }
      }
      cp0[(size_t)ncls] = (int32_t)np.size();
      F.parts.swap(np);
      F.cls_part0.swap(cp0);
      F.sub_part_base.assign((size_t)nsub + 1, 0);
      for (int32_t i = 0; i < nsub; i++) {
        const int32_t c = P.sub_cls[(size_t)i];
        F.sub_part_base[(size_t)i + 1] = F.sub_part_base[(size_t)i] + (F.cls_part0[(size_t)c + 1] - F.cls_part0[(size_t)c]);
      }
      F.nparts = F.sub_part_base[(size_t)nsub];
    }
    F.part_merge = k;
    F.part_min_updates = t;
    if (std::getenv("SC_DEBUG_FACTOR"))
      fprintf(stderr, "factor split: frames with > %d updates, %d partials per slot, %lld slots (%.1f MB)\n", std::max(t, 8), k,
              (long long)F.nparts, 8192.0 * (double)F.nparts / 1e6);
  }
  auto order = [&](int32_t s0, int32_t s1) {
    int32_t maxlev = 0;
    for (int32_t i = s0; i < s1; i++) maxlev = std::max(maxlev, F.classes[(size_t)P.sub_cls[(size_t)i]].max_level);
    std::vector<std::vector<FTask>> bylev((size_t)maxlev + 1);
    std::vector<std::vector<I2>> pbylev((size_t)maxlev + 1);
    for (int32_t i = s0; i < s1; i++) {
      const int32_t c = P.sub_cls[(size_t)i], p0 = F.cls_panel0[(size_t)c];
      for (const auto& un : cls_units[(size_t)c]) {
        const FPanel& pa = F.panels[(size_t)(p0 + un.first)];
        if (un.first < un.second) {  // subtree unit: all its frames, panel order, level 0
          const FPanel& pb = F.panels[(size_t)(p0 + un.second)];
          bylev[0].push_back(FTask{i, pa.frame_begin, pb.frame_begin + pb.nframe - pa.frame_begin, 0});
        } else {
          // partial update tasks of the panel's frames first (a frame task waits for its partials,
          // which only wait for descendants: earlier in the queue), nf = -1 marks them
          for (int32_t f = 0; f < pa.nframe; f++) {
            const FFrame& fr = F.frames[(size_t)(pa.frame_begin + f)];
            for (int32_t q = fr.part_begin; q < fr.part_end; q++)
              bylev[(size_t)pa.level].push_back(FTask{i, F.cls_part0[(size_t)c] + q, -1, 0});
          }
          if (pa.nframe <= merge) {  // small panel: one warp does the diagonal and then its rows
            bylev[(size_t)pa.level].push_back(FTask{i, pa.frame_begin, pa.nframe, 0});
          } else {
            for (int32_t f = 0; f < pa.nframe; f++) bylev[(size_t)pa.level].push_back(FTask{i, pa.frame_begin + f, 1, 0});
          }
        }
      }
      for (int32_t p = p0; p < F.cls_panel0[(size_t)c + 1]; p++) {
        // implicit forward: the split-off partial updates of the panel's diagonal frame first
        // (y = -1 - global part index), then the panel
        const FFrame& fr = F.frames[(size_t)F.panels[(size_t)p].frame_begin];
        for (int32_t q = fr.part_begin; q < fr.part_end; q++)
          pbylev[(size_t)F.panels[(size_t)p].level].push_back(I2{i, -1 - (F.cls_part0[(size_t)c] + q)});
        pbylev[(size_t)F.panels[(size_t)p].level].push_back(I2{i, p});
      }
    }
    for (auto& v : bylev) F.tasks.insert(F.tasks.end(), v.begin(), v.end());
    for (auto& v : pbylev) F.ptasks.insert(F.ptasks.end(), v.begin(), v.end());
  };
  F.tasks.clear();
  F.ptasks.clear();  // implicit apply: one task per (subdomain, panel) in level order
  order(0, nsub);
  F.task_chunk.assign(1, (int64_t)F.tasks.size());  // end of the whole-batch order
  if (F.tasks.size() > (size_t)INT32_MAX) FFAIL(SC_ERR_INVALID_ARG, "too many factorization tasks");
  return SC_OK;
}

}  // namespace sc
