// ProductRep pipeline and exact trace algebra (product_rep.cpp) on the device.
#include <algorithm>

#include "prodrep.cuh"

namespace hg {

namespace {

/// Y <- Abar^{-1} Y (inverse) or Abar Y on an n x w panel.
void leaf_step(const DFactor& f, bool inverse, double* Y, int w) {
    if (w <= 0) return;
    if (inverse) {
        leaf_solve(f, Y, f.n(), w);
    } else {
        DVec tmp(static_cast<size_t>(f.n()) * static_cast<size_t>(w));
        panel_axpby(f.n(), w, 1.0, Y, f.n(), 0.0, tmp.get(), f.n());
        leaf_mm(f.tree->leaves(), f.leaf_mat->get(), f.lstride(), f.bmax(), false, tmp.get(), f.n(), Y, f.n(), w,
                1.0, 0.0);
    }
}

/// One factor level applied to a panel: (I + v u^T)^{-1} (inverse) or (I + u v^T).
void level_op(const DFactor& f, int i, bool inverse, double* Y, int w) {
    if (w <= 0) return;
    if (inverse)
        level_inverse(f, i, true, Y, f.n(), w);
    else
        level_multiply(f, i, Y, f.n(), w);
}

}  // namespace

/// rows += p (q^T rows) per level-(i-1) node with q = u = [wbar 0; 0 xbar]
/// and p the node's m x 2R panel (product_rep.cpp:32-45): the reference's
/// association of the Woodbury update, used when HG_OPT_PRODUCT_ASSOCIATION
/// is HG_ASSOC_REFERENCE.
void level_update_pq(const DFactor& f, int i, const double* P, double* Y, int w) {
    const int R = f.Rl(i);
    if (R == 0 || w <= 0) return;
    const Partition& p = f.tree->part(i);
    const i64 n = f.n(), L = i64(p.nseg()) * R;
    DVec Q(static_cast<size_t>(L) * static_cast<size_t>(w));
    seg_tn(p, f.Wl(i), n, R, Y, n, w, Q.get(), R, int(L));
    seg_nn(p, P, n, 2 * R, Q.get(), 2 * R, int(L), TMap::parent(0, 0), Y, n, w, 1.0, 1.0);
}

void level_multiply(const DFactor& f, int i, double* Y, i64 ldy, int w) {
    const int R = f.Rl(i);
    if (R == 0 || w <= 0) return;
    const Partition& p = f.tree->part(i);
    DVec Q(static_cast<size_t>(p.nseg()) * static_cast<size_t>(R) * static_cast<size_t>(w));
    // v^T Y = [x^T Y_cr ; w^T Y_cl]; Y_cl += wbar (x^T Y_cr), Y_cr += xbar (w^T Y_cl)
    seg_tn(p, f.Fl(i), f.n(), R, Y, ldy, w, Q.get(), i64(R) * w, R);
    seg_nn(p, f.Wl(i), f.n(), R, Q.get(), i64(R) * w, R, TMap::sibling(), Y, ldy, w, 1.0, 1.0);
}

DProductRep pipeline(const DFactor& f, const DHodlr& b, bool inverse) {
    return pipeline_multi(f, std::vector<const DHodlr*>{&b}, inverse)[0];
}

std::vector<DProductRep> pipeline_multi(const DFactor& f, const std::vector<const DHodlr*>& bs, bool inverse) {
    for (const DHodlr* b : bs)
        if (!f.tree->host.same_structure(b->tree->host))
            throw std::invalid_argument("product pipeline: tree structure mismatch");
    if (!inverse && f.orient != 0) throw std::invalid_argument("multiply: factorization must be Right-oriented");
    if (inverse && f.orient != 1) throw std::invalid_argument("solve_multiply: factorization must be Left-oriented");
    const int tau = f.tau();
    const i64 n = f.n();
    const size_t P = bs.size();
    std::vector<DProductRep> reps(P);
    for (size_t j = 0; j < P; ++j) {
        DProductRep& rep = reps[j];
        rep.base = *bs[j];
        rep.base.make_asymmetric();
        rep.C.assign(static_cast<size_t>(tau), 0);
        rep.coff.assign(static_cast<size_t>(tau), 0);
        for (int i = 1; i <= tau; ++i) {
            rep.coff[static_cast<size_t>(i - 1)] = rep.sumC;
            rep.C[static_cast<size_t>(i - 1)] = 2 * f.Rl(i);
            rep.sumC += rep.C[static_cast<size_t>(i - 1)];
        }
    }
    if (P == 0) return reps;
    // Every column the pipeline rewrites lives in ONE n-row panel, ordered
    //   [G_tau | ... | G_2 | G_1 | Cu_1 | ... | Cu_tau | leaves_0 | .. | leaves_{P-1}]
    // with G_m = [U_m of base 0 | .. | U_m of base P-1], so the columns factor
    // level i acts on (every base's coarser left factors U_{m<i} and the older
    // corrections Cu_{<i}) are one contiguous block, and the final leaf step
    // is a single call over the whole panel. The corrections' left factors
    // p = -v cap^{-T}, and every factor level's update of them, depend on the
    // factorization only (product_rep.cpp:74-78, 84-104): the P reps share one
    // Cu, formed and updated once.
    std::vector<int> ucum(static_cast<size_t>(tau + 1), 0);  // ucum[m] = sum_{m' <= m} sum_j R_m'(j)
    for (int m = 1; m <= tau; ++m) {
        int g = 0;
        for (size_t j = 0; j < P; ++j) g += reps[j].base.Rl(m);
        ucum[static_cast<size_t>(m)] = ucum[static_cast<size_t>(m - 1)] + g;
    }
    const int sumR = ucum[static_cast<size_t>(tau)], cw = std::max(reps[0].sumC, 1), bm = f.bmax();
    const int cuo = sumR, lo = sumR + cw, total = lo + int(P) * bm;
    DVecP store = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(total), false);
    double* S = store->get();
    panel_axpby(n, cw, 0.0, nullptr, 0, 0.0, S + i64(cuo) * n, n);
    // Left factors are rewritten: each base gets its own copies (right factors stay aliased).
    for (int m = 1; m <= tau; ++m) {
        int off = sumR - ucum[static_cast<size_t>(m)];
        for (size_t j = 0; j < P; ++j) {
            const int R = reps[j].base.Rl(m);
            if (!R) continue;
            double* dst = S + i64(off) * n;
            panel_axpby(n, R, 1.0, bs[j]->Ul(m), n, 0.0, dst, n);
            reps[j].base.U[static_cast<size_t>(m - 1)] =
                make_view(store, dst, static_cast<size_t>(n) * static_cast<size_t>(R));
            off += R;
        }
    }
    DVecP cu_all = make_view(store, S + i64(cuo) * n, static_cast<size_t>(n) * static_cast<size_t>(cw));
    for (size_t j = 0; j < P; ++j) {
        reps[j].base.leaves = std::make_shared<DVec>(*bs[j]->leaves);
        reps[j].Cu = cu_all;
        reps[j].Cv = make_dvec(static_cast<size_t>(n) * static_cast<size_t>(cw), true);
    }

    const bool ref_assoc = inverse && current().product_assoc == HG_ASSOC_REFERENCE;
    for (int i = 1; i <= tau; ++i) {
        const int R = f.Rl(i);
        if (R == 0) continue;
        const Partition& p = f.tree->part(i);
        const int C2 = 2 * R;
        double* cu = reps[0].Cul(i);
        // p = -v cap^{-T}: rows cl = -w E[R:2R,:], rows cr = -x E[0:R,:]
        auto form_p = [&] {
            if (ref_assoc)  // the reference's LU substitution on v^T (no explicit inverse)
                form_p_reference(f, i, cu);
            else
                seg_nn(p, f.Fl(i), n, R, f.capinvT[static_cast<size_t>(i - 1)]->get(), C2, p.nseg() * R,
                       TMap::parent(R, 0), cu, n, C2, -1.0, 0.0);
        };
        // product_rep.cpp:84-104: older corrections' left factors and the
        // running bases' coarser left factors, in one call.
        const int us = ucum[static_cast<size_t>(i - 1)];
        const int wu = us + reps[0].coff[static_cast<size_t>(i - 1)];
        if (ref_assoc) {
            // The reference's association (product_rep.cpp:32-45,74-78): p is
            // formed first, then rows += p (q^T rows) with q = u.
            form_p();
            level_update_pq(f, i, cu, S + i64(cuo - us) * n, wu);
        } else {
            level_op(f, i, inverse, S + i64(cuo - us) * n, wu);
        }
        // product_rep.cpp:106-119: spawn c.u = p, c.v = B_sub^T q.
        DVec Q(static_cast<size_t>(n) * static_cast<size_t>(C2));
        if (inverse) {
            if (!ref_assoc) form_p();
            // q = u = [wbar 0; 0 xbar]
            panel_parity_select(p, R, f.Wl(i), n, 1.0, nullptr, 0, 0.0, Q.get(), n);
            panel_parity_select(p, R, nullptr, 0, 0.0, f.Wl(i), n, 1.0, Q.get() + i64(R) * n, n);
        } else {
            // p = u = [wbar 0; 0 xbar]
            panel_parity_select(p, R, f.Wl(i), n, 1.0, nullptr, 0, 0.0, cu, n);
            panel_parity_select(p, R, nullptr, 0, 0.0, f.Wl(i), n, 1.0, cu + i64(R) * n, n);
            // q = v = [0 w; x 0]
            panel_parity_select(p, R, nullptr, 0, 0.0, f.Fl(i), n, 1.0, Q.get(), n);
            panel_parity_select(p, R, f.Fl(i), n, 1.0, nullptr, 0, 0.0, Q.get() + i64(R) * n, n);
        }
        for (size_t j = 0; j < P; ++j)
            hodlr_apply(reps[j].base, Q.get(), n, C2, reps[j].Cvl(i), n, i, tau, true, true, 0.0);
    }
    // product_rep.cpp:124-152: leaf factor on every stored left factor and the leaves.
    for (size_t j = 0; j < P; ++j)
        leaves_panel(*f.tree, reps[j].base.leaves->get(), S + i64(lo + int(j) * bm) * n, true);
    leaf_step(f, inverse, S, total);
    for (size_t j = 0; j < P; ++j) {
        leaves_panel(*f.tree, reps[j].base.leaves->get(), S + i64(lo + int(j) * bm) * n, false);
        reps[j].base.leaves_zero = false;
    }
    return reps;
}

void trace_product_rep(const DProductRep& p, double* out, bool accumulate) {
    hodlr_trace(p.base, out, accumulate);
    if (p.sumC) dot_panels(p.n(), p.sumC, p.Cu->get(), p.n(), p.Cv->get(), p.n(), out, true);
}

void trace_pair(const DProductRep& pb, const DProductRep& pd, double* out, bool accumulate, bool with_corr) {
    const int tau = pb.tau();
    const i64 n = pb.n();
    const DTree& t = *pb.base.tree;
    const bool same = &pb == &pd;  // tr((A^-1 dA)^2): mirrored terms computed once
    hodlr_trace_product(pb.base, pd.base, out, accumulate);
    if (!with_corr) return;
    // Cross terms sum_i tr(Cv_i^T h_{>=i} Cu_i) (product_rep.cpp:212-224),
    // regrouped by the level of h: the leaves act on every correction, level
    // l on corrections i <= l, i.e. on the column prefix W_l of Cu / Cv, so
    //   sum = tr(Cv^T Leaves Cu) + sum_l sum_s <U_l[s]^T Cv_{<=l}[s], V_l[s^1]^T Cu_{<=l}[s^1]>
    // (two projections per level and a sibling dot; no n x C products).
    auto cross = [&](const DHodlr& h, const DProductRep& corr, double alpha) {
        if (!corr.sumC) return;
        if (!h.leaves_zero)  // tr(Cv^T Leaves Cu), the leaf products reduced in the GEMM epilogue
            leaf_mm_dot(t.leaves(), h.leaves->get(), h.lstride(), h.bmax(), corr.Cu->get(), n, corr.Cv->get(), n,
                        corr.sumC, alpha, out, true);
        // Thin levels (rank <= 16: the sigma^2 derivative everywhere, the ell
        // derivative on all but its deepest levels) take their projections of
        // Cv / Cu together in one pass (hodlr_project -> k_proj_cat); wider
        // levels one segmented GEMM pair each.
        std::vector<int> W(static_cast<size_t>(tau), 0);
        bool any_thin = false;
        for (int l = 1; l <= tau; ++l) {
            const int R = h.Rl(l);
            const int w = corr.coff[static_cast<size_t>(l - 1)] + corr.C[static_cast<size_t>(l - 1)];
            if (R > 0 && R <= 16 && w > 0) {
                W[static_cast<size_t>(l - 1)] = w;
                any_thin = true;
            }
        }
        if (any_thin) {
            auto P = hodlr_project(h, corr.Cv->get(), n, corr.sumC, true, W);
            auto Q = hodlr_project(h, corr.Cu->get(), n, corr.sumC, false, W);
            for (int l = 1; l <= tau; ++l) {
                const int R = h.Rl(l), w = W[static_cast<size_t>(l - 1)];
                if (!R || !w) continue;
                const Partition& p = t.part(l);
                for (int rep = 0; rep < int(alpha); ++rep)  // alpha in {1, 2}
                    seg_xor_dot(p.nseg(), 1, P[static_cast<size_t>(l - 1)]->get(), Q[static_cast<size_t>(l - 1)]->get(),
                                i64(R) * corr.sumC, R, R, w, out, true);
            }
        }
        for (int l = 1; l <= tau; ++l) {
            const int R = h.Rl(l);
            const int Wl = corr.coff[static_cast<size_t>(l - 1)] + corr.C[static_cast<size_t>(l - 1)];
            if (!R || !Wl || W[static_cast<size_t>(l - 1)]) continue;
            const Partition& p = t.part(l);
            const size_t sz = static_cast<size_t>(p.nseg()) * static_cast<size_t>(R) * static_cast<size_t>(Wl);
            DVec P(sz), Q(sz);
            seg_tn(p, h.Ul(l), n, R, corr.Cv->get(), n, Wl, P.get(), i64(R) * Wl, R, alpha);
            seg_tn(p, h.Vl(l), n, R, corr.Cu->get(), n, Wl, Q.get(), i64(R) * Wl, R);
            seg_xor_dot(p.nseg(), 1, P.get(), Q.get(), i64(R) * Wl, R, R, Wl, out, true);
        }
    };
    if (same) {
        cross(pb.base, pb, 2.0);
    } else {
        cross(pb.base, pd, 1.0);
        cross(pd.base, pb, 1.0);
    }
    // Correction pairs aligned by the finer level (product_rep.cpp:159-176,227-233):
    // coarse levels [c0, c0+W) columns of one operand against fine level f of the other.
    auto pairs = [&](const DProductRep& coarse, int c0, int W, const DProductRep& fine, int f, double alpha) {
        const int Cf = fine.C[static_cast<size_t>(f - 1)];
        if (!W || !Cf) return;
        const Partition& p = t.part(f - 1);
        const size_t sz = static_cast<size_t>(p.nseg()) * static_cast<size_t>(W) * static_cast<size_t>(Cf);
        DVec G1(sz), G2(sz);
        seg_tn(p, coarse.Cv->get() + i64(c0) * n, n, W, fine.Cul(f), n, Cf, G1.get(), i64(W) * Cf, W, alpha);
        // G2 = (Cv_f^T Cu_c)^T formed directly as Cu_c^T Cv_f: tr(G1 G2) is then a contiguous dot
        seg_tn(p, coarse.Cu->get() + i64(c0) * n, n, W, fine.Cvl(f), n, Cf, G2.get(), i64(W) * Cf, W);
        seg_dot(1, 0, G1.get(), 0, G2.get(), 0, i64(p.nseg()) * W * Cf, out, true);
    };
    for (int f = 1; f <= tau; ++f) {
        const int cf = pb.coff[static_cast<size_t>(f - 1)];
        if (same) {  // sum_{i<=f} + sum_{i<f} = 2 sum_{i<f} + (i = f)
            pairs(pb, 0, cf, pb, f, 2.0);
            pairs(pb, cf, pb.C[static_cast<size_t>(f - 1)], pb, f, 1.0);
        } else {
            pairs(pb, 0, cf + pb.C[static_cast<size_t>(f - 1)], pd, f, 1.0);  // i <= j: coarse from pb
            pairs(pd, 0, pd.coff[static_cast<size_t>(f - 1)], pb, f, 1.0);    // i > j: coarse from pd
        }
    }
}

std::vector<double> fisher_corrections(const std::vector<DProductRep>& reps) {
    const size_t p = reps.size();
    std::vector<double> out(p * p, 0.0);
    if (p == 0 || !reps[0].sumC) return out;
    const int tau = reps[0].tau();
    const i64 n = reps[0].n();
    const DTree& t = *reps[0].base.tree;
    for (const auto& r : reps)
        if (r.C != reps[0].C || r.n() != n) throw std::invalid_argument("fisher_corrections: reps of different factorizations");
    // cc[i + j p] = sum_f <Cv_i[<f]^T Cu_f, Cu[<f]^T Cv_j,f>, ss likewise over
    // the level-f columns themselves (product_rep.cpp:227-233: i <= j pairs
    // align by the finer level; the i = f term appears once, i < f twice for
    // a rep with itself)
    DVec cc(p * p), ss(p * p);
    cc.zero();
    ss.zero();
    for (int f = 1; f <= tau; ++f) {
        const int Cf = reps[0].C[static_cast<size_t>(f - 1)];
        const int cf = reps[0].coff[static_cast<size_t>(f - 1)];
        if (!Cf) continue;
        const Partition& pt = t.part(f - 1);
        const i64 nseg = pt.nseg();
        std::vector<DVec> G1c(p), G2c(p), G1s(p), G2s(p);
        for (size_t a = 0; a < p; ++a) {
            const DProductRep& r = reps[a];
            if (cf) {
                G1c[a].alloc(static_cast<size_t>(nseg) * cf * Cf);
                G2c[a].alloc(static_cast<size_t>(nseg) * cf * Cf);
                seg_tn(pt, r.Cv->get(), n, cf, r.Cul(f), n, Cf, G1c[a].get(), i64(cf) * Cf, cf);
                // (Cv_f^T Cu_c)^T formed directly as Cu_c^T Cv_f: the pair terms are contiguous dots
                seg_tn(pt, r.Cu->get(), n, cf, r.Cvl(f), n, Cf, G2c[a].get(), i64(cf) * Cf, cf);
            }
            G1s[a].alloc(static_cast<size_t>(nseg) * Cf * Cf);
            G2s[a].alloc(static_cast<size_t>(nseg) * Cf * Cf);
            seg_tn(pt, r.Cvl(f), n, Cf, r.Cul(f), n, Cf, G1s[a].get(), i64(Cf) * Cf, Cf);
            seg_tn(pt, r.Cul(f), n, Cf, r.Cvl(f), n, Cf, G2s[a].get(), i64(Cf) * Cf, Cf);
        }
        const i64 lc = nseg * i64(cf) * Cf, ls = nseg * i64(Cf) * Cf;
        for (size_t i = 0; i < p; ++i)
            for (size_t j = 0; j < p; ++j) {  // cc needs every ordered pair, ss only i <= j
                if (cf) seg_dot(1, 0, G1c[i].get(), 0, G2c[j].get(), 0, lc, cc.get() + i + j * p, true);
                if (i <= j) seg_dot(1, 0, G1s[i].get(), 0, G2s[j].get(), 0, ls, ss.get() + i + j * p, true);
            }
    }
    // Cross terms (product_rep.cpp:212-224) of every pair: for base a and the
    // corrections of rep b, tr(Cv_b^T h_a Cu) with the shared Cu. The leaf
    // product Leaves_a Cu is formed once per base and dotted with every Cv_b;
    // the projections V_l^T Cu once per base, U_l^T Cv_b per (a, b). A pair
    // (i, j), i < j, takes cross(base i, rep j) + cross(base j, rep i); (i, i)
    // takes 2 cross(base i, rep i) (trace_pair's mirrored-term rule).
    DVec xc(p * p);
    xc.zero();
    const int sumC = reps[0].sumC;
    const DProductRep& r0 = reps[0];
    {  // leaf parts: tr(Cv_b^T Leaves_a Cu) = sum_leaves <Leaves_a, Cv_b Cu^T>; the per-leaf
       // Grams Cv_b Cu^T (K = sumC) are formed once per b and dotted with every base's leaves
        std::vector<const double*> As, Ls;
        std::vector<size_t> la;
        for (size_t b = 0; b < p; ++b) As.push_back(reps[b].Cv->get());
        for (size_t a = 0; a < p; ++a)
            if (!reps[a].base.leaves_zero) {
                Ls.push_back(reps[a].base.leaves->get());
                la.push_back(a);
            }
        if (!Ls.empty() && p <= size_t(LEAF_DOT_MAXZ)) {
            std::vector<double*> os;
            for (size_t b = 0; b < p; ++b)
                for (size_t ia = 0; ia < la.size(); ++ia) os.push_back(xc.get() + la[ia] + b * p);
            leaf_gram_dot(t.leaves(), As, r0.Cu->get(), n, sumC, Ls, r0.base.lstride(), r0.base.bmax(), os, true);
        } else {
            for (size_t a : la) {
                std::vector<const double*> zs;
                std::vector<double> al;
                std::vector<double*> os;
                for (size_t b = 0; b < p; ++b) {
                    zs.push_back(reps[b].Cv->get());
                    al.push_back(1.0);
                    os.push_back(xc.get() + a + b * p);
                }
                leaf_mm_dot_multi(t.leaves(), reps[a].base.leaves->get(), reps[a].base.lstride(), reps[a].base.bmax(),
                                  r0.Cu->get(), n, zs, n, sumC, al, os, true);
            }
        }
    }
    for (size_t a = 0; a < p; ++a) {
        const DHodlr& h = reps[a].base;
        auto slot = [&](size_t b) { return xc.get() + a + b * p; };  // cross(base a, rep b)
        std::vector<int> W(static_cast<size_t>(tau), 0);
        bool any_thin = false;
        for (int l = 1; l <= tau; ++l) {
            const int R = h.Rl(l);
            const int w = r0.coff[static_cast<size_t>(l - 1)] + r0.C[static_cast<size_t>(l - 1)];
            if (R > 0 && R <= 16 && w > 0) {
                W[static_cast<size_t>(l - 1)] = w;
                any_thin = true;
            }
        }
        if (any_thin) {
            auto Q = hodlr_project(h, r0.Cu->get(), n, sumC, false, W);
            for (size_t b = 0; b < p; ++b) {
                auto Pp = hodlr_project(h, reps[b].Cv->get(), n, sumC, true, W);
                for (int l = 1; l <= tau; ++l) {
                    const int R = h.Rl(l), w = W[static_cast<size_t>(l - 1)];
                    if (!R || !w) continue;
                    seg_xor_dot(t.part(l).nseg(), 1, Pp[static_cast<size_t>(l - 1)]->get(),
                                Q[static_cast<size_t>(l - 1)]->get(), i64(R) * sumC, R, R, w, slot(b), true);
                }
            }
        }
        for (int l = 1; l <= tau; ++l) {
            const int R = h.Rl(l);
            const int Wl = r0.coff[static_cast<size_t>(l - 1)] + r0.C[static_cast<size_t>(l - 1)];
            if (!R || !Wl || W[static_cast<size_t>(l - 1)]) continue;
            const Partition& pl = t.part(l);
            const size_t sz = static_cast<size_t>(pl.nseg()) * static_cast<size_t>(R) * static_cast<size_t>(Wl);
            DVec Q(sz);
            seg_tn(pl, h.Vl(l), n, R, r0.Cu->get(), n, Wl, Q.get(), i64(R) * Wl, R);
            for (size_t b = 0; b < p; ++b) {
                DVec Pp(sz);
                seg_tn(pl, h.Ul(l), n, R, reps[b].Cv->get(), n, Wl, Pp.get(), i64(R) * Wl, R);
                seg_xor_dot(pl.nseg(), 1, Pp.get(), Q.get(), i64(R) * Wl, R, R, Wl, slot(b), true);
            }
        }
    }
    const std::vector<double> c = cc.download(), q = ss.download(), x = xc.download();
    for (size_t i = 0; i < p; ++i)
        for (size_t j = i; j < p; ++j)
            out[i + j * p] = i == j ? 2.0 * c[i + i * p] + q[i + i * p] + 2.0 * x[i + i * p]
                                    : c[i + j * p] + q[i + j * p] + c[j + i * p] + x[i + j * p] + x[j + i * p];
    return out;
}

std::vector<double> prodrep_densify(const DProductRep& p) {
    const i64 n = p.n();
    if (n > (i64(1) << 14)) throw std::length_error("densify: matrix too large");
    std::vector<double> flat(p.base.export_size());
    std::vector<int> ru(static_cast<size_t>(std::max<i64>((i64(1) << p.tau()) - 1, 1))), rl(ru.size());
    p.base.export_panels(flat.data(), ru.data(), rl.data());
    std::vector<double> a(static_cast<size_t>(n) * static_cast<size_t>(n), 0.0);
    const ClusterTree& t = p.base.tree->host;
    size_t off = 0;
    for (int l = 1; l <= p.tau(); ++l) {
        const int R = p.base.Rl(l);
        const double* U = flat.data() + off;
        const double* V = U + static_cast<size_t>(n) * static_cast<size_t>(R);
        off += 2 * static_cast<size_t>(n) * static_cast<size_t>(R);
        const auto& kids = t.level(l);
        for (size_t j = 0; j < kids.size() / 2; ++j) {
            const Range cl = kids[2 * j], cr = kids[2 * j + 1];
            auto blk = [&](Range rows, Range cols) {
                for (i64 c = cols.lo; c < cols.hi; ++c)
                    for (i64 r = rows.lo; r < rows.hi; ++r) {
                        double s = 0;
                        for (int q = 0; q < R; ++q) s += U[r + q * n] * V[c + q * n];
                        a[static_cast<size_t>(r + c * n)] = s;
                    }
            };
            blk(cl, cr);
            blk(cr, cl);
        }
    }
    for (const Range& r : t.leaves()) {
        const i64 m = r.size();
        for (i64 c = 0; c < m; ++c)
            for (i64 q = 0; q < m; ++q) a[static_cast<size_t>(r.lo + q + (r.lo + c) * n)] = flat[off + static_cast<size_t>(q + c * m)];
        off += static_cast<size_t>(m * m);
    }
    std::vector<double> cu = p.Cu->download(), cv = p.Cv->download();
    for (int i = 1; i <= p.tau(); ++i) {
        const int Ci = p.C[static_cast<size_t>(i - 1)];
        if (!Ci) continue;
        const size_t co = static_cast<size_t>(p.coff[static_cast<size_t>(i - 1)]) * static_cast<size_t>(n);
        for (const Range& r : t.level(i - 1))
            for (i64 c = r.lo; c < r.hi; ++c)
                for (i64 q = r.lo; q < r.hi; ++q) {
                    double s = 0;
                    for (int k = 0; k < Ci; ++k) s += cu[co + static_cast<size_t>(q + k * n)] * cv[co + static_cast<size_t>(c + k * n)];
                    a[static_cast<size_t>(q + c * n)] += s;
                }
    }
    return a;
}

}  // namespace hg
