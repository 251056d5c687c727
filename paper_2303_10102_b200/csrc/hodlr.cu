// Device HODLR container, matvec family, traces (hodlr_matrix.cpp).
#include <algorithm>
#include <cmath>
#include <random>

#include "hodlr.cuh"

namespace hg {

namespace {

__global__ void k_leaf_ggt(const int* bounds, int bmax, const double* g, double* out, double shift, int mode) {
    // mode 0: out = 0.5 (g + g^T); mode 1: out = g g^T + shift I
    const int b = blockIdx.x;
    const int m = bounds[b + 1] - bounds[b];
    const double* G = g + i64(b) * bmax * bmax;
    double* O = out + i64(b) * bmax * bmax;
    for (int e = threadIdx.x; e < m * m; e += blockDim.x) {
        const int i = e % m, j = e / m;
        double v;
        if (mode == 0) {
            v = 0.5 * (G[i + i64(j) * bmax] + G[j + i64(i) * bmax]);
        } else {
            v = 0.0;
            for (int p = 0; p < m; ++p) v = fma(G[i + i64(p) * bmax], G[j + i64(p) * bmax], v);
            if (i == j) v += shift;
        }
        O[i + i64(j) * bmax] = v;
    }
}

__global__ void k_leaves_panel(const int* bounds, int bmax, double* leaves, double* P, i64 ldp, int to_panel) {
    const int b = blockIdx.x;
    const int lo = bounds[b], m = bounds[b + 1] - lo;
    double* L = leaves + i64(b) * bmax * bmax;
    for (int e = threadIdx.x; e < m * bmax; e += blockDim.x) {
        const int r = e % m, c = e / m;
        if (to_panel)
            P[i64(lo + r) + i64(c) * ldp] = c < m ? L[r + i64(c) * bmax] : 0.0;
        else if (c < m)
            L[r + i64(c) * bmax] = P[i64(lo + r) + i64(c) * ldp];
    }
}

}  // namespace

void leaves_panel(const DTree& t, double* leaves, double* P, bool to_panel) {
    const Partition& lv = t.leaves();
    k_leaves_panel<<<unsigned(lv.nseg()), 256, 0, current().stream>>>(lv.dbounds(), t.bmax, leaves, P, t.n(),
                                                                       to_panel ? 1 : 0);
    HG_LAUNCH();
    count_launch();
}

DHodlr DHodlr::zero(DTreeP t, bool symmetric) {
    DHodlr h;
    h.tree = t;
    h.sym = symmetric;
    const int tau = t->tau();
    h.R.assign(static_cast<size_t>(tau), 0);
    h.U.assign(static_cast<size_t>(tau), nullptr);
    h.V.assign(static_cast<size_t>(tau), nullptr);
    h.rank_up.resize(static_cast<size_t>(tau));
    h.rank_lo.resize(static_cast<size_t>(tau));
    for (int l = 1; l <= tau; ++l) {
        h.rank_up[static_cast<size_t>(l - 1)].assign(static_cast<size_t>(1) << (l - 1), 0);
        h.rank_lo[static_cast<size_t>(l - 1)].assign(static_cast<size_t>(1) << (l - 1), 0);
    }
    h.leaves = make_dvec(static_cast<size_t>(t->leaves().nseg()) * static_cast<size_t>(h.lstride()), true);
    h.leaves_zero = true;
    return h;
}

DHodlr DHodlr::identity(DTreeP t) {
    DHodlr h = zero(t);
    std::vector<double> lv(h.leaves->size(), 0.0);
    const auto& hb = t->leaves().hbounds();
    for (int b = 0; b < t->leaves().nseg(); ++b)
        for (int i = 0; i < hb[static_cast<size_t>(b + 1)] - hb[static_cast<size_t>(b)]; ++i)
            lv[static_cast<size_t>(b) * static_cast<size_t>(h.lstride()) + static_cast<size_t>(i) * static_cast<size_t>(h.bmax() + 1)] = 1.0;
    h.leaves->upload(lv);
    h.leaves_zero = false;
    return h;
}

void DHodlr::set_level(int l, int r, bool symmetric_panel) {
    R[static_cast<size_t>(l - 1)] = r;
    U[static_cast<size_t>(l - 1)] = r ? make_dvec(static_cast<size_t>(n()) * static_cast<size_t>(r), true) : nullptr;
    V[static_cast<size_t>(l - 1)] = symmetric_panel ? U[static_cast<size_t>(l - 1)] : (r ? make_dvec(static_cast<size_t>(n()) * static_cast<size_t>(r), true) : nullptr);
}

// hodlr_matrix.cpp:126-172
DHodlr DHodlr::random(DTreeP t, i64 k, std::uint64_t seed, bool spd) {
    const ClusterTree& tree = t->host;
    DHodlr h = zero(t);
    const i64 n = tree.size();
    std::mt19937_64 rng(seed);
    std::normal_distribution<double> gauss(0.0, 1.0);
    for (int l = 1; l <= tree.depth(); ++l) {
        const auto& kids = tree.level(l);
        const size_t nodes = tree.level(l - 1).size();
        int Rl = 0;
        for (size_t j = 0; j < nodes; ++j)
            Rl = std::max<int>(Rl, int(std::min({k, kids[2 * j].size(), kids[2 * j + 1].size()})));
        std::vector<double> P(static_cast<size_t>(n) * static_cast<size_t>(Rl), 0.0);
        for (size_t j = 0; j < nodes; ++j) {
            const Range cl = kids[2 * j], cr = kids[2 * j + 1];
            const i64 r = std::min({k, cl.size(), cr.size()});
            const double s1 = std::sqrt(double(cl.size())), s2 = std::sqrt(double(cr.size()));
            for (i64 i = 0; i < cl.size(); ++i)
                for (i64 c = 0; c < r; ++c) P[static_cast<size_t>(cl.lo + i + c * n)] = gauss(rng) / s1;
            for (i64 i = 0; i < cr.size(); ++i)
                for (i64 c = 0; c < r; ++c) P[static_cast<size_t>(cr.lo + i + c * n)] = gauss(rng) / s2;
            h.rank_up[static_cast<size_t>(l - 1)][j] = int(r);
            h.rank_lo[static_cast<size_t>(l - 1)][j] = int(r);
        }
        h.set_level(l, Rl, true);
        if (Rl) h.U[static_cast<size_t>(l - 1)]->upload(P);
    }
    const int bmax = h.bmax();
    std::vector<double> G(h.leaves->size(), 0.0);
    for (i64 b = 0; b < tree.num_leaves(); ++b) {
        const i64 m = tree.leaves()[static_cast<size_t>(b)].size();
        const double sm = std::sqrt(double(m));
        for (i64 i = 0; i < m; ++i)
            for (i64 j = 0; j < m; ++j) G[static_cast<size_t>(b * h.lstride() + i + j * bmax)] = gauss(rng) / sm;
    }
    DVec g;
    g.upload(G);
    const double shift = spd ? 2.0 + 2.0 * tree.depth() : 0.0;
    k_leaf_ggt<<<unsigned(tree.num_leaves()), 256, 0, current().stream>>>(t->leaves().dbounds(), bmax, g.get(),
                                                                           h.leaves->get(), shift, spd ? 1 : 0);
    HG_LAUNCH();
    count_launch();
    h.leaves_zero = false;
    return h;
}

DHodlr DHodlr::import_panels(DTreeP t, bool symmetric, const int* R, const double* flat, const int* ranks_up,
                             const int* ranks_lo) {
    DHodlr h = zero(t, symmetric);
    const i64 n = t->n();
    size_t off = 0, node = 0;
    for (int l = 1; l <= t->tau(); ++l) {
        const int Rl = R[l - 1];
        h.set_level(l, Rl, symmetric);
        if (Rl) {
            h.U[static_cast<size_t>(l - 1)]->upload(flat + off, static_cast<size_t>(n) * static_cast<size_t>(Rl));
            if (!symmetric) h.V[static_cast<size_t>(l - 1)]->upload(flat + off + static_cast<size_t>(n) * static_cast<size_t>(Rl), static_cast<size_t>(n) * static_cast<size_t>(Rl));
        }
        off += 2 * static_cast<size_t>(n) * static_cast<size_t>(Rl);
        for (size_t j = 0; j < h.rank_up[static_cast<size_t>(l - 1)].size(); ++j, ++node) {
            h.rank_up[static_cast<size_t>(l - 1)][j] = ranks_up[node];
            h.rank_lo[static_cast<size_t>(l - 1)][j] = symmetric ? ranks_up[node] : ranks_lo[node];
        }
    }
    const auto& hb = t->leaves().hbounds();
    std::vector<double> lv(h.leaves->size(), 0.0);
    bool allzero = true;
    for (int b = 0; b < t->leaves().nseg(); ++b) {
        const int m = hb[static_cast<size_t>(b + 1)] - hb[static_cast<size_t>(b)];
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i) {
                double v = flat[off + static_cast<size_t>(i) + static_cast<size_t>(j) * static_cast<size_t>(m)];
                lv[static_cast<size_t>(b) * static_cast<size_t>(h.lstride()) + static_cast<size_t>(i) + static_cast<size_t>(j) * static_cast<size_t>(h.bmax())] = v;
                if (v != 0.0) allzero = false;
            }
        off += static_cast<size_t>(m) * static_cast<size_t>(m);
    }
    h.leaves->upload(lv);
    h.leaves_zero = allzero;
    return h;
}

size_t DHodlr::export_size() const {
    size_t s = 0;
    for (int r : R) s += 2 * static_cast<size_t>(n()) * static_cast<size_t>(r);
    const auto& hb = tree->leaves().hbounds();
    for (int b = 0; b < tree->leaves().nseg(); ++b) {
        size_t m = static_cast<size_t>(hb[static_cast<size_t>(b + 1)] - hb[static_cast<size_t>(b)]);
        s += m * m;
    }
    return s;
}

void DHodlr::export_panels(double* flat, int* ranks_up, int* ranks_lo) const {
    const i64 n = this->n();
    size_t off = 0, node = 0;
    for (int l = 1; l <= tau(); ++l) {
        const int Rl = this->Rl(l);
        const size_t cnt = static_cast<size_t>(n) * static_cast<size_t>(Rl);
        if (Rl) {
            HG_CUDA(cudaMemcpyAsync(flat + off, Ul(l), cnt * sizeof(double), cudaMemcpyDeviceToHost, current().stream));
            HG_CUDA(cudaMemcpyAsync(flat + off + cnt, Vl(l), cnt * sizeof(double), cudaMemcpyDeviceToHost,
                                    current().stream));
        }
        off += 2 * cnt;
        for (size_t j = 0; j < rank_up[static_cast<size_t>(l - 1)].size(); ++j, ++node) {
            ranks_up[node] = rank_up[static_cast<size_t>(l - 1)][j];
            ranks_lo[node] = rank_lo[static_cast<size_t>(l - 1)][j];
        }
    }
    std::vector<double> lv = leaves->download();  // synchronizes
    const auto& hb = tree->leaves().hbounds();
    for (int b = 0; b < tree->leaves().nseg(); ++b) {
        const int m = hb[static_cast<size_t>(b + 1)] - hb[static_cast<size_t>(b)];
        for (int j = 0; j < m; ++j)
            for (int i = 0; i < m; ++i)
                flat[off + static_cast<size_t>(i) + static_cast<size_t>(j) * static_cast<size_t>(m)] =
                    lv[static_cast<size_t>(b) * static_cast<size_t>(lstride()) + static_cast<size_t>(i) + static_cast<size_t>(j) * static_cast<size_t>(bmax())];
        off += static_cast<size_t>(m) * static_cast<size_t>(m);
    }
}

void DHodlr::make_asymmetric() {
    if (!sym) return;
    sym = false;
    for (int l = 1; l <= tau(); ++l) {
        V[static_cast<size_t>(l - 1)] = U[static_cast<size_t>(l - 1)];
        rank_lo[static_cast<size_t>(l - 1)] = rank_up[static_cast<size_t>(l - 1)];
    }
}

/// Reference implementation of hodlr_apply, one segmented GEMM pair per level
/// (kept for testing the level-fused kernels in mlapply.cu).
void hodlr_apply_levelwise(const DHodlr& h, const double* X, i64 ldx, int s, double* Y, i64 ldy, int lmin,
                           int lmax, bool with_leaves, bool transpose, double beta, double alpha) {
    if (s <= 0) return;
    const i64 n = h.n();
    if (with_leaves && !h.leaves_zero) {
        leaf_mm(h.tree->leaves(), h.leaves->get(), h.lstride(), h.bmax(), transpose, X, ldx, Y, ldy, s, alpha, beta);
    } else if (beta != 1.0) {
        panel_axpby(n, s, 0.0, nullptr, 0, beta, Y, ldy);
    }
    lmin = std::max(lmin, 1);
    lmax = std::min(lmax, h.tau());
    for (int l = lmin; l <= lmax; ++l) {
        const int R = h.Rl(l);
        if (R == 0) continue;
        const Partition& p = h.tree->part(l);
        const double* A = transpose ? h.Ul(l) : h.Vl(l);
        const double* B = transpose ? h.Vl(l) : h.Ul(l);
        DVec T(static_cast<size_t>(p.nseg()) * static_cast<size_t>(R) * static_cast<size_t>(s));
        seg_tn(p, A, n, R, X, ldx, s, T.get(), i64(R) * s, R);
        seg_nn(p, B, n, R, T.get(), i64(R) * s, R, TMap::sibling(), Y, ldy, s, alpha, 1.0);
    }
}

void hodlr_trace(const DHodlr& h, double* out, bool accumulate) {
    leaf_trace(h.tree->leaves(), h.leaves->get(), h.lstride(), h.bmax(), out, accumulate);
}

void hodlr_trace_product(const DHodlr& a, const DHodlr& b, double* out, bool accumulate) {
    if (!a.tree->host.same_structure(b.tree->host)) throw std::invalid_argument("trace_product: tree mismatch");
    leaf_pair_dot(a.tree->leaves(), a.leaves->get(), b.leaves->get(), a.lstride(), a.bmax(), out, accumulate);
    const i64 n = a.n();
    for (int l = 1; l <= a.tau(); ++l) {
        const int RA = a.Rl(l), RB = b.Rl(l);
        if (RA == 0 || RB == 0) continue;
        const Partition& p = a.tree->part(l);
        DVec G(static_cast<size_t>(p.nseg()) * static_cast<size_t>(RA) * static_cast<size_t>(RB)), H(static_cast<size_t>(p.nseg()) * static_cast<size_t>(RA) * static_cast<size_t>(RB));
        seg_tn(p, b.Vl(l), n, RB, a.Ul(l), n, RA, G.get(), i64(RB) * RA, RB);
        // H = (V_a^T U_b)^T formed as U_b^T V_a (RB x RA): the pair trace is a contiguous sibling dot
        seg_tn(p, b.Ul(l), n, RB, a.Vl(l), n, RA, H.get(), i64(RB) * RA, RB);
        seg_dot(p.nseg(), 1, G.get(), i64(RB) * RA, H.get(), i64(RB) * RA, i64(RB) * RA, out, true);
    }
}

}  // namespace hg

namespace hg {
DHodlr hodlr_deep_copy(const DHodlr& h) {
    DHodlr c = h;
    for (size_t i = 0; i < h.U.size(); ++i) {
        if (h.U[i]) c.U[i] = std::make_shared<DVec>(*h.U[i]);
        if (h.V[i]) c.V[i] = (h.V[i] == h.U[i]) ? c.U[i] : std::make_shared<DVec>(*h.V[i]);
    }
    c.leaves = std::make_shared<DVec>(*h.leaves);
    return c;
}
}  // namespace hg
