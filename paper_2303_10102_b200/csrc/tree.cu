// Cluster tree + device partitions. Reference: cluster_tree.cpp:10-90.
#include <algorithm>
#include <cmath>
#include <mutex>
#include <numeric>

#include "tree.cuh"

namespace hg {

namespace {
thread_local Ctx* g_ctx = nullptr;
Ctx g_default;
}  // namespace

Ctx& current() { return g_ctx ? *g_ctx : g_default; }
void set_current(Ctx* c) { g_ctx = c; }

// cluster_tree.cpp:10-22
ClusterTree::ClusterTree(i64 n, int tau) : n_(n), tau_(tau) {
    levels_.resize(static_cast<size_t>(tau + 1));
    levels_[0] = {Range{0, n}};
    for (int d = 1; d <= tau; ++d) {
        levels_[static_cast<size_t>(d)].reserve(static_cast<size_t>(1) << d);
        for (const Range& p : levels_[static_cast<size_t>(d - 1)]) {
            i64 left = (p.size() + 1) / 2;
            levels_[static_cast<size_t>(d)].push_back(Range{p.lo, p.lo + left});
            levels_[static_cast<size_t>(d)].push_back(Range{p.lo + left, p.hi});
        }
    }
}

i64 ClusterTree::max_leaf_size() const {
    i64 m = 0;
    for (const Range& r : leaves()) m = std::max(m, r.size());
    return m;
}

// cluster_tree.cpp:34-38
int tree_depth(i64 n, i64 leaf_min, i64 leaf_max) {
    if (n <= leaf_max) return 0;
    int tau = int(std::floor(std::log2(double(n) / double(leaf_min))));
    return std::max(tau, 1);
}

// cluster_tree.cpp:40-90
KdOrdering build_kd_ordering(const double* c, i64 n, int d, i64 leaf_min, i64 leaf_max) {
    if (n < 1) throw std::invalid_argument("build_kd_ordering: empty point set");
    if (d != 1 && d != 2) throw std::invalid_argument("build_kd_ordering: d must be 1 or 2");
    if (leaf_min < 1 || leaf_min > leaf_max)
        throw std::invalid_argument("build_kd_ordering: need 1 <= leaf_min <= leaf_max");
    for (i64 i = 0; i < n * d; ++i)
        if (!std::isfinite(c[i])) throw std::invalid_argument("build_kd_ordering: non-finite coordinates");
    auto at = [&](i64 i, int k) { return c[i + k * n]; };
    KdOrdering out;
    out.tree = ClusterTree(n, tree_depth(n, leaf_min, leaf_max));
    std::vector<i64> order(static_cast<size_t>(n));
    std::iota(order.begin(), order.end(), i64{0});
    for (int depth = 0; depth < out.tree.depth(); ++depth)
        for (const auto& node : out.tree.level(depth)) {
            auto first = order.begin() + node.lo, last = order.begin() + node.hi;
            int axis = 0;
            if (d == 2) {
                double lo0 = at(*first, 0), hi0 = lo0, lo1 = at(*first, 1), hi1 = lo1;
                for (auto it = first; it != last; ++it) {
                    lo0 = std::min(lo0, at(*it, 0));
                    hi0 = std::max(hi0, at(*it, 0));
                    lo1 = std::min(lo1, at(*it, 1));
                    hi1 = std::max(hi1, at(*it, 1));
                }
                axis = (hi1 - lo1) > (hi0 - lo0) ? 1 : 0;
            }
            std::stable_sort(first, last, [&](i64 a, i64 b) {
                if (at(a, axis) != at(b, axis)) return at(a, axis) < at(b, axis);
                return a < b;
            });
        }
    out.inv = order;
    out.perm.resize(static_cast<size_t>(n));
    for (i64 pos = 0; pos < n; ++pos) out.perm[static_cast<size_t>(order[static_cast<size_t>(pos)])] = pos;
    return out;
}

Partition::Partition(const ClusterTree& t, int d) : depth_(d) {
    const auto& lv = t.level(d);
    nseg_ = int(lv.size());
    hb_.resize(static_cast<size_t>(nseg_ + 1));
    for (int s = 0; s < nseg_; ++s) {
        hb_[static_cast<size_t>(s)] = int(lv[static_cast<size_t>(s)].lo);
        max_seg_ = std::max(max_seg_, int(lv[static_cast<size_t>(s)].size()));
    }
    hb_[static_cast<size_t>(nseg_)] = int(t.size());
    db_.upload(hb_);
}

Partition::Partition(int nseg, int len) : depth_(-1), nseg_(nseg), max_seg_(len) {
    hb_.resize(static_cast<size_t>(nseg + 1));
    for (int s = 0; s <= nseg; ++s) hb_[static_cast<size_t>(s)] = s * len;
    db_.upload(hb_);
}

Partition::Partition(const std::vector<int>& bounds) : depth_(-1), nseg_(int(bounds.size()) - 1), hb_(bounds) {
    for (int s = 0; s < nseg_; ++s)
        max_seg_ = std::max(max_seg_, hb_[static_cast<size_t>(s + 1)] - hb_[static_cast<size_t>(s)]);
    db_.upload(hb_);
}

const Partition& uniform_partition(int nseg, int len) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int>, std::unique_ptr<Partition>> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(current().device, nseg, len);
    auto it = cache.find(key);
    if (it != cache.end()) return *it->second;
    auto p = std::make_unique<Partition>(nseg, len);
    auto& ref = *p;
    cache[key] = std::move(p);
    return ref;
}

const TileList& Partition::tiles(int rows) const {
    auto it = cache_.find(rows);
    if (it != cache_.end()) return *it->second;
    auto tl = std::make_unique<TileList>();
    std::vector<WorkItem> items;
    std::vector<int> first(static_cast<size_t>(nseg_ + 1));
    for (int s = 0; s < nseg_; ++s) {
        first[static_cast<size_t>(s)] = int(items.size());
        int lo = hb_[static_cast<size_t>(s)], hi = hb_[static_cast<size_t>(s + 1)];
        int cnt = 0;
        for (int r = lo; r < hi; r += rows) {
            items.push_back(WorkItem{s, r, std::min(rows, hi - r), 0});
            ++cnt;
        }
        if (cnt == 0) {
            items.push_back(WorkItem{s, lo, 0, 0});
            cnt = 1;
        }
        if (cnt > 1) tl->one_per_seg = false;
    }
    first[static_cast<size_t>(nseg_)] = int(items.size());
    tl->count = int(items.size());
    tl->items.upload(items);
    tl->seg_first.upload(first);
    auto& ref = *tl;
    cache_[rows] = std::move(tl);
    return ref;
}

DTreeP get_tree(i64 n, int tau) {
    static std::mutex mu;
    static std::map<std::tuple<int, i64, int>, DTreeP> cache;
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(current().device, n, tau);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (n >= (i64(1) << 31)) throw std::length_error("tree: n must be < 2^31");
    auto t = std::make_shared<DTree>();
    t->host = ClusterTree(n, tau);
    for (int d = 0; d <= tau; ++d) t->parts.push_back(std::make_unique<Partition>(t->host, d));
    t->bmax = int(t->host.max_leaf_size());
    cache[key] = t;
    return t;
}

}  // namespace hg
