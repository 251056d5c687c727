// Cluster tree (host, bit-exact with the reference) and its device-side
// partitions: for every depth d the 2^d contiguous row ranges, plus cached
// work lists that tile each range without crossing a range boundary.
//
// Reference: cluster_tree.hpp:24-71, cluster_tree.cpp:10-90.
#pragma once

#include "common.cuh"

namespace hg {

struct Range {
    i64 lo = 0, hi = 0;
    i64 size() const { return hi - lo; }
};

/// cluster_tree.cpp:10-22: uniform binary bisection, left child ceil(len/2).
class ClusterTree {
public:
    ClusterTree() = default;
    ClusterTree(i64 n, int tau);
    i64 size() const { return n_; }
    int depth() const { return tau_; }
    const std::vector<Range>& level(int d) const { return levels_[static_cast<size_t>(d)]; }
    const std::vector<Range>& leaves() const { return levels_[static_cast<size_t>(tau_)]; }
    i64 num_leaves() const { return i64(levels_[static_cast<size_t>(tau_)].size()); }
    i64 max_leaf_size() const;
    bool same_structure(const ClusterTree& o) const { return n_ == o.n_ && tau_ == o.tau_; }

private:
    i64 n_ = 0;
    int tau_ = 0;
    std::vector<std::vector<Range>> levels_;
};

/// cluster_tree.cpp:34-38
int tree_depth(i64 n, i64 leaf_min, i64 leaf_max);

struct KdOrdering {
    std::vector<i64> perm, inv;
    ClusterTree tree;
};
/// cluster_tree.cpp:40-90 (host; O(n log^2 n) compare-only work, bit-exact).
KdOrdering build_kd_ordering(const double* coords, i64 n, int d, i64 leaf_min, i64 leaf_max);

/// Work item of a segmented kernel: rows [row0, row0+rows) of segment seg.
struct WorkItem {
    int seg, row0, rows, pad;
};

struct TileList {
    int count = 0;
    bool one_per_seg = true;
    DBuf<WorkItem> items;
    DBuf<int> seg_first;  // nseg+1: items of segment s are [seg_first[s], seg_first[s+1])
};

/// The 2^d row ranges of depth d.
class Partition {
public:
    Partition(const ClusterTree& t, int d);
    /// nseg equal segments of `len` rows (batched per-node small matrices).
    Partition(int nseg, int len);
    /// Explicit segment bounds (nseg + 1 nondecreasing row offsets).
    explicit Partition(const std::vector<int>& bounds);
    int depth() const { return depth_; }
    int nseg() const { return nseg_; }
    const std::vector<int>& hbounds() const { return hb_; }
    const int* dbounds() const { return db_.get(); }
    int max_seg() const { return max_seg_; }
    /// Items of at most `rows` rows (cached).
    const TileList& tiles(int rows) const;

private:
    int depth_ = 0, nseg_ = 0, max_seg_ = 0;
    std::vector<int> hb_;
    DBuf<int> db_;
    mutable std::map<int, std::unique_ptr<TileList>> cache_;
};

/// Tree plus its device partitions (immutable, shared by every object on it).
struct DTree {
    ClusterTree host;
    std::vector<std::unique_ptr<Partition>> parts;  // parts[d], d = 0..tau
    int bmax = 0;                                    // max leaf size
    i64 n() const { return host.size(); }
    int tau() const { return host.depth(); }
    const Partition& part(int d) const { return *parts[static_cast<size_t>(d)]; }
    const Partition& leaves() const { return *parts[static_cast<size_t>(tau())]; }
};
using DTreeP = std::shared_ptr<const DTree>;

/// Cached per (n, tau) on the current device.
DTreeP get_tree(i64 n, int tau);

/// Cached uniform partition (nseg segments of len rows).
const Partition& uniform_partition(int nseg, int len);

}  // namespace hg
