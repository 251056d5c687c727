// Batched Householder QR (optionally column-pivoted, Eigen 3.4
// ColPivHouseholderQR semantics) and thin-Q formation, one CTA per block.
//
// Used by the sketch build for the per-node range finder (sketch.cpp:37-76),
// the q2 residual basis (sketch.cpp:194-225) and the rank-revealing
// recompression of derivative blocks (hodlr_matrix.cpp:42-66).
#pragma once

#include "kernels.cuh"

namespace hg {

/// Early termination of a pivoted QR whose caller only reads the leading
/// diagonal up to the first |R(s,s)| <= max(rel |R(0,0)|, abs_scale *abs_ptr)
/// (or up to max_steps): the factorization stops after that step; later
/// taus are 0 (identity reflectors), later R rows and pivots are unspecified.
/// The columns the caller reads are bitwise those of the full factorization.
struct QrStop {
    double rel = 0.0;
    double abs_scale = 0.0;
    const double* abs_ptr = nullptr;  // device scalar, may be null
    int max_steps = 1 << 30;
    bool active = false;
};

struct QrDesc {
    double* A;    // block (rows x w), ld lda; overwritten by R (upper) + essentials
    i64 lda;
    int rows;
    double* tau;  // w
    double* R;    // w x w (ld ldr), may be null
    int ldr;
    int* perm;    // w (pivoted only)
    QrStop stop = {};
};

/// QR of every block (all blocks have w columns). Pivoting follows Eigen:
/// max updated norm (first index on ties), LAPACK xGEQPF downdating at sqrt(eps).
void batched_qr(const std::vector<QrDesc>& blocks, int w, bool pivot);

struct QfDesc {
    const double* A;  // Householder storage from batched_qr
    i64 lda;
    int rows;
    const double* tau;
    const double* Tin;  // top block (nref x qcols, ld ldt); null = identity
    int ldt;
    double* Q;  // out: rows x qcols, ld ldq
    i64 ldq;
};

/// Q_b = H_0 ... H_{nref-1} [Tin; 0] for every block (nref = min(w, rows)).
void batched_form_q(const std::vector<QfDesc>& blocks, int w, int qcols);

}  // namespace hg

namespace hg {

/// Tall-skinny batched QR: blocks longer than the chunk height are reduced by
/// a TSQR tree (unpivoted chunk QRs, R factors stacked, repeated), and the
/// final per-block matrix gets the (optionally pivoted) QR. Equivalent to a
/// direct (pivoted) Householder QR of each block: the pivot choice reads the
/// same column norms, and Q is recovered by applying the tree top-down.
/// Blocks of at most this many rows (w columns) are factored by one CTA
/// directly; taller ones go through the TSQR tree.
int qr_chunk_rows(int w);

class BatchedQR {
public:
    struct Block {
        double* A;
        i64 lda;
        int rows;
        QrStop stop = {};  // pivoted top-level QR only
    };
    BatchedQR(const std::vector<Block>& blocks, int w, bool pivot);
    int w() const { return w_; }
    int count() const { return int(blocks_.size()); }
    /// Final R of block b: w x w (ld w) at R() + b*w*w; column perm at perm() + b*w.
    const double* R() const { return R_.get(); }
    const int* perm() const { return perm_.get(); }
    /// Q_b [Tin_b; 0] restricted to qcols columns, written to Q[b] (ld ldq[b]).
    /// Tin (w x qcols per block, ld ldt, stride tstride) may be null (identity).
    void form_q(int qcols, const double* Tin, i64 tstride, int ldt, const std::vector<double*>& Q,
                const std::vector<i64>& ldq) const;

private:
    struct Chunk {
        int level;       // tree level of the stack this chunk's R went to (its parent)
        int parent;      // index of the parent node in that level's node list
        int index;       // chunk index inside the parent stack
        QrDesc desc;     // Householder data location
    };
    struct Node {        // a matrix factored at some level: an input block or a stack
        double* A;
        i64 lda;
        int rows;
        int block;       // original block id
    };
    int w_;
    bool pivot_;
    std::vector<Block> blocks_;
    std::vector<std::vector<Node>> nodes_;    // nodes_[L]: matrices entering level L
    std::vector<std::vector<Chunk>> chunks_;  // chunks_[L]: chunk QRs of level L (parents at L+1)
    std::vector<int> top_node_;               // per block: node index at its top level
    std::vector<int> top_level_;
    std::vector<DVecP> stacks_, taus_;
    DVec R_, top_tau_;
    DBuf<int> perm_;
};

}  // namespace hg
