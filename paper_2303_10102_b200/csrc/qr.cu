// Batched (column-pivoted) Householder QR and Q formation — see qr.cuh.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>

#include "prof.cuh"
#include "qr.cuh"
#include "tile.cuh"

namespace hg {

namespace {

constexpr int QNT = 512;   // QR: more warps share each step's column updates
constexpr int FQNT = 256;  // Q formation
constexpr int MAXW = 512;
constexpr size_t QR_SMEM = 200 * 1024;
constexpr int QR_RPL = 32;  // rows per lane a trailing column may keep in registers (in-place blocks)

__device__ double qr_block_sum(double v) {
    __shared__ double sh[32];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    __syncthreads();  // sh free (previous call's readers are done)
    if (lane == 0) sh[wid] = v;
    __syncthreads();
    double t = 0.0;  // every thread folds the warp sums in the same order (identical result)
    for (int i = 0; i < int(blockDim.x >> 5); ++i) t += sh[i];
    return t;
}

__device__ __forceinline__ double warp_sum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <bool PIVOT, bool INPLACE>
__global__ void __launch_bounds__(QNT) k_qr(const QrDesc* descs, int w, int smem_elems) {
    extern __shared__ double sm[];
    __shared__ double nu[MAXW], nd[MAXW];
    __shared__ int s_best;
    __shared__ int trans[MAXW];
    const QrDesc d = descs[blockIdx.x];
    const int rows = d.rows;
    const bool use_smem = i64(rows) * w <= smem_elems;
    double* W = use_smem ? sm : d.A;
    const i64 ldw = use_smem ? rows : d.lda;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    if (use_smem)
        for (i64 e = tid; e < i64(rows) * w; e += blockDim.x) {
            const int i = int(e % rows), j = int(e / rows);
            W[i + j * ldw] = d.A[i + j * d.lda];
        }
    __syncthreads();
    const int nsz = min(rows, w);
    if (PIVOT) {
        for (int j = warp; j < w; j += nwarps) {
            double s = 0.0;
            for (int i = lane; i < rows; i += 32) s += W[i + j * ldw] * W[i + j * ldw];
            s = warp_sum(s);
            if (lane == 0) nd[j] = nu[j] = sqrt(s);
        }
        __syncthreads();
    }
    const double downdate_thr = sqrt(DBL_EPSILON);
    int steps = nsz;
    double beta0 = 0.0, stop_abs = -1.0;
    if (PIVOT && d.stop.active && d.stop.abs_ptr) stop_abs = d.stop.abs_scale * *d.stop.abs_ptr;
    for (int k = 0; k < nsz; ++k) {
        if (PIVOT) {
            if (warp == 0) {  // first index of the largest norm (Eigen's maxCoeff), warp argmax
                int best = k;
                double bv = -1.0;
                for (int j = k + lane; j < w; j += 32)
                    if (nu[j] > bv) {
                        bv = nu[j];
                        best = j;
                    }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) {
                    const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                    const int oi = __shfl_xor_sync(0xffffffffu, best, o);
                    if (ov > bv || (ov == bv && oi < best)) {
                        bv = ov;
                        best = oi;
                    }
                }
                if (lane == 0) {
                    s_best = best;
                    trans[k] = best;
                }
            }
            __syncthreads();
            const int best = s_best;
            if (best != k) {
                for (int i = tid; i < rows; i += blockDim.x) {
                    const double t = W[i + k * ldw];
                    W[i + k * ldw] = W[i + best * ldw];
                    W[i + best * ldw] = t;
                }
                if (tid == 0) {
                    double t = nu[k];
                    nu[k] = nu[best];
                    nu[best] = t;
                    t = nd[k];
                    nd[k] = nd[best];
                    nd[best] = t;
                }
            }
            __syncthreads();
        }
        double part = 0.0;
        for (int i = k + 1 + tid; i < rows; i += blockDim.x) part += W[i + k * ldw] * W[i + k * ldw];
        const double c0 = W[k + k * ldw];  // read before the sum's barriers (thread 0 rewrites it below)
        const double tail = qr_block_sum(part);
        // every thread derives the reflector from the same sum (no extra barrier)
        const bool zero = tail <= DBL_MIN;
        double tau = 0.0, div = 1.0, beta = c0;
        if (!zero) {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            div = c0 - beta;
            tau = (beta - c0) / beta;
        }
        if (tid == 0) {
            if (!zero) W[k + k * ldw] = beta;
            d.tau[k] = tau;
        }
        if (PIVOT && d.stop.active) {  // uniform: every thread holds the same beta
            if (k == 0) beta0 = fabs(beta);
            if (fabs(beta) <= fmax(d.stop.rel * beta0, stop_abs) || k + 1 >= d.stop.max_steps) {
                for (int i = k + 1 + tid; i < rows; i += blockDim.x) W[i + k * ldw] = zero ? 0.0 : W[i + k * ldw] / div;
                for (int t = k + 1 + tid; t < nsz; t += blockDim.x) d.tau[t] = 0.0;
                steps = k + 1;
                __syncthreads();
                break;
            }
        }
        // In-place (global-memory) blocks: the scaled Householder vector is
        // staged in the otherwise unused shared buffer and each trailing
        // column is held in registers between its dot product and its update
        // (one global read and one write per element instead of three reads;
        // same operations in the same order as the resident path).
        const bool staged = INPLACE && !use_smem && rows <= min(smem_elems, 32 * QR_RPL);
        for (int i = k + 1 + tid; i < rows; i += blockDim.x) {
            const double vi = zero ? 0.0 : W[i + k * ldw] / div;
            W[i + k * ldw] = vi;
            if (staged) sm[i] = vi;
        }
        __syncthreads();
        for (int j = k + 1 + warp; j < w; j += nwarps) {
            double* cj = W + j * ldw;
            if (rows - k == 1) {
                if (lane == 0) cj[k] *= (1.0 - tau);
            } else if (tau != 0.0 && staged) {
                double cr[QR_RPL];
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < QR_RPL; ++q) {
                    const int i = k + 1 + lane + 32 * q;
                    if (i < rows) {
                        cr[q] = cj[i];
                        t += sm[i] * cr[q];
                    }
                }
                t = warp_sum(t) + cj[k];
#pragma unroll
                for (int q = 0; q < QR_RPL; ++q) {
                    const int i = k + 1 + lane + 32 * q;
                    if (i < rows) {
                        cr[q] -= tau * sm[i] * t;
                        cj[i] = cr[q];
                    }
                }
                __syncwarp();
                if (lane == 0) cj[k] -= tau * t;
            } else if (tau != 0.0) {
                double t = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) t += W[i + k * ldw] * cj[i];
                t = warp_sum(t) + cj[k];
                for (int i = k + 1 + lane; i < rows; i += 32) cj[i] -= tau * W[i + k * ldw] * t;
                __syncwarp();
                if (lane == 0) cj[k] -= tau * t;
            }
            __syncwarp();
            if (PIVOT) {
                int recompute = 0;
                if (lane == 0 && nu[j] != 0.0) {
                    double temp = fabs(cj[k]) / nu[j];
                    temp = (1.0 + temp) * (1.0 - temp);
                    temp = temp < 0.0 ? 0.0 : temp;
                    const double ratio = nu[j] / nd[j];
                    const double temp2 = temp * ratio * ratio;
                    if (temp2 <= downdate_thr)
                        recompute = 1;
                    else
                        nu[j] *= sqrt(temp);
                }
                recompute = __shfl_sync(0xffffffffu, recompute, 0);
                if (recompute) {
                    double s = 0.0;
                    for (int i = k + 1 + lane; i < rows; i += 32) s += cj[i] * cj[i];
                    s = warp_sum(s);
                    if (lane == 0) nd[j] = nu[j] = sqrt(s);
                }
            }
        }
        __syncthreads();
    }
    if (d.R)
        for (int e = tid; e < w * w; e += blockDim.x) {
            const int i = e % w, j = e / w;
            d.R[i + j * d.ldr] = (i <= j && i < nsz) ? W[i + j * ldw] : 0.0;
        }
    if (PIVOT && tid == 0) {
        for (int j = 0; j < w; ++j) d.perm[j] = j;
        for (int k = 0; k < steps; ++k) {
            const int t = d.perm[k];
            d.perm[k] = d.perm[trans[k]];
            d.perm[trans[k]] = t;
        }
    }
    if (use_smem) {
        __syncthreads();
        for (i64 e = tid; e < i64(rows) * w; e += blockDim.x) {
            const int i = int(e % rows), j = int(e / rows);
            d.A[i + j * d.lda] = W[i + j * ldw];
        }
    }
}

__global__ void __launch_bounds__(FQNT) k_form_q(const QfDesc* descs, int w, int qcols, int smem_elems) {
    extern __shared__ double sm[];
    const QfDesc d = descs[blockIdx.x];
    const int rows = d.rows;
    // identity Tin: H_i (i >= c) leaves e_c unchanged (only the first qcols reflectors act)
    const int nref = d.Tin ? min(w, rows) : min(min(w, rows), qcols);
    const bool use_smem = i64(rows) * qcols <= smem_elems;
    double* Q = use_smem ? sm : d.Q;
    const i64 ldq = use_smem ? rows : d.ldq;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    for (i64 e = tid; e < i64(rows) * qcols; e += blockDim.x) {
        const int i = int(e % rows), c = int(e / rows);
        double v = 0.0;
        if (i < nref) v = d.Tin ? d.Tin[i + i64(c) * d.ldt] : (i == c ? 1.0 : 0.0);
        Q[i + c * ldq] = v;
    }
    __syncthreads();
    double* Es = sm + smem_elems;  // the current Householder vector, staged (rows doubles)
    for (int k = nref - 1; k >= 0; --k) {
        const double tau = d.tau[k];
        if (rows - k == 1) {
            for (int c = tid; c < qcols; c += blockDim.x) Q[k + c * ldq] *= (1.0 - tau);
        } else if (tau != 0.0) {
            for (int i = k + 1 + tid; i < rows; i += blockDim.x) Es[i] = d.A[i + k * d.lda];
            __syncthreads();
            const double* ess = Es;
            for (int c = warp; c < qcols; c += nwarps) {
                double* qc = Q + c * ldq;
                double t = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) t += ess[i] * qc[i];
                t = warp_sum(t) + qc[k];
                for (int i = k + 1 + lane; i < rows; i += 32) qc[i] -= tau * ess[i] * t;
                __syncwarp();
                if (lane == 0) qc[k] -= tau * t;
            }
        }
        __syncthreads();
    }
    if (use_smem)
        for (i64 e = tid; e < i64(rows) * qcols; e += blockDim.x) {
            const int i = int(e % rows), c = int(e / rows);
            d.Q[i + c * d.ldq] = Q[i + c * ldq];
        }
}

#include "qr_blocked.cuh"
#include "qr_cluster.cuh"

/// Cluster path (qr_cluster.cuh): few blocks (the clusters fit the chip at
/// once), wide enough to be worth two cluster barriers per column, and a
/// CTA's share of the columns fits shared memory. HG_QR_CLUSTER=0 disables.
bool cluster_qr_fits(int nblocks, int max_rows, int w, int num_sms) {
    static const bool on = [] {
        const char* e = std::getenv("HG_QR_CLUSTER");
        return !(e && e[0] == '0');
    }();
    return on && w >= 64 && w <= MAXW && nblocks * QC_CS <= num_sms && qc_smem(max_rows, w) <= QR_SMEM;
}

/// INPLACE instantiation only when some block does not fit shared memory
/// (its register-held columns would cost the resident path occupancy).
template <bool PIVOT>
void launch_qr(const QrDesc* dd, int nblocks, int qnt, size_t smem, int w, int smem_elems, bool inplace) {
    auto& c = current();
    if (inplace) {
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_qr<PIVOT, true>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_qr<PIVOT, true><<<unsigned(nblocks), qnt, smem, c.stream>>>(dd, w, smem_elems);
    } else {
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_qr<PIVOT, false>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_qr<PIVOT, false><<<unsigned(nblocks), qnt, smem, c.stream>>>(dd, w, smem_elems);
    }
}

}  // namespace

void batched_qr(const std::vector<QrDesc>& blocks, int w, bool pivot) {
    if (blocks.empty() || w <= 0) return;
    if (w > MAXW) throw std::length_error("batched_qr: width above 512");
    int max_rows = 0;
    for (const auto& b : blocks) max_rows = std::max(max_rows, b.rows);
    size_t smem = static_cast<size_t>(max_rows) * w * sizeof(double);
    if (smem > QR_SMEM) smem = QR_SMEM;  // larger blocks run in place in global memory
    const int smem_elems = int(smem / sizeof(double));
    DBuf<QrDesc> dd;
    dd.upload(blocks);
    auto& c = current();
    double rows = 0;
    for (const auto& b : blocks) rows += b.rows;
    ProfScope prof(PROF_QR, 2.0 * rows * w * w, 16.0 * rows * w);
    if (prof_enabled()) prof.key(prof_tag("qr%d w=%d blocks=%d rows=%d", int(pivot), w, int(blocks.size()), max_rows));
    // short blocks: fewer threads per CTA (more CTAs per SM, cheaper barriers)
    // (the trailing update runs a warp per column: wide blocks keep 16 warps)
    const int qnt = max_rows <= 64 ? 128 : (max_rows <= 256 && w <= 48) ? 256 : QNT;
    if (!pivot && w >= 128 && cluster_qr_fits(int(blocks.size()), max_rows, w, c.num_sms)) {
        // a few wide blocks, unpivoted: the cluster kernel, one cluster barrier per column
        const size_t sb = qc_smem(max_rows, w);
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_qr_cluster<false>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));
        k_qr_cluster<false><<<unsigned(blocks.size()) * QC_CS, QC_THREADS, sb, c.stream>>>(dd.get(), w);
    } else if (!pivot && (smem_elems < max_rows * w || w >= 32) && max_rows <= QB_MAXROWS &&
               qb_smem(max_rows, w) <= QB_SMEM_MAX) {
        // wide blocks that do not fit shared memory: blocked compact-WY QR
        const size_t sb = qb_smem(max_rows, w);
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_qr_blocked),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));
        k_qr_blocked<<<unsigned(blocks.size()), QB_THREADS, sb, c.stream>>>(dd.get(), w);
    } else if (pivot && cluster_qr_fits(int(blocks.size()), max_rows, w, c.num_sms)) {
        // a few wide blocks: one thread-block cluster per block, columns resident in DSMEM
        const size_t sb = qc_smem(max_rows, w);
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_qr_cluster<true>),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));
        k_qr_cluster<true><<<unsigned(blocks.size()) * QC_CS, QC_THREADS, sb, c.stream>>>(dd.get(), w);
    } else if (pivot) {
        launch_qr<true>(dd.get(), int(blocks.size()), qnt, smem, w, smem_elems, smem_elems < max_rows * w);
    } else {
        launch_qr<false>(dd.get(), int(blocks.size()), qnt, smem, w, smem_elems, smem_elems < max_rows * w);
    }
    HG_LAUNCH();
    ++c.launches;
}

void batched_form_q(const std::vector<QfDesc>& blocks, int w, int qcols) {
    if (blocks.empty() || qcols <= 0) return;
    int max_rows = 0;
    for (const auto& b : blocks) max_rows = std::max(max_rows, b.rows);
    size_t smem = static_cast<size_t>(max_rows) * qcols * sizeof(double);
    if (smem > QR_SMEM) smem = QR_SMEM;
    const int smem_elems = int(smem / sizeof(double));
    smem += static_cast<size_t>(max_rows) * sizeof(double);  // staged Householder vector
    DBuf<QfDesc> dd;
    dd.upload(blocks);
    auto& c = current();
    double rows = 0;
    for (const auto& b : blocks) rows += b.rows;
    ProfScope prof(PROF_FORM_Q, 4.0 * rows * w * qcols, 8.0 * rows * (w + 2.0 * qcols));
    if (prof_enabled()) prof.key(prof_tag("formq w=%d q=%d blocks=%d rows=%d", w, qcols, int(blocks.size()), max_rows));
    if ((smem_elems < max_rows * qcols || qcols >= 16) && max_rows <= QB_MAXROWS &&
        qb_smem(max_rows, qcols) <= QB_SMEM_MAX) {
        const size_t sb = qb_smem(max_rows, qcols);
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_form_q_blocked),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(sb)));
        // split the columns when the blocks alone leave SMs idle
        int chunk = qcols;
        while (chunk > 32 && int(blocks.size()) * cdiv(qcols, chunk) < 2 * c.num_sms) chunk = (chunk + 1) / 2;
        k_form_q_blocked<<<dim3(unsigned(blocks.size()), unsigned(cdiv(qcols, chunk))), QB_THREADS, sb, c.stream>>>(
            dd.get(), w, qcols, chunk);
    } else {
        HG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(k_form_q),
                                     cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
        k_form_q<<<unsigned(blocks.size()), FQNT, smem, c.stream>>>(dd.get(), w, qcols, smem_elems);
    }
    HG_LAUNCH();
    ++c.launches;
}

}  // namespace hg

namespace hg {

namespace {
int chunk_rows(int w) {
    static const size_t budget = [] {  // HG_QR_CHUNK_KB: TSQR chunk budget (tuning knob)
        const char* e = std::getenv("HG_QR_CHUNK_KB");
        const long v = e ? std::atol(e) : 0;
        return v > 0 ? static_cast<size_t>(v) * 1024 : QR_SMEM;
    }();
    int fit = int(std::min(budget, QR_SMEM) / (sizeof(double) * static_cast<size_t>(std::max(w, 1))));
    fit = (fit / 32) * 32;
    int rows = std::max(fit, 4 * w);
    // very wide panels (w > ~250: derivative blocks at k > 80): shorter chunks, down to 2w rows,
    // keep the blocked kernels' shared-memory budget (a taller TSQR tree instead of the in-place path)
    while (rows - 32 >= 2 * w && (rows > QB_MAXROWS || qb_smem(rows, w) > QB_SMEM_MAX)) rows -= 32;
    return rows;
}
}  // namespace

int qr_chunk_rows(int w) { return chunk_rows(w); }

BatchedQR::BatchedQR(const std::vector<Block>& blocks, int w, bool pivot) : w_(w), pivot_(pivot), blocks_(blocks) {
    const int CH = chunk_rows(w);
    std::vector<Node> cur;
    for (size_t b = 0; b < blocks.size(); ++b)
        cur.push_back(Node{blocks[b].A, blocks[b].lda, blocks[b].rows, int(b)});
    top_node_.assign(blocks.size(), -1);
    top_level_.assign(blocks.size(), 0);
    int L = 0;
    for (;;) {
        nodes_.push_back(cur);
        bool any = false;
        for (const auto& nd : cur) any |= nd.rows > CH;
        if (!any) break;
        // Split every long node into balanced chunks; stack their R factors.
        std::vector<Chunk> ch;
        std::vector<Node> next;
        size_t stack_elems = 0, tau_elems = 0;
        struct Plan {
            int node, nch;
        };
        std::vector<Plan> plans;
        for (size_t i = 0; i < cur.size(); ++i) {
            if (cur[i].rows > CH) {
                const int nch = cdiv(cur[i].rows, CH);
                plans.push_back(Plan{int(i), nch});
                stack_elems += static_cast<size_t>(nch) * w * w;
                tau_elems += static_cast<size_t>(nch) * w;
            }
        }
        auto stack = make_dvec(stack_elems, true);
        auto tau = make_dvec(std::max<size_t>(tau_elems, 1), false);
        size_t so = 0, to = 0;
        size_t pi = 0;
        for (size_t i = 0; i < cur.size(); ++i) {
            if (pi < plans.size() && plans[pi].node == int(i)) {
                const int nch = plans[pi].nch;
                double* S = stack->get() + so;
                const int srows = nch * w;
                const int base = cur[i].rows / nch, rem = cur[i].rows % nch;
                int r0 = 0;
                for (int c = 0; c < nch; ++c) {
                    const int rr = base + (c < rem ? 1 : 0);
                    QrDesc d{cur[i].A + r0, cur[i].lda, rr, tau->get() + to, S + i64(c) * w, srows, nullptr};
                    ch.push_back(Chunk{L + 1, int(next.size()), c, d});
                    to += static_cast<size_t>(w);
                    r0 += rr;
                }
                next.push_back(Node{S, srows, srows, cur[i].block});
                so += static_cast<size_t>(nch) * w * w;
                ++pi;
            } else {
                next.push_back(cur[i]);  // passes through unchanged
                ch.push_back(Chunk{L + 1, int(next.size()) - 1, -1, QrDesc{}});
            }
        }
        std::vector<QrDesc> descs;
        for (const auto& c : ch)
            if (c.index >= 0) descs.push_back(c.desc);
        batched_qr(descs, w, false);
        chunks_.push_back(ch);
        stacks_.push_back(stack);
        taus_.push_back(tau);
        cur = next;
        ++L;
    }
    // Top level: the (pivoted) QR of every remaining node.
    const size_t nb = blocks.size();
    R_.alloc(nb * static_cast<size_t>(w) * w);
    top_tau_.alloc(nb * static_cast<size_t>(w));
    perm_.alloc(nb * static_cast<size_t>(w));
    std::vector<QrDesc> descs;
    for (size_t i = 0; i < cur.size(); ++i) {
        const int b = cur[i].block;
        top_node_[static_cast<size_t>(b)] = int(i);
        top_level_[static_cast<size_t>(b)] = L;
        descs.push_back(QrDesc{cur[i].A, cur[i].lda, cur[i].rows, top_tau_.get() + static_cast<size_t>(b) * w,
                               R_.get() + static_cast<size_t>(b) * w * w, w, perm_.get() + static_cast<size_t>(b) * w,
                               pivot ? blocks[static_cast<size_t>(b)].stop : QrStop{}});
    }
    batched_qr(descs, w, pivot);
}

void BatchedQR::form_q(int qcols, const double* Tin, i64 tstride, int ldt, const std::vector<double*>& Q,
                       const std::vector<i64>& ldq) const {
    const int w = w_;
    const int Ltop = int(nodes_.size()) - 1;
    // Q buffers for every level's nodes above level 0 (their rows feed chunk Tin).
    std::vector<std::vector<std::pair<double*, i64>>> qbuf(static_cast<size_t>(Ltop + 1));
    std::vector<DVecP> keep;
    for (int L = Ltop; L >= 0; --L) {
        const auto& nodes = nodes_[static_cast<size_t>(L)];
        qbuf[static_cast<size_t>(L)].resize(nodes.size());
        if (L == 0) {
            for (size_t i = 0; i < nodes.size(); ++i)
                qbuf[0][i] = {Q[static_cast<size_t>(nodes[i].block)], ldq[static_cast<size_t>(nodes[i].block)]};
        } else {
            size_t tot = 0;
            for (const auto& nd : nodes) tot += static_cast<size_t>(nd.rows) * qcols;
            auto buf = make_dvec(std::max<size_t>(tot, 1), false);
            keep.push_back(buf);
            size_t o = 0;
            for (size_t i = 0; i < nodes.size(); ++i) {
                qbuf[static_cast<size_t>(L)][i] = {buf->get() + o, nodes[i].rows};
                o += static_cast<size_t>(nodes[i].rows) * qcols;
            }
        }
    }
    // Top: H_top [Tin; 0].
    {
        std::vector<QfDesc> d;
        const auto& nodes = nodes_[static_cast<size_t>(Ltop)];
        for (size_t i = 0; i < nodes.size(); ++i) {
            const int b = nodes[i].block;
            d.push_back(QfDesc{nodes[i].A, nodes[i].lda, nodes[i].rows, top_tau_.get() + static_cast<size_t>(b) * w,
                               Tin ? Tin + i64(b) * tstride : nullptr, ldt, qbuf[static_cast<size_t>(Ltop)][i].first,
                               qbuf[static_cast<size_t>(Ltop)][i].second});
        }
        batched_form_q(d, w, qcols);
    }
    // Down the tree: chunk c of a stack gets rows [c w, (c+1) w) of the stack's Q.
    for (int L = Ltop - 1; L >= 0; --L) {
        std::vector<QfDesc> d;
        std::vector<std::pair<int, int>> copies;  // pass-through nodes: (child idx, parent idx)
        const auto& ch = chunks_[static_cast<size_t>(L)];
        const auto& nodes = nodes_[static_cast<size_t>(L)];
        size_t ci = 0;
        for (size_t i = 0; i < nodes.size(); ++i) {
            // chunks of node i are consecutive in ch
            if (ch[ci].index < 0) {
                copies.push_back({int(i), ch[ci].parent});
                ++ci;
                continue;
            }
            const int parent = ch[ci].parent;
            const auto pq = qbuf[static_cast<size_t>(L + 1)][static_cast<size_t>(parent)];
            const auto child = qbuf[static_cast<size_t>(L)][i];
            int r0 = 0;
            while (ci < ch.size() && ch[ci].index >= 0 && ch[ci].parent == parent) {
                const QrDesc& qd = ch[ci].desc;
                d.push_back(QfDesc{qd.A, qd.lda, qd.rows, qd.tau, pq.first + i64(ch[ci].index) * w, int(pq.second),
                                   child.first + r0, child.second});
                r0 += qd.rows;
                ++ci;
            }
        }
        batched_form_q(d, w, qcols);
        for (auto [c, p] : copies) {
            const auto src = qbuf[static_cast<size_t>(L + 1)][static_cast<size_t>(p)];
            const auto dst = qbuf[static_cast<size_t>(L)][static_cast<size_t>(c)];
            HG_CUDA(cudaMemcpy2DAsync(dst.first, static_cast<size_t>(dst.second) * sizeof(double), src.first,
                                      static_cast<size_t>(src.second) * sizeof(double), static_cast<size_t>(nodes[static_cast<size_t>(c)].rows) * sizeof(double),
                                      static_cast<size_t>(qcols), cudaMemcpyDeviceToDevice, current().stream));
        }
    }
}

}  // namespace hg
