// Column-pivoted Householder QR of a few wide blocks by thread-block clusters
// (included by qr.cu inside its anonymous namespace).
//
// The roots of the TSQR trees and the single-CTA levels of the derivative
// recompression are a handful of w x w .. 4w x w blocks (w up to 239 at C5):
// one CTA per block leaves 140+ SMs idle and, above the 200 KB shared-memory
// budget, runs every column update out of L2 (~23 us per column step). Here a
// cluster of QC_CS CTAs owns one block: the columns are dealt cyclically to
// the CTAs and stay resident in their shared memory for the whole
// factorization; columns never move (a position <-> column map replaces the
// swaps). Per step: every CTA posts its best remaining column norm into all
// peers' shared memory (DSMEM), barrier, the owner of the pivot column forms
// the reflector and broadcasts it through DSMEM, barrier, every CTA updates
// its own columns. Two cluster barriers per step (one when unpivoted: the
// reflector buffers alternate) instead of ~5 CTA barriers over an L2-resident
// matrix.
//
// Same arithmetic as k_qr<true>: per column the same lane-strided dot product
// and update, the same 512-thread tail norm, Eigen's pivot rule (largest
// updated norm, first position on ties) and xGEQPF downdating.
#pragma once
// (qr.cu includes <cooperative_groups.h> at global scope)

constexpr int QC_CS = 8;         // portable cluster size
constexpr int QC_THREADS = QNT;  // 512: the tail-norm reduction order of k_qr

struct QcShared {
    double cand_v[QC_CS];
    int cand_p[QC_CS];
    double bc[2][4];  // per step parity: beta, tau, zero flag (broadcast by the pivot column's owner)
    int pos_of[MAXW], at_pos[MAXW];
};

__host__ __device__ inline size_t qc_smem(int rows, int w) {
    const int cpc = (w + QC_CS - 1) / QC_CS;
    return sizeof(double) * (size_t(rows) * cpc + 2 * size_t(rows) + 2 * size_t(cpc));
}

template <bool PIVOT>
__global__ void __cluster_dims__(QC_CS, 1, 1) __launch_bounds__(QC_THREADS)
    k_qr_cluster(const QrDesc* descs, int w) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = int(cluster.block_rank());
    extern __shared__ double sm[];
    __shared__ QcShared sh;
    const QrDesc d = descs[blockIdx.x / QC_CS];
    const int rows = d.rows, cpc = (w + QC_CS - 1) / QC_CS;
    double* W = sm;                     // owned columns: local c <-> column c * QC_CS + rank
    double* vb2 = W + size_t(rows) * cpc;  // Householder vectors of even / odd steps (2 x rows)
    double* nu = vb2 + 2 * size_t(rows);   // updated / direct norms of the owned columns
    double* nd = nu + cpc;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    const int nown = rank < w ? (w - rank + QC_CS - 1) / QC_CS : 0;
    for (int c = 0; c < nown; ++c)
        for (int i = tid; i < rows; i += blockDim.x) W[i + size_t(c) * rows] = d.A[i + i64(c * QC_CS + rank) * d.lda];
    for (int j = tid; j < w; j += blockDim.x) sh.pos_of[j] = sh.at_pos[j] = j;
    __syncthreads();
    if (PIVOT)
        for (int c = warp; c < nown; c += nwarps) {
            double s = 0.0;
            for (int i = lane; i < rows; i += 32) s += W[i + size_t(c) * rows] * W[i + size_t(c) * rows];
            s = warp_sum(s);
            if (lane == 0) nd[c] = nu[c] = sqrt(s);
        }
    cluster.sync();  // every CTA has read its columns of A (they are rewritten at the end) and is running
    const int nsz = min(rows, w);
    const double downdate_thr = sqrt(DBL_EPSILON);
    int steps = nsz;
    double beta0 = 0.0, stop_abs = -1.0;
    if (PIVOT && d.stop.active && d.stop.abs_ptr) stop_abs = d.stop.abs_scale * *d.stop.abs_ptr;
    for (int k = 0; k < nsz; ++k) {
        // ---- pivot: best owned column among positions >= k, posted to every CTA
        if (PIVOT && warp == 0) {
            double bv = -1.0;
            int bp = 1 << 30;
            for (int c = lane; c < nown; c += 32) {
                const int p = sh.pos_of[c * QC_CS + rank];
                if (p >= k && (nu[c] > bv || (nu[c] == bv && p < bp))) {
                    bv = nu[c];
                    bp = p;
                }
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
                const int op = __shfl_xor_sync(0xffffffffu, bp, o);
                if (ov > bv || (ov == bv && op < bp)) {
                    bv = ov;
                    bp = op;
                }
            }
            if (lane < QC_CS) {
                QcShared* peer = cluster.map_shared_rank(&sh, lane);
                peer->cand_v[rank] = bv;
                peer->cand_p[rank] = bp;
            }
        }
        int best = k;
        if (PIVOT) {
            cluster.sync();
            double bv = -1.0;
#pragma unroll
            for (int r = 0; r < QC_CS; ++r)
                if (sh.cand_v[r] > bv || (sh.cand_v[r] == bv && sh.cand_p[r] < best)) {
                    bv = sh.cand_v[r];
                    best = sh.cand_p[r];
                }
            __syncthreads();  // everyone has read the map before it changes
        }
        // (vb and bc alternate between two buffers: step k's owner may write while peers
        // still read step k-1's; everyone passed step k-1's barrier after finishing step k-2)
        double* vb = vb2 + size_t(k & 1) * rows;
        if (tid == 0 && best != k) {  // positions k and best trade columns (identically in every CTA)
            const int ck = sh.at_pos[k], cb = sh.at_pos[best];
            sh.at_pos[k] = cb;
            sh.at_pos[best] = ck;
            sh.pos_of[cb] = k;
            sh.pos_of[ck] = best;
        }
        __syncthreads();
        const int pc = sh.at_pos[k];  // the pivot column
        // ---- reflector by the pivot column's owner, broadcast through DSMEM
        if (pc % QC_CS == rank) {
            double* col = W + size_t(pc / QC_CS) * rows;
            double part = 0.0;
            for (int i = k + 1 + tid; i < rows; i += blockDim.x) part += col[i] * col[i];
            const double c0 = col[k];
            const double tail = qr_block_sum(part);
            const bool zero = tail <= DBL_MIN;
            double tau = 0.0, div = 1.0, beta = c0;
            if (!zero) {
                beta = sqrt(c0 * c0 + tail);
                if (c0 >= 0.0) beta = -beta;
                div = c0 - beta;
                tau = (beta - c0) / beta;
            }
            if (tid == 0) {
                if (!zero) col[k] = beta;
                d.tau[k] = tau;
            }
            for (int i = k + 1 + tid; i < rows; i += blockDim.x) {
                const double vi = zero ? 0.0 : col[i] / div;
                col[i] = vi;
#pragma unroll
                for (int r = 0; r < QC_CS; ++r) cluster.map_shared_rank(vb, r)[i] = vi;
            }
            if (tid < QC_CS) {
                QcShared* peer = cluster.map_shared_rank(&sh, tid);
                peer->bc[k & 1][0] = beta;
                peer->bc[k & 1][1] = tau;
                peer->bc[k & 1][2] = zero ? 1.0 : 0.0;
            }
        }
        cluster.sync();
        const double beta = sh.bc[k & 1][0], tau = sh.bc[k & 1][1];
        if (PIVOT && d.stop.active) {  // uniform over the cluster: every CTA holds the same beta
            if (k == 0) beta0 = fabs(beta);
            if (fabs(beta) <= fmax(d.stop.rel * beta0, stop_abs) || k + 1 >= d.stop.max_steps) {
                if (rank == 0)
                    for (int t = k + 1 + tid; t < nsz; t += blockDim.x) d.tau[t] = 0.0;
                steps = k + 1;
                break;
            }
        }
        // ---- trailing update of the owned columns at positions > k
        for (int c = warp; c < nown; c += nwarps) {
            if (sh.pos_of[c * QC_CS + rank] <= k) continue;
            double* cj = W + size_t(c) * rows;
            if (rows - k == 1) {
                if (lane == 0) cj[k] *= (1.0 - tau);
            } else if (tau != 0.0) {
                double t = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) t += vb[i] * cj[i];
                t = warp_sum(t) + cj[k];
                for (int i = k + 1 + lane; i < rows; i += 32) cj[i] -= tau * vb[i] * t;
                __syncwarp();
                if (lane == 0) cj[k] -= tau * t;
            }
            __syncwarp();
            if (!PIVOT) continue;
            int recompute = 0;
            if (lane == 0 && nu[c] != 0.0) {
                double temp = fabs(cj[k]) / nu[c];
                temp = (1.0 + temp) * (1.0 - temp);
                temp = temp < 0.0 ? 0.0 : temp;
                const double ratio = nu[c] / nd[c];
                const double temp2 = temp * ratio * ratio;
                if (temp2 <= downdate_thr)
                    recompute = 1;
                else
                    nu[c] *= sqrt(temp);
            }
            recompute = __shfl_sync(0xffffffffu, recompute, 0);
            if (recompute) {
                double s = 0.0;
                for (int i = k + 1 + lane; i < rows; i += 32) s += cj[i] * cj[i];
                s = warp_sum(s);
                if (lane == 0) nd[c] = nu[c] = sqrt(s);
            }
        }
        __syncthreads();  // nu and the columns are final before the next pivot search
    }
    __syncthreads();
    // ---- results in pivoted order: column at position p = at_pos[p]
    for (int c = 0; c < nown; ++c) {
        const int p = sh.pos_of[c * QC_CS + rank];
        const double* col = W + size_t(c) * rows;
        for (int i = tid; i < rows; i += blockDim.x) d.A[i + i64(p) * d.lda] = col[i];
        if (d.R)
            for (int i = tid; i < w; i += blockDim.x) d.R[i + i64(p) * d.ldr] = (i <= p && i < nsz) ? col[i] : 0.0;
    }
    if (PIVOT && rank == 0)
        for (int p = tid; p < w; p += blockDim.x) d.perm[p] = sh.at_pos[p];
    (void)steps;
    cluster.sync();  // no CTA leaves while a peer may still write into its shared memory
}
