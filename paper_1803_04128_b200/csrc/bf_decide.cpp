// bf_decide.cpp -- Algorithm 6 on the host: does the NUFFT apply to
// K = (U2 V2^T) o e^{2 pi i U1 V1^T}?  (include/bf_nufft.h, bf_nufft_decide.)  Plan-construction work, untimed, FP64,
// with r = 1 (the one-dimensional NUFFT of the device path):
//   1. the r-leading SVD of the rank-r1 phase U1 V1^T by a randomized range finder with r1 + 4 test vectors
//      ([Gu, randomSVD]): Y = U1 (V1^T Omega), Q = orth(Y), B = Q^T U1 V1^T, B = Ub S W^T; P = Q Ub_1 S_1, q = W_1;
//   2. rq sampled columns of (U2 V2^T) o e^{2 pi i (U1 V1^T - P q^T)}, Householder QR with column pivoting, n = the
//      number of |R_kk| > |R_11| eps;
//   3. y = (n <= r_eps) (reading R24).
// When y = 1 and the column factor is a multiple of the column frequencies (q_j = alpha xi_j: uniform integer
// frequencies, the type-2 NUFFT of bf_nufft_create), the targets t(x_i) = alpha P_i are returned.
// Independent of the oracle (oracle/nufft.py does the same steps with numpy / scipy).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <numeric>
#include <vector>

#include "../../include/bf.h"
#include "../../include/bf_nufft.h"
#include "bf_plan_internal.h"

namespace {

using cd = std::complex<double>;

struct Rng {   // splitmix64 + Box-Muller: deterministic, seeded
    uint64_t s;
    uint64_t next()
    {
        uint64_t z = (s += 0x9e3779b97f4a7c15ull);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
        return z ^ (z >> 31);
    }
    double uni() { return (double(next() >> 11) + 0.5) * 0x1.0p-53; }
    double gauss() { return std::sqrt(-2.0 * std::log(uni())) * std::cos(2.0 * M_PI * uni()); }
};

// symmetric eigen-decomposition of a small k x k matrix (cyclic Jacobi); A overwritten, V = eigenvectors (columns)
void jacobi_eig(std::vector<double>& A, int k, std::vector<double>& V)
{
    V.assign(size_t(k) * k, 0.0);
    for (int i = 0; i < k; i++) V[size_t(i) * k + i] = 1.0;
    for (int sweep = 0; sweep < 60; sweep++) {
        double off = 0;
        for (int i = 0; i < k; i++)
            for (int j = i + 1; j < k; j++) off += A[size_t(i) * k + j] * A[size_t(i) * k + j];
        if (off < 1e-300) break;
        for (int p = 0; p < k; p++)
            for (int q = p + 1; q < k; q++) {
                const double apq = A[size_t(p) * k + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double th = 0.5 * (A[size_t(q) * k + q] - A[size_t(p) * k + p]) / apq;
                const double t = (th >= 0 ? 1.0 : -1.0) / (std::fabs(th) + std::sqrt(th * th + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int r = 0; r < k; r++) {   // A <- J^T A J
                    const double arp = A[size_t(r) * k + p], arq = A[size_t(r) * k + q];
                    A[size_t(r) * k + p] = c * arp - s * arq;
                    A[size_t(r) * k + q] = s * arp + c * arq;
                }
                for (int r = 0; r < k; r++) {
                    const double apr = A[size_t(p) * k + r], aqr = A[size_t(q) * k + r];
                    A[size_t(p) * k + r] = c * apr - s * aqr;
                    A[size_t(q) * k + r] = s * apr + c * aqr;
                }
                for (int r = 0; r < k; r++) {
                    const double vrp = V[size_t(r) * k + p], vrq = V[size_t(r) * k + q];
                    V[size_t(r) * k + p] = c * vrp - s * vrq;
                    V[size_t(r) * k + q] = s * vrp + c * vrq;
                }
            }
    }
}

// |R_kk| of the Householder QR with column pivoting of the column-major m x n complex matrix A (overwritten)
std::vector<double> qrcp_diag(std::vector<cd>& A, int64_t m, int n)
{
    std::vector<double> d;
    std::vector<int> perm(n);
    std::iota(perm.begin(), perm.end(), 0);
    auto col = [&](int j) { return A.data() + size_t(j) * m; };
    for (int k = 0; k < std::min<int64_t>(m, n); k++) {
        int best = k;
        double bn = -1;
        for (int j = k; j < n; j++) {   // column norms of the trailing block, recomputed (robust, n small)
            double s = 0;
            const cd* a = col(j);
            for (int64_t i = k; i < m; i++) s += std::norm(a[i]);
            if (s > bn) {
                bn = s;
                best = j;
            }
        }
        if (best != k)
            for (int64_t i = 0; i < m; i++) std::swap(col(k)[i], col(best)[i]);
        cd* a = col(k);
        const double nrm = std::sqrt(bn);
        d.push_back(nrm);
        if (nrm == 0) break;
        // Householder v = a_k + e^{i arg a_kk} ||a_k|| e_k, applied to the trailing columns
        const cd ph = std::abs(a[k]) > 0 ? a[k] / std::abs(a[k]) : cd(1, 0);
        std::vector<cd> v(a + k, a + m);
        v[0] += ph * nrm;
        double vn = 0;
        for (const cd& x : v) vn += std::norm(x);
        if (vn == 0) continue;
        for (int j = k + 1; j < n; j++) {
            cd* b = col(j);
            cd dot = 0;
            for (int64_t i = k; i < m; i++) dot += std::conj(v[size_t(i - k)]) * b[i];
            const cd f = 2.0 * dot / vn;
            for (int64_t i = k; i < m; i++) b[i] -= f * v[size_t(i - k)];
        }
    }
    return d;
}

}  // namespace

extern "C" bf_status_t bf_nufft_decide(const bf_nufft_decide_t* d, int32_t* y, int32_t* n_rank, double* targets)
{
    if (!d || !y || !n_rank || !d->u1 || !d->v1 || !d->u2 || !d->v2)
        return bfp_fail(BF_ERR_INVALID_ARG, "bf_nufft_decide: null argument");
    const int64_t m = d->m, n = d->n;
    const int r1 = d->r1, r2 = d->r2;
    if (m < 2 || n < 2 || r1 < 1 || r1 > 16 || r2 < 1 || r2 > 16 || d->rank_budget < 1 || d->q < 1 ||
        !(d->eps > 0 && d->eps < 1))
        return bfp_fail(BF_ERR_SHAPE, "bf_nufft_decide: m, n >= 2; r1, r2 in 1..16; rank_budget, q >= 1; 0 < eps < 1");
    Rng rng{uint64_t(d->seed) * 0x2545f4914f6cdd1dull + 1};
    // ---- step 1: randomized r-leading SVD of U1 V1^T (r = 1) ----
    const int k = r1 + 4;
    std::vector<double> T(size_t(r1) * k, 0.0);   // V1^T Omega, r1 x k
    for (int64_t j = 0; j < n; j++)
        for (int c = 0; c < k; c++) {
            const double om = rng.gauss();
            for (int a = 0; a < r1; a++) T[size_t(a) * k + c] += d->v1[size_t(a) * n + j] * om;
        }
    std::vector<double> Y(size_t(k) * m, 0.0);    // columns of U1 T, then orthonormalized (modified Gram-Schmidt)
    for (int c = 0; c < k; c++)
        for (int a = 0; a < r1; a++)
            for (int64_t i = 0; i < m; i++) Y[size_t(c) * m + i] += d->u1[size_t(a) * m + i] * T[size_t(a) * k + c];
    int kq = 0;
    double ref = 0;
    for (int c = 0; c < k; c++) {
        double* yc = Y.data() + size_t(c) * m;
        for (int b = 0; b < kq; b++) {
            const double* qb = Y.data() + size_t(b) * m;
            double dot = 0;
            for (int64_t i = 0; i < m; i++) dot += qb[i] * yc[i];
            for (int64_t i = 0; i < m; i++) yc[i] -= dot * qb[i];
        }
        double nr = 0;
        for (int64_t i = 0; i < m; i++) nr += yc[i] * yc[i];
        nr = std::sqrt(nr);
        ref = std::max(ref, nr);
        if (nr <= 1e-12 * ref) continue;   // dependent direction (the range has rank r1 < k)
        double* dst = Y.data() + size_t(kq) * m;
        for (int64_t i = 0; i < m; i++) dst[i] = yc[i] / nr;
        kq++;
    }
    // C = Q^T U1 (kq x r1); B = C V1^T (kq x n); B B^T = C (V1^T V1) C^T
    std::vector<double> C(size_t(kq) * r1, 0.0), G1(size_t(r1) * r1, 0.0);
    for (int b = 0; b < kq; b++)
        for (int a = 0; a < r1; a++) {
            double s = 0;
            for (int64_t i = 0; i < m; i++) s += Y[size_t(b) * m + i] * d->u1[size_t(a) * m + i];
            C[size_t(b) * r1 + a] = s;
        }
    for (int a = 0; a < r1; a++)
        for (int b = 0; b < r1; b++) {
            double s = 0;
            for (int64_t j = 0; j < n; j++) s += d->v1[size_t(a) * n + j] * d->v1[size_t(b) * n + j];
            G1[size_t(a) * r1 + b] = s;
        }
    std::vector<double> BBt(size_t(kq) * kq, 0.0), V;
    for (int p = 0; p < kq; p++)
        for (int q = 0; q < kq; q++) {
            double s = 0;
            for (int a = 0; a < r1; a++)
                for (int b = 0; b < r1; b++) s += C[size_t(p) * r1 + a] * G1[size_t(a) * r1 + b] * C[size_t(q) * r1 + b];
            BBt[size_t(p) * kq + q] = s;
        }
    jacobi_eig(BBt, kq, V);
    int top = 0;
    for (int p = 1; p < kq; p++)
        if (BBt[size_t(p) * kq + p] > BBt[size_t(top) * kq + top]) top = p;
    const double s1 = std::sqrt(std::max(BBt[size_t(top) * kq + top], 0.0));
    if (!(s1 > 0)) return bfp_fail(BF_ERR_INVALID_ARG, "bf_nufft_decide: the phase factorization is zero");
    std::vector<double> ub(kq), cu(r1, 0.0), P(static_cast<size_t>(m), 0.0), qv(static_cast<size_t>(n), 0.0);
    for (int p = 0; p < kq; p++) ub[p] = V[size_t(p) * kq + top];
    for (int a = 0; a < r1; a++)
        for (int p = 0; p < kq; p++) cu[a] += ub[p] * C[size_t(p) * r1 + a];   // ub^T C
    for (int p = 0; p < kq; p++)
        for (int64_t i = 0; i < m; i++) P[size_t(i)] += Y[size_t(p) * m + i] * ub[p] * s1;   // P = Q ub s1
    for (int64_t j = 0; j < n; j++)
        for (int a = 0; a < r1; a++) qv[size_t(j)] += cu[a] * d->v1[size_t(a) * n + j] / s1;   // q = B^T ub / s1
    // ---- step 2: rq sampled columns of the modulated amplitude, pivoted QR ----
    const int rq = int(std::min<int64_t>(n, int64_t(d->q)));   // r q with r = 1
    std::vector<int64_t> J(static_cast<size_t>(n));
    std::iota(J.begin(), J.end(), 0);
    for (int t = 0; t < rq; t++) std::swap(J[size_t(t)], J[size_t(t + int64_t(rng.next() % uint64_t(n - t)))]);
    J.resize(size_t(rq));
    std::sort(J.begin(), J.end());
    std::vector<cd> A(size_t(m) * rq);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < m; i++)
        for (int t = 0; t < rq; t++) {
            const int64_t j = J[size_t(t)];
            double ph = -P[size_t(i)] * qv[size_t(j)];
            for (int a = 0; a < r1; a++) ph += d->u1[size_t(a) * m + i] * d->v1[size_t(a) * n + j];
            cd amp = 0;
            for (int b = 0; b < r2; b++)
                amp += cd(d->u2[(size_t(b) * m + i) * 2], d->u2[(size_t(b) * m + i) * 2 + 1]) *
                       cd(d->v2[(size_t(b) * n + j) * 2], d->v2[(size_t(b) * n + j) * 2 + 1]);
            ph -= std::floor(ph);
            A[size_t(t) * m + i] = amp * std::polar(1.0, 2.0 * M_PI * ph);
        }
    const std::vector<double> dg = qrcp_diag(A, m, rq);
    int cnt = 0;
    for (double x : dg) cnt += (x > dg[0] * d->eps);
    *n_rank = cnt;
    // ---- step 3 (reading R24) ----
    *y = cnt <= d->rank_budget ? 1 : 0;
    if (*y && targets) {
        if (!d->xi) return bfp_fail(BF_ERR_INVALID_ARG, "bf_nufft_decide: targets requested without xi");
        double num = 0, den = 0, mq = 0;
        for (int64_t j = 0; j < n; j++) {
            num += qv[size_t(j)] * d->xi[j];
            den += d->xi[j] * d->xi[j];
            mq = std::max(mq, std::fabs(qv[size_t(j)]));
        }
        const double alpha = den > 0 ? num / den : 0;
        for (int64_t j = 0; j < n; j++)
            if (std::fabs(qv[size_t(j)] - alpha * d->xi[j]) > 1e-9 * mq)
                return bfp_fail(BF_ERR_NOT_SUPPORTED,
                                "bf_nufft_decide: the phase's column factor is not a multiple of xi (type-3 NUFFT)");
        for (int64_t i = 0; i < m; i++) targets[i] = alpha * P[size_t(i)];
    }
    return BF_OK;
}
