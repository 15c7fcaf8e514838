// BiCGStab(l) / CG on device vectors: a line-by-line restatement of the
// reference control flow (proj/include/sap/krylov.hpp:110-442) whose vector
// work runs in fused sm_100a kernels and whose reductions are deterministic
// (vec.cu). Scalars follow the reference's formulas on the host.
#include <cmath>
#include <cstring>
#include <random>

#include "kernels.h"
#include "krylov.h"

namespace sapgpu {

namespace {

constexpr int kMaxEll = 8;
// device scalar slots: [0, kMaxDots) batch outputs; [16, 16 + kMaxEll * kMaxEll) MGS dot numerators
// (tau_ij at 16 + i * kMaxEll + j, sigma_j at 16 + j * kMaxEll + j, gamma'_j at 16 + j)
constexpr int kScal = 16 + kMaxEll * kMaxEll + 16;

struct VecSet {
    double* p[2 * kMaxEll + 2];
    // k_final_update packs 3 coefficients per j = 1..ell-1 after c[0..2]: highest index 3 ell - 1
    double c[3 * kMaxEll];
};
static_assert(3 * (kMaxEll - 1) + 2 < 3 * kMaxEll, "VecSet::c holds every polynomial-update coefficient");

inline int vgrid(int n) { return std::max(1, std::min(ceil_div(n, 256), 148 * 8)); }

// u[i] = r[i] - beta * u[i], i = 0..j   (krylov.hpp:195-199)
__global__ void k_u_update(VecSet v, int j, double beta, int n) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        for (int i = 0; i <= j; ++i) v.p[kMaxEll + 1 + i][t] = fma(-beta, v.p[kMaxEll + 1 + i][t], v.p[i][t]);
}
// r[i] -= alpha * u[i+1], i = 0..j      (krylov.hpp:211-214)
__global__ void k_r_update(VecSet v, int j, double alpha, int n) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x)
        for (int i = 0; i <= j; ++i) v.p[i][t] = fma(-alpha, v.p[kMaxEll + 2 + i][t], v.p[i][t]);
}
// k_r_update and then x += alpha * u[0] (flag if x becomes non-finite) in one pass: the x update reads neither
// r[0..j] nor r[j+1], so BiCGStab's step runs both before A r_j (each element's operations unchanged)
__global__ void k_r_update_x(VecSet v, int j, double alpha, double* __restrict__ x, int n, int* flag) {
    int bad = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        for (int i = 0; i <= j; ++i) v.p[i][t] = fma(-alpha, v.p[kMaxEll + 2 + i][t], v.p[i][t]);
        const double xv = fma(alpha, v.p[kMaxEll + 1][t], x[t]);
        x[t] = xv;
        if (!isfinite(xv)) bad = 1;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}
// y += a * x, flag if y becomes non-finite
__global__ void k_axpy_check(double* __restrict__ y, double a, const double* __restrict__ x, int n, int* flag) {
    int bad = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        const double v = fma(a, x[t], y[t]);
        y[t] = v;
        if (!isfinite(v)) bad = 1;
    }
    if (flag && __syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}
// y = z + a * y  (CG direction update)
__global__ void k_xpay(double* __restrict__ y, double a, const double* __restrict__ z, int n) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) y[t] = fma(a, y[t], z[t]);
}
// xc = x + sum_{i=1..d} c_i r[i-1]    (krylov.hpp:249-253)
__global__ void k_xc(double* __restrict__ xc, const double* __restrict__ x, VecSet v, int d, int n) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double acc = x[t];
        for (int i = 1; i <= d; ++i) acc = fma(v.c[i - 1], v.p[i - 1][t], acc);
        xc[t] = acc;
    }
}
// Polynomial update (krylov.hpp:304-319), fused over all vectors.
// c layout: [0] gamma1, [1] gamma_p[ell], [2] gamma[ell], then for j=1..ell-1:
// [2+3j-2] gamma[j], [2+3j-1] gamma_pp[j], [2+3j] gamma_p[j].
__global__ void k_final_update(double* __restrict__ x, VecSet v, int ell, int n, int* flag) {
    int bad = 0;
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
        double xv = x[t];
        double r0 = v.p[0][t];
        double u0 = v.p[kMaxEll + 1][t];
        xv = fma(v.c[0], r0, xv);
        r0 = fma(-v.c[1], v.p[ell][t], r0);
        u0 = fma(-v.c[2], v.p[kMaxEll + 1 + ell][t], u0);
        for (int j = 1; j < ell; ++j) {
            u0 = fma(-v.c[3 * j], v.p[kMaxEll + 1 + j][t], u0);
            xv = fma(v.c[3 * j + 1], v.p[j][t], xv);
            r0 = fma(-v.c[3 * j + 2], v.p[j][t], r0);
        }
        x[t] = xv;
        v.p[0][t] = r0;
        v.p[kMaxEll + 1][t] = u0;
        if (!isfinite(xv)) bad = 1;
    }
    if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flag, 1);
}

}  // namespace

KrylovSolver::~KrylovSolver() {
    if (buf_) cudaFree(buf_);
    if (partials_) cudaFree(partials_);
    if (dscal_) cudaFree(dscal_);
    if (counter_) cudaFree(counter_);
    if (dflag_) cudaFree(dflag_);
    if (hpinned_) cudaFreeHost(hpinned_);
    if (hflag_) cudaFreeHost(hflag_);
}

void KrylovSolver::ensure(int n, int ell) {
    if (n == n_ && ell == ell_ && buf_) return;
    if (buf_) cudaFree(buf_);
    if (partials_) cudaFree(partials_);
    buf_ = nullptr;
    partials_ = nullptr;
    const size_t N = (size_t)std::max(n, 1);
    const int nvec = 2 * (ell + 1) + 5;
    SAP_CUDA(cudaMalloc(&buf_, sizeof(double) * N * nvec));
    SAP_CUDA(cudaMemset(buf_, 0, sizeof(double) * N * nvec));
    SAP_CUDA(cudaMalloc(&partials_, sizeof(double) * (size_t)reduce_blocks(n) * kMaxDots));
    if (!dscal_) SAP_CUDA(cudaMalloc(&dscal_, sizeof(double) * kScal));
    if (!counter_) {
        SAP_CUDA(cudaMalloc(&counter_, sizeof(unsigned)));
        SAP_CUDA(cudaMemset(counter_, 0, sizeof(unsigned)));
    }
    if (!dflag_) SAP_CUDA(cudaMalloc(&dflag_, sizeof(int)));
    if (!hpinned_) {
        SAP_CUDA(cudaHostAlloc(&hpinned_, sizeof(double) * kScal, cudaHostAllocMapped));
        SAP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dhpinned_), hpinned_, 0));
    }
    if (!hflag_) {
        SAP_CUDA(cudaHostAlloc(&hflag_, sizeof(int), cudaHostAllocMapped));
        SAP_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&dhflag_), hflag_, 0));
    }
    r_.assign(ell + 1, nullptr);
    u_.assign(ell + 1, nullptr);
    for (int i = 0; i <= ell; ++i) {
        r_[i] = buf_ + N * i;
        u_[i] = buf_ + N * (ell + 1 + i);
    }
    tmp_ = buf_ + N * (2 * (ell + 1));
    rtilde_ = tmp_ + N;
    scratch_ = rtilde_ + N;
    xc_ = scratch_ + N;
    noise_ = xc_ + N;
    n_ = n;
    ell_ = ell;
}

void KrylovSolver::sync_host() {
    SAP_CUDA(cudaStreamSynchronize(s_));
    ++syncs_;
}

double KrylovSolver::dot(const double* a, const double* b) {
    if (!dreduce_) return dots({DotReq{a, b, 0}})[0];  // k_dots with one pair is bitwise k_dot
    launch_dot(a, b, n_, partials_, counter_, dscal_, s_);
    if (dreduce_) dreduce_(dscal_, 1, s_);
    SAP_CUDA(cudaMemcpyAsync(hpinned_, dscal_, sizeof(double), cudaMemcpyDeviceToHost, s_));
    sync_host();
    if (reduce_ && !dreduce_) reduce_(hpinned_, 1);
    return hpinned_[0];
}

// Several dot products (kind 1: squared norm of a - b) in one kernel, one device->host copy and one
// synchronisation; each value bitwise the dot() of the same operands. The x-update's non-finite flag rides
// along when flag_too is set.
std::vector<double> KrylovSolver::dots(const std::vector<DotReq>& rq, bool flag_too) {
    const int m = (int)rq.size();
    // single batch, no device-side reduction over ranks: the kernel writes the values (and the x-update flag)
    // straight into the mapped host buffers -- no device->host copies between it and the synchronisation
    const bool direct = !dreduce_ && m <= kMaxDots;
    for (int q0 = 0; q0 < m; q0 += kMaxDots) {
        DotBatch d{};
        d.m = std::min(kMaxDots, m - q0);
        for (int q = 0; q < d.m; ++q) {
            d.a[q] = rq[q0 + q].a;
            d.b[q] = rq[q0 + q].b;
            d.kind[q] = rq[q0 + q].kind;
        }
        if (direct) {
            d.hout = dhpinned_;
            if (flag_too) {
                d.flag_src = dflag_;
                d.flag_dst = dhflag_;
            }
        }
        launch_dots(d, n_, partials_, counter_, dscal_ + q0, s_);
    }
    if (!direct) {
        if (dreduce_) dreduce_(dscal_, m, s_);
        SAP_CUDA(cudaMemcpyAsync(hpinned_, dscal_, sizeof(double) * m, cudaMemcpyDeviceToHost, s_));
        if (flag_too) SAP_CUDA(cudaMemcpyAsync(hflag_, dflag_, sizeof(int), cudaMemcpyDeviceToHost, s_));
    }
    sync_host();
    if (reduce_ && !dreduce_) reduce_(hpinned_, m);
    return std::vector<double>(hpinned_, hpinned_ + m);
}

bool KrylovSolver::any_flag(int local) {
    if (!reduce_) return local != 0;
    double v = local ? 1.0 : 0.0;
    reduce_(&v, 1);
    return v > 0.0;
}

bool KrylovSolver::nonfinite(const double* v) {
    SAP_CUDA(cudaMemsetAsync(dflag_, 0, sizeof(int), s_));
    launch_nonfinite(v, n_, dflag_, s_);
    SAP_CUDA(cudaMemcpyAsync(hflag_, dflag_, sizeof(int), cudaMemcpyDeviceToHost, s_));
    sync_host();
    return *hflag_ != 0;
}

KrylovResult KrylovSolver::run(const DeviceOp& A, const DeviceOp& M, const double* b, double* x, int n,
                               const KrylovConfig& cfg, cudaStream_t s, const DeviceOp2& A2) {
    s_ = s;
    syncs_ = 0;
    reduce_ = cfg.reduce;
    dreduce_ = cfg.dreduce;
    int method = cfg.method;
    if (method == 2) method = cfg.caller_asserts_spd ? 1 : 0;  // run_krylov dispatch (krylov.hpp:437-441)
    if (method == 0) {
        if (cfg.ell < 1) throw InvalidArgument("solve_krylov: ell must be at least 1");
        if (cfg.ell > kMaxEll) throw InvalidArgument("solve_krylov: ell above the supported maximum of 8");
    }
    ensure(n, method == 0 ? cfg.ell : 1);
    return method == 0 ? bicgstab(A, M, b, x, cfg, A2) : cg(A, M, b, x, cfg);
}

KrylovResult KrylovSolver::bicgstab(const DeviceOp& A, const DeviceOp& M, const double* b, double* x,
                                    const KrylovConfig& cfg, const DeviceOp2& A2) {
    const int n = n_, ell = cfg.ell;
    const int G = vgrid(n);
    KrylovResult st;
    SAP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, s_));
    double bnorm = 0.0, thr = 0.0, tr = 0.0;  // ||b||, the stopping threshold, the true residual norm
    auto record = [&](int sweep, int step, double res) {
        const long steps = (long)sweep * 2 * ell + step;
        const long quarters = (4 * steps + 2 * ell - 1) / (2 * ell);
        st.iterations = (double)quarters / 4.0;
        st.residual_history.push_back(res / bnorm);
        st.final_relative_residual = res / bnorm;
    };
    VecSet vs;
    std::memset(&vs, 0, sizeof(vs));
    for (int i = 0; i <= ell; ++i) {
        vs.p[i] = r_[i];
        vs.p[kMaxEll + 1 + i] = u_[i];
    }
    // A then M in place on the output (M's apply may alias: no copy of A's result into M's output first)
    auto apply_hat = [&](const double* in, double* out) {
        A(in, out);
        M(out, out);
    };
    // true_residual (krylov.hpp:62-72): ||b - A x|| -- A x into scratch, then the residual's squared norm in
    // the same one-sync reduction as the dot products the next step needs (each value bitwise the separate
    // k_xpay + k_dot of round 1)
    // (with A x already in scratch_ when have_ax: the fused A2 pass below)
    auto tres = [&](const double* xv, std::vector<DotReq> more, bool flag, std::vector<double>& extra,
                    bool have_ax = false) -> double {
        if (!have_ax) A(xv, scratch_);
        more.insert(more.begin(), DotReq{b, scratch_, 1});
        std::vector<double> v = dots(more, flag);
        extra.assign(v.begin() + 1, v.end());
        return std::sqrt(v[0]);
    };
    bool x_is_zero = true;  // x was just zeroed (krylov.hpp:117); false once any update is applied
    // dot products computed ahead of their use in the same synchronisation as the previous true residual
    bool have_rho = false, have_gram = false;
    double rho_next = 0.0, g11 = 0.0, g10 = 0.0;
    auto reset_iteration_state = [&](bool perturb) {
        have_rho = have_gram = false;
        if (x_is_zero && cfg.zero_guess_exact) {
            SAP_CUDA(cudaMemcpyAsync(tmp_, b, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s_));
        } else {
            A(x, tmp_);
            k_xpay<<<G, 256, 0, s_>>>(tmp_, -1.0, b, n);
            SAP_LAUNCHED();
        }
        M(tmp_, r_[0]);
        SAP_CUDA(cudaMemcpyAsync(rtilde_, r_[0], sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s_));
        if (perturb) {
            // krylov.hpp:160-165: rtilde += 1e-8 ||r0|| * U(-1,1) from mt19937(0x9d2c5680)
            std::mt19937 gen(0x9d2c5680u);
            std::uniform_real_distribution<double> dist(-1.0, 1.0);
            const double scale = 1e-8 * std::sqrt(dot(r_[0], r_[0]));
            std::vector<double> h(static_cast<size_t>(n));
            for (long long i = 0; i < cfg.row_offset; ++i) (void)dist(gen);  // this rank's slice of the stream
            for (int i = 0; i < n; ++i) h[static_cast<size_t>(i)] = dist(gen);
            SAP_CUDA(cudaMemcpyAsync(noise_, h.data(), sizeof(double) * (size_t)n, cudaMemcpyHostToDevice, s_));
            k_axpy_check<<<G, 256, 0, s_>>>(rtilde_, scale, noise_, n, nullptr);
            SAP_LAUNCHED();
            sync_host();
        }
        SAP_CUDA(cudaMemsetAsync(u_[0], 0, sizeof(double) * (size_t)n, s_));
    };

    // ||b|| and the early exits (krylov.hpp:118-133). With the exact zero-guess shortcut the first
    // preconditioned residual r0 = M b does not depend on ||b||: it is enqueued first and rho1 = (r0, r~) (r~ = r0)
    // rides with (b, b) in the same synchronisation (both values bitwise the separate dots'); if the solve
    // ends at ||b|| the speculative M b is simply not used.
    const bool spec = x_is_zero && cfg.zero_guess_exact;
    if (spec) reset_iteration_state(false);
    {
        const std::vector<double> v =
            spec ? dots({DotReq{b, b, 0}, DotReq{r_[0], rtilde_, 0}}) : std::vector<double>{dot(b, b)};
        bnorm = std::sqrt(v[0]);
        if (bnorm == 0.0) {
            st.converged = true;
            st.residual_history.push_back(0.0);
            return st;
        }
        thr = cfg.rel_tol * bnorm + cfg.abs_tol;
        tr = bnorm;
        st.residual_history.push_back(tr / bnorm);
        st.final_relative_residual = tr / bnorm;
        if (tr <= thr) {
            st.converged = true;
            return st;
        }
        if (spec) {
            rho_next = v[1];
            have_rho = true;
        }
    }
    if (!spec) reset_iteration_state(false);
    x_is_zero = false;  // the restart (reset_iteration_state(true)) always applies A to the current x
    double rho0 = 1.0, alpha = 0.0, omega = 1.0;
    bool restarted = false, breakdown = false;
    std::vector<double> gamma(ell + 1), gamma_p(ell + 1), gamma_pp(ell + 1), sigma(ell + 1);
    std::vector<double> tau((size_t)(ell + 1) * (ell + 1));
    std::vector<double> extra;
    // MGS on the device (no host round trip per tau) needs a device-side reduction; the host-callback
    // transport (gloo tests) keeps the per-dot path
    const bool device_mgs = !(reduce_ && !dreduce_);

    for (int sweep = 0; sweep < cfg.max_iterations; ++sweep) {
        breakdown = false;
        rho0 = -omega * rho0;
        for (int j = 0; j < ell && !breakdown; ++j) {
            const double rho1 = have_rho ? rho_next : dot(r_[j], rtilde_);
            have_rho = false;
            if (!std::isfinite(rho1)) { st.failure = 3; return st; }
            if (rho0 == 0.0 || rho1 == 0.0) { breakdown = true; break; }
            const double beta = alpha * rho1 / rho0;
            rho0 = rho1;
            k_u_update<<<G, 256, 0, s_>>>(vs, j, beta, n);
            SAP_LAUNCHED();
            apply_hat(u_[j], u_[j + 1]);
            const double g = dot(u_[j + 1], rtilde_);
            if (!std::isfinite(g)) { st.failure = 3; return st; }
            if (g == 0.0) { breakdown = true; break; }
            alpha = rho0 / g;
            if (A2) {
                // x += alpha u_0 does not read r_j or r_{j+1}: update x with r, then A r_j and the true
                // residual's A x in one pass over the operator (each product bitwise its own A call)
                SAP_CUDA(cudaMemsetAsync(dflag_, 0, sizeof(int), s_));
                k_r_update_x<<<G, 256, 0, s_>>>(vs, j, alpha, x, n, dflag_);
                SAP_LAUNCHED();
                A2(r_[j], r_[j + 1], x, scratch_);
                M(r_[j + 1], r_[j + 1]);
            } else {
                k_r_update<<<G, 256, 0, s_>>>(vs, j, alpha, n);
                SAP_LAUNCHED();
                apply_hat(r_[j], r_[j + 1]);
                SAP_CUDA(cudaMemsetAsync(dflag_, 0, sizeof(int), s_));
                k_axpy_check<<<G, 256, 0, s_>>>(x, alpha, u_[0], n, dflag_);
                SAP_LAUNCHED();
            }
            // with the residual: the next step's rho1 = (r_{j+1}, r~), or after the last step the first Gram
            // entries (r_1, r_1), (r_1, r_0) of the MGS trial / first MGS column (r_0..r_l are final here)
            std::vector<DotReq> ahead;
            if (j + 1 < ell)
                ahead.push_back(DotReq{r_[j + 1], rtilde_, 0});
            else if (ell >= 2) {
                ahead.push_back(DotReq{r_[1], r_[1], 0});
                ahead.push_back(DotReq{r_[1], r_[0], 0});
            }
            tr = tres(x, ahead, true, extra, (bool)A2);
            if (j + 1 < ell) {
                rho_next = extra[0];
                have_rho = true;
            } else if (ell >= 2) {
                g11 = extra[0];
                g10 = extra[1];
                have_gram = true;
            }
            if (any_flag(*hflag_)) { st.failure = 3; return st; }
            if (!std::isfinite(tr)) { st.failure = 3; return st; }
            record(sweep, j + 1, tr);
            if (tr <= thr) { st.converged = true; return st; }
        }
        if (!breakdown) {
            for (int d = 1; d < ell; ++d) {
                std::vector<double> gram((size_t)d * d), rhs(d);
                if (d == 1 && have_gram) {
                    gram[0] = g11;
                    rhs[0] = g10;
                } else {
                    std::vector<DotReq> rq;
                    for (int a = 1; a <= d; ++a) {
                        for (int c = 1; c <= d; ++c) rq.push_back(DotReq{r_[a], r_[c], 0});
                        rq.push_back(DotReq{r_[a], r_[0], 0});
                    }
                    const std::vector<double> v = dots(rq);
                    for (int a = 1; a <= d; ++a) {
                        for (int c = 1; c <= d; ++c) gram[(size_t)(a - 1) * d + (c - 1)] = v[(size_t)(a - 1) * (d + 1) + (c - 1)];
                        rhs[a - 1] = v[(size_t)(a - 1) * (d + 1) + d];
                    }
                }
                // tiny_solve with partial pivoting (krylov.hpp:76-99)
                bool solvable = true;
                {
                    std::vector<double>& am = gram;
                    for (int jj = 0; jj < d && solvable; ++jj) {
                        int piv = jj;
                        for (int i = jj + 1; i < d; ++i)
                            if (std::abs(am[(size_t)i * d + jj]) > std::abs(am[(size_t)piv * d + jj])) piv = i;
                        if (am[(size_t)piv * d + jj] == 0.0) { solvable = false; break; }
                        if (piv != jj) {
                            for (int c = 0; c < d; ++c) std::swap(am[(size_t)jj * d + c], am[(size_t)piv * d + c]);
                            std::swap(rhs[jj], rhs[piv]);
                        }
                        for (int i = jj + 1; i < d; ++i) {
                            const double l = am[(size_t)i * d + jj] / am[(size_t)jj * d + jj];
                            if (l == 0.0) continue;
                            for (int c = jj; c < d; ++c) am[(size_t)i * d + c] -= l * am[(size_t)jj * d + c];
                            rhs[i] -= l * rhs[jj];
                        }
                    }
                    if (solvable)
                        for (int i = d - 1; i >= 0; --i) {
                            double acc = rhs[i];
                            for (int jj = i + 1; jj < d; ++jj) acc -= am[(size_t)i * d + jj] * rhs[jj];
                            rhs[i] = acc / am[(size_t)i * d + i];
                        }
                }
                if (!solvable) continue;
                bool ok = true;
                for (double c : rhs) ok = ok && std::isfinite(c);
                if (!ok) continue;
                VecSet xs = vs;
                for (int i = 1; i <= d; ++i) xs.c[i - 1] = rhs[i - 1];
                k_xc<<<G, 256, 0, s_>>>(xc_, x, xs, d, n);
                SAP_LAUNCHED();
                tr = tres(xc_, {}, false, extra);
                if (!std::isfinite(tr)) continue;
                record(sweep, ell + d, tr);
                if (tr <= thr) {
                    SAP_CUDA(cudaMemcpyAsync(x, xc_, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s_));
                    st.converged = true;
                    return st;
                }
            }
            // modified Gram-Schmidt (krylov.hpp:323-334)
            if (device_mgs) {
                // every dot into its own device slot, each tau_ij = (r_j, r_i) / sigma_i formed and applied on
                // the device; one copy back, then the reference's checks in its order on the same values
                double* slot = dscal_ + 16;
                auto sl = [&](int i, int jj) { return slot + i * kMaxEll + jj; };  // tau_ij (i < j), sigma_j (i == j)
                if (have_gram) {  // sigma_1 for the device-side tau_1j quotients
                    hpinned_[kScal - 1] = g11;
                    SAP_CUDA(cudaMemcpyAsync(sl(1, 1), hpinned_ + kScal - 1, sizeof(double), cudaMemcpyHostToDevice,
                                             s_));
                }
                for (int jj = 1; jj <= ell; ++jj) {
                    for (int i = 1; i < jj; ++i) {
                        DotBatch dq{};
                        dq.m = 1;
                        dq.a[0] = r_[jj];
                        dq.b[0] = r_[i];
                        launch_dots(dq, n_, partials_, counter_, sl(i, jj), s_);
                        if (dreduce_) dreduce_(sl(i, jj), 1, s_);
                        launch_axpy_quot(r_[jj], sl(i, jj), sl(i, i), r_[i], n, s_);
                    }
                    if (jj == 1 && have_gram) continue;  // sigma_1 = (r_1, r_1), gamma'_1 from (r_1, r_0)
                    DotBatch dq{};
                    dq.m = 2;
                    dq.a[0] = r_[jj];
                    dq.b[0] = r_[jj];
                    dq.a[1] = r_[0];
                    dq.b[1] = r_[jj];
                    launch_dots(dq, n_, partials_, counter_, dscal_, s_);
                    if (dreduce_) dreduce_(dscal_, 2, s_);
                    SAP_CUDA(cudaMemcpyAsync(sl(jj, jj), dscal_, sizeof(double), cudaMemcpyDeviceToDevice, s_));
                    SAP_CUDA(cudaMemcpyAsync(slot + kMaxEll * kMaxEll + jj, dscal_ + 1, sizeof(double),
                                             cudaMemcpyDeviceToDevice, s_));
                }
                SAP_CUDA(cudaMemcpyAsync(hpinned_ + 16, slot, sizeof(double) * (kMaxEll * kMaxEll + kMaxEll + 1),
                                         cudaMemcpyDeviceToHost, s_));
                sync_host();
                const double* hs = hpinned_ + 16;
                for (int jj = 1; jj <= ell && !breakdown; ++jj) {
                    for (int i = 1; i < jj; ++i) tau[(size_t)i * (ell + 1) + jj] = hs[i * kMaxEll + jj] / sigma[i];
                    sigma[jj] = (jj == 1 && have_gram) ? g11 : hs[jj * kMaxEll + jj];
                    if (!std::isfinite(sigma[jj])) { st.failure = 3; return st; }
                    if (sigma[jj] == 0.0) { breakdown = true; break; }
                    gamma_p[jj] = ((jj == 1 && have_gram) ? g10 : hs[kMaxEll * kMaxEll + jj]) / sigma[jj];
                }
            } else {
                for (int j = 1; j <= ell && !breakdown; ++j) {
                    for (int i = 1; i < j; ++i) {
                        const double tij = dot(r_[j], r_[i]) / sigma[i];
                        tau[(size_t)i * (ell + 1) + j] = tij;
                        k_axpy_check<<<G, 256, 0, s_>>>(r_[j], -tij, r_[i], n, nullptr);
                        SAP_LAUNCHED();
                    }
                    sigma[j] = dot(r_[j], r_[j]);
                    if (!std::isfinite(sigma[j])) { st.failure = 3; return st; }
                    if (sigma[j] == 0.0) { breakdown = true; break; }
                    gamma_p[j] = dot(r_[0], r_[j]) / sigma[j];
                }
            }
            have_gram = false;
        }
        if (!breakdown) {
            gamma[ell] = gamma_p[ell];
            omega = gamma[ell];
            for (int j = ell - 1; j >= 1; --j) {
                double acc = gamma_p[j];
                for (int i = j + 1; i <= ell; ++i) acc -= tau[(size_t)j * (ell + 1) + i] * gamma[i];
                gamma[j] = acc;
            }
            for (int j = 1; j < ell; ++j) {
                double acc = gamma[j + 1];
                for (int i = j + 1; i < ell; ++i) acc += tau[(size_t)j * (ell + 1) + i] * gamma[i + 1];
                gamma_pp[j] = acc;
            }
            VecSet fs = vs;
            fs.c[0] = gamma[1];
            fs.c[1] = gamma_p[ell];
            fs.c[2] = gamma[ell];
            for (int j = 1; j < ell; ++j) {
                fs.c[3 * j] = gamma[j];
                fs.c[3 * j + 1] = gamma_pp[j];
                fs.c[3 * j + 2] = gamma_p[j];
            }
            SAP_CUDA(cudaMemsetAsync(dflag_, 0, sizeof(int), s_));
            k_final_update<<<G, 256, 0, s_>>>(x, fs, ell, n, dflag_);
            SAP_LAUNCHED();
            // with the residual: the next sweep's first rho1 = (r_0, r~)
            tr = tres(x, {DotReq{r_[0], rtilde_, 0}}, true, extra);
            rho_next = extra[0];
            have_rho = true;
            if (any_flag(*hflag_)) { st.failure = 3; return st; }
            if (!std::isfinite(tr)) { st.failure = 3; return st; }
            record(sweep, 2 * ell, tr);
            if (tr <= thr) { st.converged = true; return st; }
        }
        if (breakdown) {
            if (restarted) { st.failure = 2; return st; }
            restarted = true;
            reset_iteration_state(true);
            rho0 = 1.0;
            alpha = 0.0;
            omega = 1.0;
        }
    }
    st.iterations = (double)cfg.max_iterations;
    st.failure = 1;
    return st;
}

KrylovResult KrylovSolver::cg(const DeviceOp& A, const DeviceOp& M, const double* b, double* x,
                              const KrylovConfig& cfg) {
    // solve_cg (krylov.hpp:355-430); vectors: r = r_[0], z = r_[1], p = u_[0], q = u_[1]
    const int n = n_;
    const int G = vgrid(n);
    KrylovResult st;
    SAP_CUDA(cudaMemsetAsync(x, 0, sizeof(double) * (size_t)n, s_));
    const double bnorm = std::sqrt(dot(b, b));
    if (bnorm == 0.0) {
        st.converged = true;
        st.residual_history.push_back(0.0);
        return st;
    }
    const double thr = cfg.rel_tol * bnorm + cfg.abs_tol;
    st.residual_history.push_back(1.0);
    st.final_relative_residual = 1.0;
    if (bnorm <= thr) {
        st.converged = true;
        return st;
    }
    double *r = r_[0], *z = r_[1], *p = u_[0], *q = u_[1];
    SAP_CUDA(cudaMemcpyAsync(r, b, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s_));
    M(r, z);
    double rz = dot(r, z);
    if (!std::isfinite(rz) || rz <= 0.0) {
        st.failure = rz <= 0.0 ? 4 : 3;
        return st;
    }
    SAP_CUDA(cudaMemcpyAsync(p, z, sizeof(double) * (size_t)n, cudaMemcpyDeviceToDevice, s_));
    for (int it = 1; it <= cfg.max_iterations; ++it) {
        A(p, q);
        const double curv = dot(p, q);
        if (!std::isfinite(curv)) { st.failure = 3; return st; }
        if (curv <= 0.0) { st.failure = 4; return st; }
        const double alpha = rz / curv;
        k_axpy_check<<<G, 256, 0, s_>>>(x, alpha, p, n, nullptr);
        SAP_LAUNCHED();
        k_axpy_check<<<G, 256, 0, s_>>>(r, -alpha, q, n, nullptr);
        SAP_LAUNCHED();
        A(x, scratch_);
        k_xpay<<<G, 256, 0, s_>>>(scratch_, -1.0, b, n);
        SAP_LAUNCHED();
        const double tr = std::sqrt(dot(scratch_, scratch_));
        if (!std::isfinite(tr)) { st.failure = 3; return st; }
        st.iterations = (double)it;
        st.residual_history.push_back(tr / bnorm);
        st.final_relative_residual = tr / bnorm;
        if (tr <= thr) { st.converged = true; return st; }
        M(r, z);
        const double rz_next = dot(r, z);
        if (!std::isfinite(rz_next)) { st.failure = 3; return st; }
        if (rz_next <= 0.0) { st.failure = 4; return st; }
        const double beta = rz_next / rz;
        rz = rz_next;
        k_xpay<<<G, 256, 0, s_>>>(p, beta, z, n);
        SAP_LAUNCHED();
    }
    st.failure = 1;
    return st;
}

}  // namespace sapgpu
