// precompute.cpp -- host-side, once-per-experiment IEWPF precomputes (fp64):
//   dc_precompute_S          S = (HQH^T + R)^-1, 2x2
//   dc_precompute_local_svd  49x49 block + U Sigma^1/2
// Small dense work (a handful of coarse points and 49x49 matrices); runs on the host in
// the time of a kernel launch and is passed to the device kernels as an input.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/driftcast_gpu.h"

namespace {

int wrapm(int a, int n) {
    int r = a % n;
    return r < 0 ? r + n : r;
}

struct Geo {
    int nx, ny, c, nxc, nyc;
    double dx, dy, dxc, dyc, g, f, H, q0, l0;
};

Geo geo_of(const dc_config* cfg) {
    Geo G;
    G.nx = cfg->nx;
    G.ny = cfg->ny;
    G.c = cfg->c_omega;
    G.nxc = cfg->nx / cfg->c_omega;
    G.nyc = cfg->ny / cfg->c_omega;
    G.dx = cfg->dx;
    G.dy = cfg->dy;
    G.dxc = cfg->c_omega * cfg->dx;
    G.dyc = cfg->c_omega * cfg->dy;
    G.g = cfg->g;
    G.f = cfg->f;
    G.H = cfg->h_eq;
    G.q0 = cfg->q0;
    G.l0 = cfg->l0;
    return G;
}

// SOAR weights of the coarse spacing (stochastic.hpp:43-57), w[(db+2)*5+(da+2)]
void soar_w(const Geo& G, double dxc, double dyc, double w[25]) {
    if (G.q0 == 0.0) {
        for (int i = 0; i < 25; ++i) w[i] = 0.0;
        return;
    }
    for (int db = -2; db <= 2; ++db)
        for (int da = -2; da <= 2; ++da) {
            const double d = std::hypot(da * dxc, db * dyc);
            w[(db + 2) * 5 + (da + 2)] = G.q0 * (1.0 + d / G.l0) * std::exp(-d / G.l0);
        }
}

// apply_soar on a periodic nxc x nyc field (stochastic.hpp:49-69)
void soar(const double w[25], int nxc, int nyc, const double* in, double* out) {
    for (int b = 0; b < nyc; ++b)
        for (int a = 0; a < nxc; ++a) {
            double s = 0.0;
            for (int db = -2; db <= 2; ++db) {
                const int bb = wrapm(b + db, nyc);
                for (int da = -2; da <= 2; ++da)
                    s += w[(db + 2) * 5 + (da + 2)] * in[bb * nxc + wrapm(a + da, nxc)];
            }
            out[b * nxc + a] = s;
        }
}

// adjoint_geo_balance dipole accumulated into a zeroed field (stochastic.hpp:178-188)
void dipole(double cxc, double cyc, int nxc, int nyc, double y_hu, double y_hv, int a, int b,
            double* out) {
    out[wrapm(b + 1, nyc) * nxc + wrapm(a, nxc)] += -cyc * y_hu;
    out[wrapm(b - 1, nyc) * nxc + wrapm(a, nxc)] += cyc * y_hu;
    out[wrapm(b, nyc) * nxc + wrapm(a + 1, nxc)] += cxc * y_hv;
    out[wrapm(b, nyc) * nxc + wrapm(a - 1, nxc)] += -cxc * y_hv;
}

double catmull(double fm1, double f0, double f1, double f2, double t) { // stochastic.hpp:81-87
    double a = 2.0 * f0;
    double b = f1 - fm1;
    double c = 2.0 * fm1 - 5.0 * f0 + 4.0 * f1 - f2;
    double d = -fm1 + 3.0 * f0 - 3.0 * f1 + f2;
    return 0.5 * (a + t * (b + t * (c + t * d)));
}

// interpolate_bicubic at one fine cell (stochastic.hpp:96-114)
double interp_at(const Geo& G, int oj, int ok, const double* cf, int j, int k) {
    const double inv_c = 1.0 / G.c;
    const double yc = (k - ok) * inv_c;
    const int b0 = static_cast<int>(std::floor(yc));
    const double ty = yc - b0;
    const double xc = (j - oj) * inv_c;
    const int a0 = static_cast<int>(std::floor(xc));
    const double tx = xc - a0;
    int as[4], bs[4];
    for (int m = 0; m < 4; ++m) {
        as[m] = wrapm(a0 - 1 + m, G.nxc);
        bs[m] = wrapm(b0 - 1 + m, G.nyc);
    }
    double col[4];
    for (int m = 0; m < 4; ++m) {
        const double* row = cf + bs[m] * G.nxc;
        col[m] = catmull(row[as[0]], row[as[1]], row[as[2]], row[as[3]], tx);
    }
    return catmull(col[0], col[1], col[2], col[3], ty);
}

// cyclic Jacobi eigen-decomposition of a symmetric n x n matrix: A = V diag(l) V^T
void jacobi_eigh(int n, std::vector<double> A, std::vector<double>& V, std::vector<double>& l) {
    V.assign(static_cast<size_t>(n) * n, 0.0);
    for (int i = 0; i < n; ++i) V[i * n + i] = 1.0;
    double norm = 0.0;
    for (double x : A) norm += x * x;
    for (int sweep = 0; sweep < 100; ++sweep) {
        double off = 0.0;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) off += A[p * n + q] * A[p * n + q];
        if (off <= 1e-34 * norm) break;
        for (int p = 0; p < n; ++p)
            for (int q = p + 1; q < n; ++q) {
                const double apq = A[p * n + q];
                if (std::fabs(apq) < 1e-300) continue;
                const double app = A[p * n + p], aqq = A[q * n + q];
                const double theta = (aqq - app) / (2.0 * apq);
                const double t = (theta >= 0.0 ? 1.0 : -1.0) /
                                 (std::fabs(theta) + std::sqrt(theta * theta + 1.0));
                const double c = 1.0 / std::sqrt(t * t + 1.0), s = t * c;
                for (int k = 0; k < n; ++k) {
                    const double akp = A[k * n + p], akq = A[k * n + q];
                    A[k * n + p] = c * akp - s * akq;
                    A[k * n + q] = s * akp + c * akq;
                }
                for (int k = 0; k < n; ++k) {
                    const double apk = A[p * n + k], aqk = A[q * n + k];
                    A[p * n + k] = c * apk - s * aqk;
                    A[q * n + k] = s * apk + c * aqk;
                }
                for (int k = 0; k < n; ++k) {
                    const double vkp = V[k * n + p], vkq = V[k * n + q];
                    V[k * n + p] = c * vkp - s * vkq;
                    V[k * n + q] = s * vkp + c * vkq;
                }
            }
    }
    l.resize(n);
    for (int i = 0; i < n; ++i) l[i] = A[i * n + i];
}

} // namespace

extern "C" {

// S at observation cell (0,0): push [1,0] and [0,1] through
// H^T -> Lambda -> GB^T -> SOAR -> SOAR -> I -> GB -> H, add R, invert.
dc_status dc_precompute_S(const dc_config* cfg, double r_hu, double r_hv, double* hqht,
                          double* S) {
    if (!cfg || cfg->c_omega <= 0 || cfg->nx % cfg->c_omega || cfg->ny % cfg->c_omega)
        return DC_EINVAL;
    const Geo G = geo_of(cfg);
    const int j = 0, k = 0, oj = 0, ok = 0, a = 0, b = 0;  // aligned: (0 % c, 0 % c)
    double w[25];
    soar_w(G, G.dxc, G.dyc, w);
    const double cyc = G.g * G.H / (G.f * 2.0 * G.dyc), cxc = G.g * G.H / (G.f * 2.0 * G.dxc);
    const double cy = G.g * G.H / (G.f * 2.0 * G.dy), cx = G.g * G.H / (G.f * 2.0 * G.dx);
    const size_t nr = static_cast<size_t>(G.nxc) * G.nyc;
    std::vector<double> dip(nr), s1(nr), s2(nr);
    double m[4];
    for (int col = 0; col < 2; ++col) {
        std::fill(dip.begin(), dip.end(), 0.0);
        dipole(cxc, cyc, G.nxc, G.nyc, col == 0 ? 1.0 : 0.0, col == 0 ? 0.0 : 1.0, a, b, dip.data());
        if (G.q0 == 0.0) {
            std::fill(s2.begin(), s2.end(), 0.0);
        } else {
            soar(w, G.nxc, G.nyc, dip.data(), s1.data());
            soar(w, G.nxc, G.nyc, s1.data(), s2.data());
        }
        const double dN = interp_at(G, oj, ok, s2.data(), j, wrapm(k + 1, G.ny));
        const double dS = interp_at(G, oj, ok, s2.data(), j, wrapm(k - 1, G.ny));
        const double dE = interp_at(G, oj, ok, s2.data(), wrapm(j + 1, G.nx), k);
        const double dW = interp_at(G, oj, ok, s2.data(), wrapm(j - 1, G.nx), k);
        m[0 * 2 + col] = -cy * (dN - dS);
        m[1 * 2 + col] = cx * (dE - dW);
    }
    for (int i = 0; i < 4; ++i) hqht[i] = m[i];
    const double A = m[0] + r_hu, B = m[1], C = m[2], D = m[3] + r_hv;
    const double det = A * D - B * C;
    if (!(det != 0.0) || !std::isfinite(det)) return DC_EINVAL;
    S[0] = D / det;
    S[1] = -B / det;
    S[2] = -C / det;
    S[3] = A / det;
    return DC_OK;
}

dc_status dc_precompute_local_svd(const dc_config* cfg, const double* S, double* block,
                                  double* usig) {
    if (!cfg || !S || cfg->c_omega <= 0) return DC_EINVAL;
    const Geo G = geo_of(cfg);
    const int N = 15, ca = N / 2, cb = N / 2;
    double w[25];
    soar_w(G, G.dxc, G.dyc, w);
    const double cyc = G.g * G.H / (G.f * 2.0 * G.dyc), cxc = G.g * G.H / (G.f * 2.0 * G.dxc);
    std::vector<double> dip(N * N), K0(N * N), K1(N * N);
    std::fill(dip.begin(), dip.end(), 0.0);
    dipole(cxc, cyc, N, N, 1.0, 0.0, ca, cb, dip.data());
    soar(w, N, N, dip.data(), K0.data());
    std::fill(dip.begin(), dip.end(), 0.0);
    dipole(cxc, cyc, N, N, 0.0, 1.0, ca, cb, dip.data());
    soar(w, N, N, dip.data(), K1.data());
    std::vector<double> B(49 * 49);
    for (int r = 0; r < 49; ++r) {
        const int ra = ca + (r % 7) - 3, rb = cb + (r / 7) - 3;
        const double kr0 = K0[rb * N + ra], kr1 = K1[rb * N + ra];
        for (int c2 = 0; c2 < 49; ++c2) {
            const int sa = ca + (c2 % 7) - 3, sb = cb + (c2 / 7) - 3;
            const double kc0 = K0[sb * N + sa], kc1 = K1[sb * N + sa];
            const double a = kr0 * (S[0] * kc0 + S[1] * kc1) + kr1 * (S[2] * kc0 + S[3] * kc1);
            B[r * 49 + c2] = (r == c2 ? 1.0 : 0.0) - a;
        }
    }
    if (block) std::memcpy(block, B.data(), B.size() * sizeof(double));
    std::vector<double> V, l;
    jacobi_eigh(49, B, V, l);
    for (int r = 0; r < 49; ++r)
        for (int c2 = 0; c2 < 49; ++c2) usig[r * 49 + c2] = V[r * 49 + c2] * std::sqrt(std::max(l[c2], 0.0));
    return DC_OK;
}

} // extern "C"
