// ============================================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A plain, slow, obviously-correct CPU implementation of the GS-SLAM differentiable RGB-D
// splatting renderer (arXiv 2311.11700), written from PAPER.md and the readings recorded in
// DESIGN.md §3 (= SURVEY.md §8(c) O1-O4). Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library. It shares NO code, header,
// table or constant generator with the CUDA path (paper_2311_11700_b200/csrc).
//
// Precision: templated on the decision type R.
//   R = double : everything in fp64 (used by the finite-difference pins).
//   R = float  : every value that feeds a DISCRETE decision (cull, radius, tile rect, depth
//                key, alpha skip, termination) is computed in fp32 with a fixed operation
//                order and no FMA contraction (build with -ffp-contract=off), because the
//                kernel takes those decisions in fp32 (task rule: "both sides take that
//                decision in the same precision ... the kernel's"). Image accumulation and
//                all gradients are fp64.
//
// Build: g++ -O2 -fopenmp -ffp-contract=off -fno-fast-math -shared -fPIC oracle.cpp
//
// Citations: P:n = /root/reference/PAPER.md line n (section / equation named beside it).
// ============================================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <numeric>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

extern "C" {
struct OracleCam {          // host camera, doubles; the float path rounds each field to float once
    double fx, fy, cx, cy;
    int32_t width, height;
    double znear;           // DESIGN.md reading C13 (0.2 m)
    double bg[3];           // C15
    double dil;             // C11 (0.3 px^2 added to Sigma')
};
}

namespace {

constexpr int TILE = 16;    // BASELINE.json north_star: 16x16 tiles

template <class R> struct Cam {
    R fx, fy, cx, cy, znear, dil;
    int W, H, GX, GY;
    int sh;                 // colour model: 0 = RGB rows 11-13 (reading C17), 1 = degree-1 SH (C29)
    bool orad;              // radius: false = 3 sigma (C11), true = alpha >= 1/255 reach (C33)
    bool o3pow;             // power in SURVEY.md §8(c) O3's printed order instead of R1's fma order
    double bg[3];
    // mode = sh_degree | (opacity_radius << 8) | (o3_power_order << 9)
    explicit Cam(const OracleCam& c, int mode = 0)
        : fx(R(c.fx)), fy(R(c.fy)), cx(R(c.cx)), cy(R(c.cy)), znear(R(c.znear)), dil(R(c.dil)),
          W(c.width), H(c.height), GX((c.width + TILE - 1) / TILE), GY((c.height + TILE - 1) / TILE),
          sh(mode & 0xff), orad(((mode >> 8) & 1) != 0), o3pow(((mode >> 9) & 1) != 0) {
        for (int k = 0; k < 3; ++k) bg[k] = c.bg[k];
    }
};

constexpr int MAXP = 23;    // parameter rows: 14 (RGB) or 23 (degree-1 SH, 12 coefficients)
inline int n_rows(int sh) { return sh == 1 ? 23 : 14; }

// Degree-1 real spherical harmonics (reading C29: the basis and the 0.5 offset / clamp at 0 of the
// 3DGS rasterizer the paper extends; the paper fixes only "1-degree SH per colour channel,
// 12 coefficients"). Coefficient Y[k][c] is parameter row 11 + 3k + c (k = 0 the constant
// term, k = 1..3 the linear terms), so degree 0 keeps the RGB rows' positions.
constexpr double SH_C0 = 0.28209479177387814;   // 1 / (2 sqrt(pi))
constexpr double SH_C1 = 0.4886025119029199;    // sqrt(3) / (2 sqrt(pi))

// ---------------------------------------------------------------- O1: projection (Eq. 2-3)
template <class R> struct Proj {
    bool in_front = false;             // passed the cull tests (z > znear, |q| > 0, det > 0)
    R xc = 0, yc = 0, zc = 0;          // X^c = W X + t   ("X_i^c = P X_i")
    R A = 0, B = 0, C = 0, det = 0;    // Sigma' (+ dilation), Eq. 3
    R ca = 0, cb = 0, cc = 0;          // conic = Sigma'^-1
    R mx = 0, my = 0;                  // projected mean m_i
    int32_t radius = 0;
    int32_t xlo = 0, xhi = 0, ylo = 0, yhi = 0;
    uint32_t tiles = 0;
    R rgb[3] = {0, 0, 0};              // colour (RGB rows, or degree-1 SH at the view direction)
    bool lit[3] = {true, true, true};  // SH: channel not clamped at 0 (the gradient flows)
};

// Colour of one Gaussian (SH degree 1): view direction from the camera centre c = -W^T t to the
// mean, in world coordinates; fp32 in the fixed order below when R = float (the clamp at 0 decides
// whether the channel's gradient flows, so both sides take it in fp32).
template <class R> static void sh1_colour(const R* p, const R* V, R rgb[3], bool lit[3]) {
    const R cwx = -((V[0] * V[3] + V[4] * V[7]) + V[8] * V[11]);
    const R cwy = -((V[1] * V[3] + V[5] * V[7]) + V[9] * V[11]);
    const R cwz = -((V[2] * V[3] + V[6] * V[7]) + V[10] * V[11]);
    const R dx = p[0] - cwx, dy = p[1] - cwy, dz = p[2] - cwz;
    const R len = std::sqrt((dx * dx + dy * dy) + dz * dz);
    const R ux = dx / len, uy = dy / len, uz = dz / len;
    for (int c = 0; c < 3; ++c) {
        const R lin = ((-(uy * p[14 + c]) + uz * p[17 + c]) - ux * p[20 + c]);
        const R v = (R(SH_C0) * p[11 + c] + R(SH_C1) * lin) + R(0.5);
        lit[c] = v > R(0);
        rgb[c] = lit[c] ? v : R(0);
    }
}

template <class R> static inline int32_t clamp_tile(R v, int hi) {
    // clamp in floating point first (no UB on huge values), then convert exactly
    if (!(v > R(0))) return 0;   // also maps NaN -> 0
    if (v > R(hi)) return hi;
    return int32_t(v);
}

template <class R> static inline uint32_t bits_of(R z);
template <> inline uint32_t bits_of<float>(float z) { uint32_t u; std::memcpy(&u, &z, 4); return u; }
template <> inline uint32_t bits_of<double>(double z) { float f = float(z); uint32_t u; std::memcpy(&u, &f, 4); return u; }

// p[k] = parameter row k of one Gaussian: mean xyz, scale xyz, quat r i j k, opacity, rgb.
// V = world->camera 3x4 row-major. Steps numbered as DESIGN.md §3 O1.
template <class R> static Proj<R> project_one(const R* p, const R* V, const Cam<R>& cam) {
    Proj<R> g;
    if (cam.sh == 1) sh1_colour(p, V, g.rgb, g.lit);
    else for (int c = 0; c < 3; ++c) g.rgb[c] = p[11 + c];
    const R x = p[0], y = p[1], z = p[2];
    // 1. camera coordinates
    g.xc = ((V[0] * x + V[1] * y) + V[2] * z) + V[3];
    g.yc = ((V[4] * x + V[5] * y) + V[6] * z) + V[7];
    g.zc = ((V[8] * x + V[9] * y) + V[10] * z) + V[11];
    // 2. near-plane cull (NaN fails)
    if (!(g.zc > cam.znear)) return g;
    // 3. normalise the rotation quaternion (Eq. 2 stores R "as a 4D quaternion")
    const R qr0 = p[6], qi0 = p[7], qj0 = p[8], qk0 = p[9];
    const R n2 = ((qr0 * qr0 + qi0 * qi0) + qj0 * qj0) + qk0 * qk0;
    if (!(n2 > R(0))) return g;
    const R nq = std::sqrt(n2);
    const R qr = qr0 / nq, qi = qi0 / nq, qj = qj0 / nq, qk = qk0 / nq;
    // 4. rotation matrix, Eq. S1, evaluated as printed
    R Rm[3][3];
    Rm[0][0] = R(1) - R(2) * (qj * qj + qk * qk);
    Rm[0][1] = R(2) * (qi * qj - qr * qk);
    Rm[0][2] = R(2) * (qi * qk + qr * qj);
    Rm[1][0] = R(2) * (qi * qj + qr * qk);
    Rm[1][1] = R(1) - R(2) * (qi * qi + qk * qk);
    Rm[1][2] = R(2) * (qj * qk - qr * qi);
    Rm[2][0] = R(2) * (qi * qk - qr * qj);
    Rm[2][1] = R(2) * (qj * qk + qr * qi);
    Rm[2][2] = R(1) - R(2) * (qi * qi + qj * qj);
    // 5. Sigma = R S S^T R^T (Eq. 2), M = R diag(s)
    R M[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) M[a][k] = Rm[a][k] * p[3 + k];
    R S[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = a; b < 3; ++b) {
            S[a][b] = (M[a][0] * M[b][0] + M[a][1] * M[b][1]) + M[a][2] * M[b][2];
            S[b][a] = S[a][b];
        }
    // 6. Sigma' = J W Sigma W^T J^T + dil I  (Eq. 3 with the rotation block W, readings C1/C2)
    const R tx = g.xc / g.zc, ty = g.yc / g.zc;
    const R j00 = cam.fx / g.zc, j11 = cam.fy / g.zc;
    const R j02 = -(j00 * tx), j12 = -(j11 * ty);
    R E[2][3];
    for (int k = 0; k < 3; ++k) {
        E[0][k] = j00 * V[0 * 4 + k] + j02 * V[2 * 4 + k];
        E[1][k] = j11 * V[1 * 4 + k] + j12 * V[2 * 4 + k];
    }
    R U[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) U[a][k] = (E[a][0] * S[0][k] + E[a][1] * S[1][k]) + E[a][2] * S[2][k];
    g.A = ((U[0][0] * E[0][0] + U[0][1] * E[0][1]) + U[0][2] * E[0][2]) + cam.dil;
    g.B = (U[0][0] * E[1][0] + U[0][1] * E[1][1]) + U[0][2] * E[1][2];
    g.C = ((U[1][0] * E[1][0] + U[1][1] * E[1][1]) + U[1][2] * E[1][2]) + cam.dil;
    // 7. conic
    g.det = g.A * g.C - g.B * g.B;
    if (!(g.det > R(0))) return g;
    const R inv = R(1) / g.det;
    g.ca = g.C * inv;
    g.cb = -(g.B * inv);
    g.cc = g.A * inv;
    // 8. 3-sigma radius of the larger eigenvalue (reading C11), clamped to 2^24 px; or (reading
    //    C33) the reach of alpha = o exp(-q/2) >= 1/255: q <= q_o = 2 ln(255 o) (o <= 1/255 never
    //    reaches the skip threshold: culled), with a margin q_m = q_o + 2e-3; r = ceil(sqrt(q_m
    //    lambda_max)) and the ellipse's bounding box |x| <= sqrt(q_m A), |y| <= sqrt(q_m C)
    const R mid = R(0.5) * (g.A + g.C);
    const R lam1 = mid + std::sqrt(std::max(R(0.1), mid * mid - g.det));
    R rf, rx = 0, ry = 0;
    if (cam.orad) {
        const R qo = R(2.0 * std::log(255.0 * double(p[10])));
        if (!(qo > R(0))) return g;   // radius 0, no tiles
        const R qm = qo + R(2e-3f);
        rf = std::ceil(std::sqrt(qm * lam1));
        rx = std::sqrt(qm * g.A);
        ry = std::sqrt(qm * g.C);
    } else {
        rf = std::ceil(R(3) * std::sqrt(lam1));
    }
    if (!(rf < R(16777216))) rf = R(16777216);
    g.radius = int32_t(rf);
    // 9. projected mean m_i (pinhole)
    g.mx = cam.fx * tx + cam.cx;
    g.my = cam.fy * ty + cam.cy;
    // 10. tile rect [xlo, xhi) x [ylo, yhi): the 3DGS box of the 3-sigma radius, or (C33) the tiles
    //     holding the integer pixels of [ceil(m - r), floor(m + r)] per axis
    if (cam.orad) {
        g.xlo = clamp_tile(std::floor(std::ceil(g.mx - rx) / R(TILE)), cam.GX);
        g.xhi = clamp_tile(std::floor(std::floor(g.mx + rx) / R(TILE)) + R(1), cam.GX);
        g.ylo = clamp_tile(std::floor(std::ceil(g.my - ry) / R(TILE)), cam.GY);
        g.yhi = clamp_tile(std::floor(std::floor(g.my + ry) / R(TILE)) + R(1), cam.GY);
    } else {
        const R r = R(g.radius);
        g.xlo = clamp_tile(std::floor((g.mx - r) / R(TILE)), cam.GX);
        g.xhi = clamp_tile(std::floor(((g.mx + r) + R(TILE - 1)) / R(TILE)), cam.GX);
        g.ylo = clamp_tile(std::floor((g.my - r) / R(TILE)), cam.GY);
        g.yhi = clamp_tile(std::floor(((g.my + r) + R(TILE - 1)) / R(TILE)), cam.GY);
    }
    g.tiles = uint32_t(std::max(0, g.xhi - g.xlo)) * uint32_t(std::max(0, g.yhi - g.ylo));
    g.in_front = true;
    return g;
}

template <class R> static void gather_params(const R* params, int64_t ld, int64_t i, R* p, int rows) {
    for (int k = 0; k < rows; ++k) p[k] = params[k * ld + i];
}

template <class R> static std::vector<Proj<R>> project_all(const R* params, int64_t n, int64_t ld, const R* V,
                                                           const Cam<R>& cam) {
    std::vector<Proj<R>> out(static_cast<size_t>(n));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; ++i) {
        R p[MAXP];
        gather_params(params, ld, i, p, n_rows(cam.sh));
        out[size_t(i)] = project_one(p, V, cam);
    }
    return out;
}

// Global depth order of on-screen Gaussians, ties by index (reading C16): the plain definition
// of "sorting the Gaussians in depth order" (Eq. 4 text).
template <class R> static std::vector<int64_t> depth_order(const std::vector<Proj<R>>& pj) {
    std::vector<int64_t> idx;
    for (int64_t i = 0; i < int64_t(pj.size()); ++i)
        if (pj[size_t(i)].tiles > 0) idx.push_back(i);
    std::stable_sort(idx.begin(), idx.end(), [&](int64_t a, int64_t b) {
        return pj[size_t(a)].zc < pj[size_t(b)].zc;   // z > znear > 0: float order == key-bit order
    });
    return idx;
}

// ---------------------------------------------------------------- O3: per-pixel blending
template <class R> static inline R exp_r(R x);
template <> inline float exp_r<float>(float x) { return float(std::exp(double(x))); }
template <> inline double exp_r<double>(double x) { return std::exp(x); }

struct Contrib {          // one blended Gaussian of one pixel
    int64_t i;
    double alpha, G, dx, dy;
    bool clamped;
};

struct PixelResult {
    double color[3] = {0, 0, 0}, depth = 0, T = 1;
    uint32_t n_last = 0, examined = 0;
    uint8_t ambiguous = 0;
    uint64_t hash = 1469598103934665603ull;   // FNV-1a over the decision sequence
    std::vector<Contrib> list;
};

static inline void fnv(uint64_t& h, uint64_t v) {
    for (int b = 0; b < 8; ++b) { h ^= (v >> (8 * b)) & 0xff; h *= 1099511628211ull; }
}

// Eq. 4-5 and the cumulative opacity of Eq. 8, front to back over the
// global depth order; Gaussian i is a candidate for pixel (u,v) iff the pixel's tile lies in
// rect_i (O3). alpha = min(0.99, o G); skip alpha < 1/255; stop before blending a
// Gaussian that would take T below 1e-4 (reading C9). replay_nlast >= 0 replaces the
// termination test by "blend every non-skipped candidate at positions <= replay_nlast"
// (parity tie rule).
template <class R>
static void blend_pixel(int u, int v, const std::vector<Proj<R>>& pj, const std::vector<int64_t>& order,
                        const R* params, int64_t ld, const Cam<R>& cam, int64_t replay_nlast, bool keep_list,
                        PixelResult& out, bool flip_skip_ties = false) {
    const int tx = u / TILE, ty = v / TILE;
    const R fu = R(u), fv = R(v);
    const R a_min = R(1) / R(255), a_max = R(0.99), t_min = R(1e-4);
    R T = R(1);
    uint32_t j = 0;
    // Tie band (reading R1): a conforming fp32 evaluation may differ from this one by
    // the exp's error (<= 2^-20 relative incl. argument rounding) and the power's evaluation order
    // (perr below) in every unclamped alpha; the resulting relative divergence of T is bounded by
    // sum_k ((2^-20 + perr_k) alpha_k / (1 - alpha_k) + 2^-23). A decision value within that band
    // (floor 1e-5 relative) of its threshold marks the pixel ambiguous.
    double t_band = 0.0;
    for (int64_t i : order) {
        const Proj<R>& g = pj[size_t(i)];
        if (tx < g.xlo || tx >= g.xhi || ty < g.ylo || ty >= g.yhi) continue;
        ++j;
        if (replay_nlast >= 0 && int64_t(j) > replay_nlast) break;
        out.examined = j;
        const R dx = g.mx - fu, dy = g.my - fv;
        // power = -1/2 (a dx^2 + 2 b dx dy + c dy^2), evaluated in fp32 as two fused multiply-adds on
        // the exactly scaled coefficients A = -a/2, B = -b, C = -c/2 (reading R1: the
        // order every fp32 evaluation of this decision value uses, oracle and kernel alike)
        const R A2 = R(-0.5) * g.ca, B2 = -g.cb, C2 = R(-0.5) * g.cc;
        // cam.o3pow: the order SURVEY.md §8(c) O3 prints, each operation rounded separately; used
        // only by the pin that both orders take the same decisions outside the tie band
        const R power = cam.o3pow ? R(R(-0.5) * ((g.ca * dx) * dx + (g.cc * dy) * dy)) - (g.cb * dx) * dy
                                  : std::fma(A2 * dx, dx, std::fma(C2 * dy, dy, (B2 * dx) * dy));
        if (power > R(0)) continue;
        const R G = exp_r<R>(power);
        const R o = params[10 * ld + i];
        const R og = o * G;
        const R alpha = std::min(a_max, og);
        // any fp32 evaluation order of the power's three terms (R1's fma order, O3's printed order)
        // is within 4 u (sum of the terms' magnitudes) of the exact value, u = 2^-24; the relative
        // change of alpha is that absolute change of the power
        const double perr = 2.384185791015625e-07 * (std::fabs(double(A2) * double(dx) * double(dx)) +
                                                     std::fabs(double(C2) * double(dy) * double(dy)) +
                                                     std::fabs(double(B2) * double(dx) * double(dy)));
        const bool amb_skip = std::fabs(double(alpha) - double(a_min)) <= std::max(1e-5, 9.5367431640625e-07 + perr) * double(a_min);
        if (amb_skip) out.ambiguous = 1;
        bool skip = alpha < a_min;
        if (flip_skip_ties && amb_skip) skip = !skip;   // tie-rule replay: take the other decision
        if (skip) continue;
        const R Tn = T * (R(1) - alpha);
        const bool clamped = og > a_max;
        const double step_band =
            (clamped ? 0.0 : (9.5367431640625e-07 + perr) * double(alpha) / (1.0 - double(alpha))) +
            1.1920928955078125e-07;
        if (replay_nlast < 0) {
            const double band = std::max(1e-5, t_band + step_band);
            if (std::fabs(double(Tn) - double(t_min)) <= band * double(t_min)) out.ambiguous = 1;
            if (Tn < t_min) break;   // terminating Gaussian is not blended
        }
        t_band += step_band;
        const double w = double(alpha) * double(T);
        for (int c = 0; c < 3; ++c) out.color[c] += w * double(g.rgb[c]);
        out.depth += w * double(g.zc);
        T = Tn;
        out.n_last = j;
        fnv(out.hash, uint64_t(i) * 2 + (clamped ? 1 : 0));
        if (keep_list) out.list.push_back(Contrib{i, double(alpha), double(G), double(dx), double(dy), clamped});
    }
    out.T = double(T);
    for (int c = 0; c < 3; ++c) out.color[c] += out.T * cam.bg[c];
}

// ---------------------------------------------------------------- O4: analytic backward
struct ScreenGrad {      // per-Gaussian dL/d(screen quantities), fp64
    double mx, my, a, b, c, o, r, g, bl, d;
};

static inline void atomic_add(double& dst, double v) {
#pragma omp atomic update
    dst += v;
}

// Per-pixel gradient of L through Eq. 4-5 for the fixed contributor set. dL/dalpha_i is Eq. S6
// for depth and its colour analogue, plus the background term; suffix sums in fp64.
template <class R>
static void backward_pixel(const PixelResult& px, const std::vector<Proj<R>>& pj, const R* params, int64_t ld,
                           const Cam<R>& cam, const double dLdC[3], double dLdD, std::vector<ScreenGrad>& sg,
                           std::vector<ScreenGrad>* sa = nullptr) {
    const size_t n = px.list.size();
    if (n == 0) return;
    std::vector<double> T(static_cast<size_t>(n + 1));
    T[0] = 1.0;
    for (size_t k = 0; k < n; ++k) T[k + 1] = T[k] * (1.0 - px.list[k].alpha);
    const double Tf = T[n];
    double bg_dot = 0;
    for (int c = 0; c < 3; ++c) bg_dot += cam.bg[c] * dLdC[c];
    // suffix sums  Rsum_k = sum_{m>k} c_m w_m ,  Dsum_k = sum_{m>k} d_m w_m
    double Rs[3] = {0, 0, 0}, Ds = 0;
    for (size_t kk = n; kk-- > 0;) {
        const Contrib& ct = px.list[kk];
        const int64_t i = ct.i;
        const double rgb[3] = {double(pj[size_t(i)].rgb[0]), double(pj[size_t(i)].rgb[1]), double(pj[size_t(i)].rgb[2])};
        const double d = double(pj[size_t(i)].zc);
        const double Ti = T[kk], a = ct.alpha, w = a * Ti;
        // dC/dalpha_i = c_i T_i - (sum_{m>i} c_m w_m + T_f bg)/(1 - alpha_i);  same for D without bg
        double g_alpha = 0;
        for (int c = 0; c < 3; ++c) g_alpha += (rgb[c] * Ti - Rs[c] / (1.0 - a)) * dLdC[c];
        g_alpha += (d * Ti - Ds / (1.0 - a)) * dLdD;
        g_alpha -= Tf / (1.0 - a) * bg_dot;
        ScreenGrad& s = sg[size_t(i)];
        atomic_add(s.r, w * dLdC[0]);
        atomic_add(s.g, w * dLdC[1]);
        atomic_add(s.bl, w * dLdC[2]);
        atomic_add(s.d, w * dLdD);   // Eq. S6 second line: dD/dd_i = alpha_i T_i
        if (!ct.clamped) {           // reading C10: zero derivative past the 0.99 clamp
            const Proj<R>& g = pj[size_t(i)];
            const double o = double(params[10 * ld + i]);
            const double ca = double(g.ca), cb = double(g.cb), cc = double(g.cc);
            const double gp = o * ct.G * g_alpha;   // dL/dpower
            atomic_add(s.o, ct.G * g_alpha);
            atomic_add(s.mx, -gp * (ca * ct.dx + cb * ct.dy));
            atomic_add(s.my, -gp * (cb * ct.dx + cc * ct.dy));
            atomic_add(s.a, -0.5 * gp * ct.dx * ct.dx);
            atomic_add(s.b, -gp * ct.dx * ct.dy);
            atomic_add(s.c, -0.5 * gp * ct.dy * ct.dy);
        }
        if (sa) {   // magnitude of every term of this pixel's contribution (the error-bound scale)
            double ga = 0;
            for (int c = 0; c < 3; ++c)
                ga += (std::fabs(rgb[c]) * Ti + std::fabs(Rs[c]) / (1.0 - a)) * std::fabs(dLdC[c]);
            ga += (std::fabs(d) * Ti + std::fabs(Ds) / (1.0 - a)) * std::fabs(dLdD);
            double bga = 0;
            for (int c = 0; c < 3; ++c) bga += std::fabs(cam.bg[c] * dLdC[c]);
            ga += Tf / (1.0 - a) * bga;
            ScreenGrad& m = (*sa)[size_t(i)];
            atomic_add(m.r, std::fabs(w * dLdC[0]));
            atomic_add(m.g, std::fabs(w * dLdC[1]));
            atomic_add(m.bl, std::fabs(w * dLdC[2]));
            atomic_add(m.d, std::fabs(w * dLdD));
            if (!ct.clamped) {
                const Proj<R>& g = pj[size_t(i)];
                const double o = std::fabs(double(params[10 * ld + i]));
                const double ca = std::fabs(double(g.ca)), cb = std::fabs(double(g.cb)), cc = std::fabs(double(g.cc));
                const double adx = std::fabs(ct.dx), ady = std::fabs(ct.dy), gp = o * ct.G * ga;
                atomic_add(m.o, ct.G * ga);
                atomic_add(m.mx, gp * (ca * adx + cb * ady));
                atomic_add(m.my, gp * (cb * adx + cc * ady));
                atomic_add(m.a, 0.5 * gp * adx * adx);
                atomic_add(m.b, gp * adx * ady);
                atomic_add(m.c, 0.5 * gp * ady * ady);
            }
        }
        for (int c = 0; c < 3; ++c) Rs[c] += rgb[c] * w;
        Ds += d * w;
    }
}

// dR(q)/dq of Eq. S1 for unit q = (r, i, j, k): dR[a][b][m] = dR_ab / dq_m
static void dR_dq(const double q[4], double dR[3][3][4]) {
    const double r = q[0], i = q[1], j = q[2], k = q[3];
    const double t[3][3][4] = {
        {{0, 0, -4 * j, -4 * k}, {-2 * k, 2 * j, 2 * i, -2 * r}, {2 * j, 2 * k, 2 * r, 2 * i}},
        {{2 * k, 2 * j, 2 * i, 2 * r}, {0, -4 * i, 0, -4 * k}, {-2 * i, -2 * r, 2 * k, 2 * j}},
        {{-2 * j, 2 * k, -2 * r, 2 * i}, {2 * i, 2 * r, 2 * k, 2 * j}, {0, -4 * i, -4 * j, 0}}};
    std::memcpy(dR, t, sizeof(t));
}

static void rot_of(const double q[4], double Rm[3][3]) {   // Eq. S1
    const double r = q[0], i = q[1], j = q[2], k = q[3];
    Rm[0][0] = 1 - 2 * (j * j + k * k); Rm[0][1] = 2 * (i * j - r * k); Rm[0][2] = 2 * (i * k + r * j);
    Rm[1][0] = 2 * (i * j + r * k); Rm[1][1] = 1 - 2 * (i * i + k * k); Rm[1][2] = 2 * (j * k - r * i);
    Rm[2][0] = 2 * (i * k - r * j); Rm[2][1] = 2 * (j * k + r * i); Rm[2][2] = 1 - 2 * (i * i + j * j);
}

struct GaussianBack {     // result of the per-Gaussian chain (fp64)
    double grad[MAXP];    // dL/d(mean xyz, scale xyz, raw quat rijk, opacity, rgb | SH coefficients)
    double gdir[3];       // dL/dX (world) through the SH view direction (0 for RGB)
    double dXc_full[3];   // dL/dX^c through mean, depth and J paths
    double dXc_noJ[3];    // dL/dX^c through mean and depth only (paper mode)
    double dW[3][3];      // dL/dW through Sigma' (covariance path, Eq. S4-S5)
    double Xc[3];
};

// Chain the screen-space gradient of Gaussian i back to its 14 parameters and the pose
// (Eq. 11 P:155-168 and Supplement A). Recomputed in fp64 from the fp32 inputs.
template <class R>
static GaussianBack gaussian_backward(const R* params, int64_t ld, int64_t i, const R* Vr, const Cam<R>& camr,
                                      const ScreenGrad& s, const Proj<R>& pr) {
    GaussianBack out{};
    double p[MAXP], V[12];
    for (int k = 0; k < n_rows(camr.sh); ++k) p[k] = double(params[k * ld + i]);
    for (int k = 0; k < 12; ++k) V[k] = double(Vr[k]);
    const double fx = double(camr.fx), fy = double(camr.fy);
    double W[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a][b] = V[a * 4 + b];
    double Xc[3];
    for (int a = 0; a < 3; ++a) Xc[a] = W[a][0] * p[0] + W[a][1] * p[1] + W[a][2] * p[2] + V[a * 4 + 3];
    for (int a = 0; a < 3; ++a) out.Xc[a] = Xc[a];
    const double x = Xc[0], y = Xc[1], z = Xc[2];
    const double nq = std::sqrt(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
    const double q[4] = {p[6] / nq, p[7] / nq, p[8] / nq, p[9] / nq};
    double Rm[3][3];
    rot_of(q, Rm);
    double M[3][3], S[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) M[a][k] = Rm[a][k] * p[3 + k];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) S[a][b] = M[a][0] * M[b][0] + M[a][1] * M[b][1] + M[a][2] * M[b][2];
    // J (entry (0,2) typo fixed: reading C3)
    const double J[2][3] = {{fx / z, 0, -fx * x / (z * z)}, {0, fy / z, -fy * y / (z * z)}};
    double E[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) E[a][k] = J[a][0] * W[0][k] + J[a][1] * W[1][k] + J[a][2] * W[2][k];
    double Sp[2][2] = {{0, 0}, {0, 0}};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < 3; ++k)
                for (int l = 0; l < 3; ++l) Sp[a][b] += E[a][k] * S[k][l] * E[b][l];
    Sp[0][0] += double(camr.dil);
    Sp[1][1] += double(camr.dil);
    const double det = Sp[0][0] * Sp[1][1] - Sp[0][1] * Sp[1][0];
    const double Q[2][2] = {{Sp[1][1] / det, -Sp[0][1] / det}, {-Sp[1][0] / det, Sp[0][0] / det}};
    // conic -> Sigma':  dSigma' = -Q Gbar Q   (Gbar symmetric, off-diagonal g_b/2)
    const double Gb[2][2] = {{s.a, 0.5 * s.b}, {0.5 * s.b, s.c}};
    double QG[2][2] = {{0, 0}, {0, 0}}, dSp[2][2] = {{0, 0}, {0, 0}};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < 2; ++k) QG[a][b] += Q[a][k] * Gb[k][b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < 2; ++k) dSp[a][b] -= QG[a][k] * Q[k][b];
    // Sigma' = E Sigma E^T:  dSigma = E^T dSp E ;  dE = 2 dSp E Sigma  (Eq. S5 blocks)
    double dS[3][3], dE[2][3];
    for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) {
            double acc = 0;
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) acc += E[a][k] * dSp[a][b] * E[b][l];
            dS[k][l] = acc;
        }
    for (int a = 0; a < 2; ++a)
        for (int l = 0; l < 3; ++l) {
            double acc = 0;
            for (int b = 0; b < 2; ++b)
                for (int k = 0; k < 3; ++k) acc += dSp[a][b] * E[b][k] * S[k][l];
            dE[a][l] = 2 * acc;
        }
    // E = J W:  dJ = dE W^T ; dW = J^T dE
    double dJ[2][3];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) dJ[a][b] = dE[a][0] * W[b][0] + dE[a][1] * W[b][1] + dE[a][2] * W[b][2];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) out.dW[a][b] = J[0][a] * dE[0][b] + J[1][a] * dE[1][b];
    // J path to X^c
    const double z2 = z * z, z3 = z2 * z;
    const double dXcJ[3] = {dJ[0][2] * (-fx / z2), dJ[1][2] * (-fy / z2),
                            dJ[0][0] * (-fx / z2) + dJ[0][2] * (2 * fx * x / z3) + dJ[1][1] * (-fy / z2) +
                                dJ[1][2] * (2 * fy * y / z3)};
    // mean path (dm/dX^c = J) and depth path (d = z^c)
    const double dXcm[3] = {J[0][0] * s.mx, J[1][1] * s.my, J[0][2] * s.mx + J[1][2] * s.my + s.d};
    for (int a = 0; a < 3; ++a) {
        out.dXc_noJ[a] = dXcm[a];
        out.dXc_full[a] = dXcm[a] + dXcJ[a];
    }
    // mean: dL/dX = W^T dL/dX^c
    for (int k = 0; k < 3; ++k)
        out.grad[k] = W[0][k] * out.dXc_full[0] + W[1][k] * out.dXc_full[1] + W[2][k] * out.dXc_full[2];
    // Sigma = M M^T: dM = 2 dS M ; ds_k = sum_a dM_ak R_ak ; dR_ak = dM_ak s_k
    double dM[3][3], dRm[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) dM[a][k] = 2 * (dS[a][0] * M[0][k] + dS[a][1] * M[1][k] + dS[a][2] * M[2][k]);
    for (int k = 0; k < 3; ++k) out.grad[3 + k] = dM[0][k] * Rm[0][k] + dM[1][k] * Rm[1][k] + dM[2][k] * Rm[2][k];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) dRm[a][k] = dM[a][k] * p[3 + k];
    double dR[3][3][4], dqh[4] = {0, 0, 0, 0};
    dR_dq(q, dR);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int m = 0; m < 4; ++m) dqh[m] += dRm[a][b] * dR[a][b][m];
    // q_hat = q/|q| (reading C19): dq = (I - q_hat q_hat^T) dq_hat / |q|
    const double dot = dqh[0] * q[0] + dqh[1] * q[1] + dqh[2] * q[2] + dqh[3] * q[3];
    for (int m = 0; m < 4; ++m) out.grad[6 + m] = (dqh[m] - q[m] * dot) / nq;
    out.grad[10] = s.o;
    if (camr.sh == 1) {
        // colour = SH_C0 Y0 + SH_C1 (-u_y Y1 + u_z Y2 - u_x Y3) + 1/2 per channel, clamped at 0 (C29);
        // u = (X - c) / |X - c|, c = -W^T t. The clamp decisions are the projection's (pr.lit).
        double cw[3];
        for (int k = 0; k < 3; ++k) cw[k] = -(W[0][k] * V[3] + W[1][k] * V[7] + W[2][k] * V[11]);
        const double d[3] = {p[0] - cw[0], p[1] - cw[1], p[2] - cw[2]};
        const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const double u[3] = {d[0] / len, d[1] / len, d[2] / len};
        const double gc[3] = {pr.lit[0] ? s.r : 0.0, pr.lit[1] ? s.g : 0.0, pr.lit[2] ? s.bl : 0.0};
        const double basis[4] = {SH_C0, -SH_C1 * u[1], SH_C1 * u[2], -SH_C1 * u[0]};
        double du[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c) {
            for (int k = 0; k < 4; ++k) out.grad[11 + 3 * k + c] = gc[c] * basis[k];
            du[0] += gc[c] * (-SH_C1 * p[20 + c]);
            du[1] += gc[c] * (-SH_C1 * p[14 + c]);
            du[2] += gc[c] * (SH_C1 * p[17 + c]);
        }
        // u = d / |d|:  dL/dd = (dL/du - u (u . dL/du)) / |d|
        const double ud = u[0] * du[0] + u[1] * du[1] + u[2] * du[2];
        for (int k = 0; k < 3; ++k) {
            out.gdir[k] = (du[k] - u[k] * ud) / len;
            out.grad[k] += out.gdir[k];
        }
    } else {
        out.grad[11] = s.r;
        out.grad[12] = s.g;
        out.grad[13] = s.bl;
    }
    return out;
}

// Magnitude of the per-Gaussian chain (the rounding scale of any fp32 evaluation of it, DESIGN.md
// §4.3): gaussian_backward's steps with every quantity replaced by its absolute value and every sum
// of products by the sum of the products' magnitudes, applied to the screen magnitudes S (the
// backward's sums of per-pixel term magnitudes). An evaluation of the chain in precision u differs
// from the exact one by at most about (steps) u times this value; where the exact gradient cancels
// to 0 (e.g. the rotation gradient of an isotropic Gaussian) the rounding is all that remains.
template <class R>
static void gaussian_chain_scale(const R* params, int64_t ld, int64_t i, const R* Vr, const Cam<R>& camr,
                                 const ScreenGrad& s, const Proj<R>& pr, double* out) {
    double p[MAXP], V[12];
    const int rows = n_rows(camr.sh);
    for (int k = 0; k < rows; ++k) p[k] = double(params[k * ld + i]);
    for (int k = 0; k < 12; ++k) V[k] = double(Vr[k]);
    const double fx = std::fabs(double(camr.fx)), fy = std::fabs(double(camr.fy));
    double W[3][3], aW[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) {
            W[a][b] = V[a * 4 + b];
            aW[a][b] = std::fabs(W[a][b]);
        }
    double Xc[3];
    for (int a = 0; a < 3; ++a) Xc[a] = W[a][0] * p[0] + W[a][1] * p[1] + W[a][2] * p[2] + V[a * 4 + 3];
    const double x = std::fabs(Xc[0]), y = std::fabs(Xc[1]), z = std::fabs(Xc[2]);
    const double nq = std::sqrt(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
    const double q[4] = {p[6] / nq, p[7] / nq, p[8] / nq, p[9] / nq};
    double Rm[3][3];
    rot_of(q, Rm);
    double aR[3][3], aM[3][3], aS[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) {
            aR[a][k] = std::fabs(Rm[a][k]);
            aM[a][k] = aR[a][k] * std::fabs(p[3 + k]);
        }
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) aS[a][b] = aM[a][0] * aM[b][0] + aM[a][1] * aM[b][1] + aM[a][2] * aM[b][2];
    const double aJ[2][3] = {{fx / z, 0, fx * x / (z * z)}, {0, fy / z, fy * y / (z * z)}};
    double aE[2][3];
    for (int a = 0; a < 2; ++a)
        for (int k = 0; k < 3; ++k) aE[a][k] = aJ[a][0] * aW[0][k] + aJ[a][1] * aW[1][k] + aJ[a][2] * aW[2][k];
    const double aQ[2][2] = {{std::fabs(double(pr.ca)), std::fabs(double(pr.cb))},
                             {std::fabs(double(pr.cb)), std::fabs(double(pr.cc))}};
    const double aG[2][2] = {{s.a, 0.5 * s.b}, {0.5 * s.b, s.c}};
    double aQG[2][2] = {{0, 0}, {0, 0}}, adSp[2][2] = {{0, 0}, {0, 0}};
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < 2; ++k) aQG[a][b] += aQ[a][k] * aG[k][b];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 2; ++b)
            for (int k = 0; k < 2; ++k) adSp[a][b] += aQG[a][k] * aQ[k][b];
    double adS[3][3], adE[2][3];
    for (int k = 0; k < 3; ++k)
        for (int l = 0; l < 3; ++l) {
            double acc = 0;
            for (int a = 0; a < 2; ++a)
                for (int b = 0; b < 2; ++b) acc += aE[a][k] * adSp[a][b] * aE[b][l];
            adS[k][l] = acc;
        }
    for (int a = 0; a < 2; ++a)
        for (int l = 0; l < 3; ++l) {
            double acc = 0;
            for (int b = 0; b < 2; ++b)
                for (int k = 0; k < 3; ++k) acc += adSp[a][b] * aE[b][k] * aS[k][l];
            adE[a][l] = 2 * acc;
        }
    double adJ[2][3];
    for (int a = 0; a < 2; ++a)
        for (int b = 0; b < 3; ++b) adJ[a][b] = adE[a][0] * aW[b][0] + adE[a][1] * aW[b][1] + adE[a][2] * aW[b][2];
    const double z2 = z * z, z3 = z2 * z;
    const double adXcJ[3] = {adJ[0][2] * fx / z2, adJ[1][2] * fy / z2,
                             adJ[0][0] * fx / z2 + adJ[0][2] * 2 * fx * x / z3 + adJ[1][1] * fy / z2 +
                                 adJ[1][2] * 2 * fy * y / z3};
    const double adXcm[3] = {aJ[0][0] * s.mx, aJ[1][1] * s.my, aJ[0][2] * s.mx + aJ[1][2] * s.my + s.d};
    double adXc[3];
    for (int a = 0; a < 3; ++a) adXc[a] = adXcm[a] + adXcJ[a];
    for (int k = 0; k < 3; ++k) out[k] = aW[0][k] * adXc[0] + aW[1][k] * adXc[1] + aW[2][k] * adXc[2];
    double adM[3][3], adRm[3][3];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) adM[a][k] = 2 * (adS[a][0] * aM[0][k] + adS[a][1] * aM[1][k] + adS[a][2] * aM[2][k]);
    for (int k = 0; k < 3; ++k) out[3 + k] = adM[0][k] * aR[0][k] + adM[1][k] * aR[1][k] + adM[2][k] * aR[2][k];
    for (int a = 0; a < 3; ++a)
        for (int k = 0; k < 3; ++k) adRm[a][k] = adM[a][k] * std::fabs(p[3 + k]);
    double dR[3][3][4], adqh[4] = {0, 0, 0, 0};
    dR_dq(q, dR);
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b)
            for (int m = 0; m < 4; ++m) adqh[m] += adRm[a][b] * std::fabs(dR[a][b][m]);
    double adot = 0;
    for (int m = 0; m < 4; ++m) adot += adqh[m] * std::fabs(q[m]);
    for (int m = 0; m < 4; ++m) out[6 + m] = (adqh[m] + std::fabs(q[m]) * adot) / nq;
    out[10] = s.o;
    if (camr.sh == 1) {
        double cw[3];
        for (int k = 0; k < 3; ++k) cw[k] = -(W[0][k] * V[3] + W[1][k] * V[7] + W[2][k] * V[11]);
        const double d[3] = {p[0] - cw[0], p[1] - cw[1], p[2] - cw[2]};
        const double len = std::sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]);
        const double au[3] = {std::fabs(d[0] / len), std::fabs(d[1] / len), std::fabs(d[2] / len)};
        const double gc[3] = {pr.lit[0] ? s.r : 0.0, pr.lit[1] ? s.g : 0.0, pr.lit[2] ? s.bl : 0.0};
        const double basis[4] = {SH_C0, SH_C1 * au[1], SH_C1 * au[2], SH_C1 * au[0]};
        double adu[3] = {0, 0, 0};
        for (int c = 0; c < 3; ++c) {
            for (int k = 0; k < 4; ++k) out[11 + 3 * k + c] = gc[c] * basis[k];
            adu[0] += gc[c] * SH_C1 * std::fabs(p[20 + c]);
            adu[1] += gc[c] * SH_C1 * std::fabs(p[14 + c]);
            adu[2] += gc[c] * SH_C1 * std::fabs(p[17 + c]);
        }
        const double aud = au[0] * adu[0] + au[1] * adu[1] + au[2] * adu[2];
        for (int k = 0; k < 3; ++k) out[k] += (adu[k] + au[k] * aud) / len;
    } else {
        out[11] = s.r;
        out[12] = s.g;
        out[13] = s.bl;
    }
}

// Error-bound scale of every gradient (parity tolerance): the sums over pixels of
// the magnitudes of the per-pixel terms, S_j = sum_p |c_pj| for the 10 screen quantities j
// (backward_pixel with `sa`), carried through the per-Gaussian chain, which is linear in the screen
// gradient: bound_k = sum_j |d grad_k / d s_j| S_j, i.e. the chain of S_j e_j for each j separately,
// in absolute value. Same for the pose twist, with and without the covariance path. A result summed
// in another order and precision p from the same terms differs from the exact sum by at most about
// (number of terms) p bound_k; a dropped term, a wrong sign or a transposed operand moves a gradient
// by the size of its terms, O(bound_k), so a tolerance of 2e-3 bound_k keeps the comparison's power.
template <class R>
static void error_bound(const R* params, int64_t n, int64_t ld, const R* view, const Cam<R>& cam,
                        const std::vector<Proj<R>>& pj, const std::vector<ScreenGrad>& sabs, double* grad_bound,
                        double* pose_bound, double* pose_bound_paper, double* chain_scale) {
    const int rows = n_rows(cam.sh);
    double W[3][3];
    for (int a = 0; a < 3; ++a)
        for (int b = 0; b < 3; ++b) W[a][b] = double(view[a * 4 + b]);
    double pb[6] = {0, 0, 0, 0, 0, 0}, pbp[6] = {0, 0, 0, 0, 0, 0};
#pragma omp parallel
    {
        double lpb[6] = {0, 0, 0, 0, 0, 0}, lpbp[6] = {0, 0, 0, 0, 0, 0};
#pragma omp for schedule(dynamic, 256)
        for (int64_t i = 0; i < n; ++i) {
            if (!pj[size_t(i)].in_front || pj[size_t(i)].tiles == 0) continue;
            const ScreenGrad& m = sabs[size_t(i)];
            if (chain_scale) {
                double cs[MAXP];
                gaussian_chain_scale<R>(params, ld, i, view, cam, m, pj[size_t(i)], cs);
                for (int k = 0; k < rows; ++k) chain_scale[k * n + i] = cs[k];
            }
            const double v10[10] = {m.mx, m.my, m.a, m.b, m.c, m.o, m.r, m.g, m.bl, m.d};
            for (int j = 0; j < 10; ++j) {
                if (v10[j] == 0) continue;
                double e[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
                e[j] = v10[j];
                const ScreenGrad ej{e[0], e[1], e[2], e[3], e[4], e[5], e[6], e[7], e[8], e[9]};
                const GaussianBack gb = gaussian_backward<R>(params, ld, i, view, cam, ej, pj[size_t(i)]);
                if (grad_bound)
                    for (int k = 0; k < rows; ++k) grad_bound[k * n + i] += std::fabs(gb.grad[k]);
                const double* X = gb.Xc;
                const double* g = gb.dXc_full;
                const double* gp = gb.dXc_noJ;
                double A[3][3];   // this Gaussian's share of A = W (sum_i dW_i)^T
                for (int a = 0; a < 3; ++a)
                    for (int b = 0; b < 3; ++b)
                        A[a][b] = W[a][0] * gb.dW[b][0] + W[a][1] * gb.dW[b][1] + W[a][2] * gb.dW[b][2];
                double WG[3];
                for (int a = 0; a < 3; ++a)
                    WG[a] = W[a][0] * gb.gdir[0] + W[a][1] * gb.gdir[1] + W[a][2] * gb.gdir[2];
                const double tw[6] = {g[0] + WG[0], g[1] + WG[1], g[2] + WG[2],
                                      X[1] * g[2] - X[2] * g[1] + (A[1][2] - A[2][1]),
                                      X[2] * g[0] - X[0] * g[2] + (A[2][0] - A[0][2]),
                                      X[0] * g[1] - X[1] * g[0] + (A[0][1] - A[1][0])};
                const double twp[6] = {gp[0], gp[1], gp[2], X[1] * gp[2] - X[2] * gp[1],
                                       X[2] * gp[0] - X[0] * gp[2], X[0] * gp[1] - X[1] * gp[0]};
                for (int k = 0; k < 6; ++k) {
                    lpb[k] += std::fabs(tw[k]);
                    lpbp[k] += std::fabs(twp[k]);
                }
            }
        }
#pragma omp critical
        for (int k = 0; k < 6; ++k) {
            pb[k] += lpb[k];
            pbp[k] += lpbp[k];
        }
    }
    for (int k = 0; k < 6; ++k) {
        if (pose_bound) pose_bound[k] = pb[k];
        if (pose_bound_paper) pose_bound_paper[k] = pbp[k];
    }
}

}  // namespace

// ============================================================================================
// C ABI of the oracle (ctypes). All arrays are host pointers; SoA rows with leading dim ld.
// ============================================================================================
extern "C" {

int oracle_num_threads() {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void oracle_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

#define ORACLE_PROJECT(SUF, R)                                                                             \
    int oracle_project_##SUF(const R* params, int64_t n, int64_t ld, const R* view, const OracleCam* oc,    \
                             R* mean2d, R* conic, R* depth, int32_t* radius, int32_t* rect,                \
                             uint32_t* tiles, uint32_t* depth_bits, R* cov2d, int32_t mode, R* rgb) { \
        Cam<R> cam(*oc, mode);                                                                        \
        auto pj = project_all<R>(params, n, ld, view, cam);                                                \
        for (int64_t i = 0; i < n; ++i) {                                                                  \
            const Proj<R>& g = pj[size_t(i)];                                                              \
            const bool on = g.in_front;                                                                    \
            mean2d[i] = on ? g.mx : R(0); mean2d[n + i] = on ? g.my : R(0);                                \
            conic[i] = on ? g.ca : R(0); conic[n + i] = on ? g.cb : R(0); conic[2 * n + i] = on ? g.cc : R(0); \
            if (cov2d) { cov2d[i] = g.A; cov2d[n + i] = g.B; cov2d[2 * n + i] = g.C; }                   \
            depth[i] = g.zc;                                                                               \
            radius[i] = on ? g.radius : 0;                                                                 \
            rect[i] = g.xlo; rect[n + i] = g.xhi; rect[2 * n + i] = g.ylo; rect[3 * n + i] = g.yhi;        \
            tiles[i] = on ? g.tiles : 0u;                                                                  \
            depth_bits[i] = bits_of<R>(g.zc);                                                              \
            if (rgb) for (int c = 0; c < 3; ++c) rgb[c * n + i] = g.rgb[c];                                \
        }                                                                                                  \
        return 0;                                                                                          \
    }
ORACLE_PROJECT(f32, float)
ORACLE_PROJECT(f64, double)

// O2: binning + sort (integer, bit-exact). Keys emitted in Gaussian-index order, rect rows then
// columns; key = (tile << 32) | depth_bits; stable sort on the key (= sort by (key, index)).
// Returns K (the number of keys); writes at most `cap` entries. ranges: [tiles][2] (start, end).
int64_t oracle_bin(const uint32_t* depth_bits, const int32_t* rect, const uint32_t* tiles, int64_t n, int32_t GX,
                   int32_t GY, uint64_t* keys, uint32_t* vals, uint32_t* ranges, int64_t cap) {
    int64_t K = 0;
    for (int64_t i = 0; i < n; ++i) K += tiles[i];
    if (K > cap) return K;
    std::vector<uint64_t> k(static_cast<size_t>(K));
    std::vector<uint32_t> v(static_cast<size_t>(K));
    int64_t o = 0;
    for (int64_t i = 0; i < n; ++i) {
        if (tiles[i] == 0) continue;
        for (int32_t ty = rect[2 * n + i]; ty < rect[3 * n + i]; ++ty)
            for (int32_t tx = rect[i]; tx < rect[n + i]; ++tx) {
                k[size_t(o)] = (uint64_t(uint32_t(ty * GX + tx)) << 32) | uint64_t(depth_bits[i]);
                v[size_t(o)] = uint32_t(i);
                ++o;
            }
    }
    std::vector<int64_t> perm(static_cast<size_t>(K));
    std::iota(perm.begin(), perm.end(), 0);
    std::stable_sort(perm.begin(), perm.end(), [&](int64_t a, int64_t b) { return k[size_t(a)] < k[size_t(b)]; });
    for (int64_t j = 0; j < K; ++j) {
        if (keys) keys[j] = k[size_t(perm[size_t(j)])];
        vals[j] = v[size_t(perm[size_t(j)])];
    }
    const int64_t T = int64_t(GX) * GY;
    for (int64_t t = 0; t < T; ++t) {
        const uint64_t lo = uint64_t(t) << 32, hi = uint64_t(t + 1) << 32;
        // equal_range on key >> 32 == t
        int64_t s = 0, e = K;
        {
            int64_t a = 0, b = K;
            while (a < b) { int64_t m = (a + b) / 2; if (k[size_t(perm[size_t(m)])] < lo) a = m + 1; else b = m; }
            s = a;
            a = s; b = K;
            while (a < b) { int64_t m = (a + b) / 2; if (k[size_t(perm[size_t(m)])] < hi) a = m + 1; else b = m; }
            e = a;
        }
        ranges[2 * t] = s == e ? 0u : uint32_t(s);
        ranges[2 * t + 1] = s == e ? 0u : uint32_t(e);
    }
    return K;
}

// O3 forward. pixels: optional list of linear pixel ids (v*W+u); when NULL all pixels are
// rendered and the outputs are full images [3][H][W] / [H][W]; otherwise outputs are per listed
// pixel ([3][n_pix] / [n_pix]). replay_nlast: optional per-output n_last to replay (tie rule).
#define ORACLE_FORWARD(SUF, R)                                                                            \
    int oracle_forward_##SUF(const R* params, int64_t n, int64_t ld, const R* view, const OracleCam* oc,  \
                             const int64_t* pixels, int64_t n_pix, const uint32_t* replay_nlast,          \
                             double* color, double* depth, double* alpha, uint32_t* n_last,               \
                             uint32_t* examined, uint8_t* ambiguous, uint64_t* hash,                      \
                             double* accum_weight, int32_t flip_skip_ties, int32_t mode) {                \
        Cam<R> cam(*oc, mode);                                                                       \
        auto pj = project_all<R>(params, n, ld, view, cam);                                               \
        auto order = depth_order(pj);                                                                     \
        const int64_t P = pixels ? n_pix : int64_t(cam.W) * cam.H;                                        \
        uint64_t h = 0;                                                                                   \
        _Pragma("omp parallel for schedule(dynamic, 64) reduction(^ : h)")                               \
        for (int64_t q = 0; q < P; ++q) {                                                                 \
            const int64_t pid = pixels ? pixels[q] : q;                                                   \
            const int u = int(pid % cam.W), v = int(pid / cam.W);                                         \
            PixelResult r;                                                                                \
            blend_pixel<R>(u, v, pj, order, params, ld, cam, replay_nlast ? int64_t(replay_nlast[q]) : -1, \
                           accum_weight != nullptr, r, flip_skip_ties != 0);                              \
            if (accum_weight) { /* Eq. 12 reading C24: per-Gaussian sum of alpha_i T_i */                 \
                double Tk = 1.0;                                                                          \
                for (const Contrib& ct : r.list) { atomic_add(accum_weight[ct.i], ct.alpha * Tk); Tk *= 1.0 - ct.alpha; } \
            }                                                                                             \
            for (int c = 0; c < 3; ++c) color[c * P + q] = r.color[c];                                    \
            depth[q] = r.depth; alpha[q] = 1.0 - r.T;                                                     \
            n_last[q] = r.n_last; examined[q] = r.examined;                                               \
            if (ambiguous) ambiguous[q] = r.ambiguous;                                                    \
            uint64_t hp = r.hash; fnv(hp, uint64_t(pid)); h ^= hp;                                        \
        }                                                                                                 \
        if (hash) {                                                                                       \
            for (int64_t i = 0; i < n; ++i) {                                                             \
                const Proj<R>& g = pj[size_t(i)];                                                         \
                fnv(h, uint64_t(uint32_t(g.xlo)) | (uint64_t(uint32_t(g.xhi)) << 16) |                   \
                           (uint64_t(uint32_t(g.ylo)) << 32) | (uint64_t(uint32_t(g.yhi)) << 48));        \
            }                                                                                             \
            *hash = h;                                                                                    \
        }                                                                                                 \
        return 0;                                                                                         \
    }
ORACLE_FORWARD(f32, float)
ORACLE_FORWARD(f64, double)

// O4 backward for the whole image with upstream dL/dC [3][H][W], dL/dD [H][W].
// Outputs (all fp64, may be NULL): grad_params [14][n] (+=), grad_screen [10][n]
// (error-bound scales, see error_bound: grad_bound [rows][n], pose_bound[6], pose_bound_paper[6],
// screen_bound [10][n] = S_j, the sums of the per-pixel terms' magnitudes; all =)
// (mx,my,a,b,c,o,r,g,b,d) (=), pose_twist[6] (rho, phi) with the covariance path,
// pose_twist_paper[6] without it, pose_qt[7] = dL/d(q_r,q_i,q_j,q_k, t_x,t_y,t_z) of the
// world->camera pose through Eq. S1/S3 (the second, independent pose path), computed with the
// covariance path iff qt_cov != 0. replay_nlast as in oracle_forward ([H*W] or NULL).
#define ORACLE_BACKWARD(SUF, R)                                                                                \
    int oracle_backward_##SUF(const R* params, int64_t n, int64_t ld, const R* view, const OracleCam* oc,      \
                              const float* dLdC, const float* dLdD, const uint32_t* replay_nlast,              \
                              double* grad_params, double* grad_screen, double* pose_twist,                    \
                              double* pose_twist_paper, double* pose_qt, int32_t qt_cov,                       \
                              const int64_t* pixels, int64_t n_pix, int32_t mode, double* grad_bound,          \
                              double* pose_bound, double* pose_bound_paper, double* screen_bound,              \
                              double* chain_scale) {                                                           \
        Cam<R> cam(*oc, mode);                                                                            \
        auto pj = project_all<R>(params, n, ld, view, cam);                                                    \
        auto order = depth_order(pj);                                                                          \
        const int64_t P = int64_t(cam.W) * cam.H;                                                              \
        const int64_t NQ = pixels ? n_pix : P; /* optional pixel subset (bounded CPU-baseline sample) */       \
        std::vector<ScreenGrad> sg(size_t(n), ScreenGrad{0, 0, 0, 0, 0, 0, 0, 0, 0, 0});                       \
        const bool want_bound = grad_bound || pose_bound || pose_bound_paper || screen_bound || chain_scale;   \
        std::vector<ScreenGrad> sabs(want_bound ? size_t(n) : 0, ScreenGrad{0, 0, 0, 0, 0, 0, 0, 0, 0, 0});   \
        _Pragma("omp parallel for schedule(dynamic, 64)")                                                     \
        for (int64_t qi = 0; qi < NQ; ++qi) {                                                                  \
            const int64_t q = pixels ? pixels[qi] : qi;                                                        \
            const int u = int(q % cam.W), v = int(q / cam.W);                                                  \
            PixelResult r;                                                                                     \
            blend_pixel<R>(u, v, pj, order, params, ld, cam, replay_nlast ? int64_t(replay_nlast[q]) : -1,     \
                           true, r);                                                                           \
            const double dc[3] = {double(dLdC[q]), double(dLdC[P + q]), double(dLdC[2 * P + q])};             \
            backward_pixel<R>(r, pj, params, ld, cam, dc, double(dLdD[q]), sg, want_bound ? &sabs : nullptr);  \
        }                                                                                                      \
        if (want_bound) error_bound<R>(params, n, ld, view, cam, pj, sabs, grad_bound, pose_bound, pose_bound_paper, \
                                       chain_scale);                                                           \
        if (screen_bound) for (int64_t i = 0; i < n; ++i) {                                                    \
            const ScreenGrad& m = sabs[size_t(i)];                                                             \
            const double v10[10] = {m.mx, m.my, m.a, m.b, m.c, m.o, m.r, m.g, m.bl, m.d};                      \
            for (int k = 0; k < 10; ++k) screen_bound[k * n + i] = v10[k];                                     \
        }                                                                                                      \
        double rho[3] = {0, 0, 0}, phi[3] = {0, 0, 0}, rho_p[3] = {0, 0, 0}, phi_p[3] = {0, 0, 0};            \
        double A[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};                                                    \
        double dRpose[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};                                               \
        double dWsum[3][3] = {{0, 0, 0}, {0, 0, 0}, {0, 0, 0}};                                                \
        double dqS3[4] = {0, 0, 0, 0};                                                                         \
        double Gdir[3] = {0, 0, 0};                                                                            \
        double qp[4];                                                                                          \
        {   /* pose quaternion of W (for the Eq. S3 path): robust matrix -> quaternion */                     \
            double W[3][3];                                                                                    \
            for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) W[a][b] = double(view[a * 4 + b]);        \
            const double tr = W[0][0] + W[1][1] + W[2][2];                                                     \
            if (tr > 0) { double s = std::sqrt(tr + 1.0) * 2; qp[0] = 0.25 * s; qp[1] = (W[2][1] - W[1][2]) / s; \
                          qp[2] = (W[0][2] - W[2][0]) / s; qp[3] = (W[1][0] - W[0][1]) / s; }                  \
            else if (W[0][0] > W[1][1] && W[0][0] > W[2][2]) { double s = std::sqrt(1.0 + W[0][0] - W[1][1] - W[2][2]) * 2; \
                          qp[0] = (W[2][1] - W[1][2]) / s; qp[1] = 0.25 * s; qp[2] = (W[0][1] + W[1][0]) / s;  \
                          qp[3] = (W[0][2] + W[2][0]) / s; }                                                   \
            else if (W[1][1] > W[2][2]) { double s = std::sqrt(1.0 + W[1][1] - W[0][0] - W[2][2]) * 2;         \
                          qp[0] = (W[0][2] - W[2][0]) / s; qp[1] = (W[0][1] + W[1][0]) / s; qp[2] = 0.25 * s;  \
                          qp[3] = (W[1][2] + W[2][1]) / s; }                                                   \
            else { double s = std::sqrt(1.0 + W[2][2] - W[0][0] - W[1][1]) * 2;                                \
                          qp[0] = (W[1][0] - W[0][1]) / s; qp[1] = (W[0][2] + W[2][0]) / s;                    \
                          qp[2] = (W[1][2] + W[2][1]) / s; qp[3] = 0.25 * s; }                                 \
        }                                                                                                      \
        for (int64_t i = 0; i < n; ++i) {                                                                      \
            if (!pj[size_t(i)].in_front || pj[size_t(i)].tiles == 0) continue;                                 \
            GaussianBack gb = gaussian_backward<R>(params, ld, i, view, cam, sg[size_t(i)], pj[size_t(i)]);    \
            if (grad_params) for (int k = 0; k < n_rows(cam.sh); ++k) grad_params[k * n + i] += gb.grad[k];    \
            for (int a = 0; a < 3; ++a) Gdir[a] += gb.gdir[a];   /* SH view-direction path (C29) */          \
            const double* X = gb.Xc;                                                                           \
            for (int a = 0; a < 3; ++a) { rho[a] += gb.dXc_full[a]; rho_p[a] += gb.dXc_noJ[a]; }               \
            const double* g = gb.dXc_full; const double* gp = gb.dXc_noJ;                                      \
            phi[0] += X[1] * g[2] - X[2] * g[1]; phi[1] += X[2] * g[0] - X[0] * g[2]; phi[2] += X[0] * g[1] - X[1] * g[0]; \
            phi_p[0] += X[1] * gp[2] - X[2] * gp[1]; phi_p[1] += X[2] * gp[0] - X[0] * gp[2];                  \
            phi_p[2] += X[0] * gp[1] - X[1] * gp[0];                                                           \
            for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) dWsum[a][b] += gb.dW[a][b];                \
            /* Eq. S3 path: X (world) and dL/dX^c; S3 gives dX^c/dq for X^c = R(q) X + t */                   \
            const double xw = double(params[i]), yw = double(params[ld + i]), zw = double(params[2 * ld + i]); \
            const double* gq = qt_cov ? gb.dXc_full : gb.dXc_noJ;                                              \
            const double r_ = qp[0], i_ = qp[1], j_ = qp[2], k_ = qp[3];                                       \
            /* Eq. S3, row 3 of dX^c/dq_i with the sign typo fixed (reading C4) */                \
            const double S3[4][3] = {                                                                          \
                {2 * (-k_ * yw + j_ * zw), 2 * (k_ * xw - i_ * zw), 2 * (-j_ * xw + i_ * yw)},                 \
                {2 * (j_ * yw + k_ * zw), 2 * (j_ * xw - 2 * i_ * yw - r_ * zw), 2 * (k_ * xw + r_ * yw - 2 * i_ * zw)}, \
                {2 * (-2 * j_ * xw + i_ * yw + r_ * zw), 2 * (i_ * xw + k_ * zw), 2 * (-r_ * xw + k_ * yw - 2 * j_ * zw)}, \
                {2 * (-2 * k_ * xw - r_ * yw + i_ * zw), 2 * (r_ * xw - 2 * k_ * yw + j_ * zw), 2 * (i_ * xw + j_ * yw)}}; \
            for (int m = 0; m < 4; ++m) dqS3[m] += S3[m][0] * gq[0] + S3[m][1] * gq[1] + S3[m][2] * gq[2];      \
            (void)dRpose;                                                                                      \
            if (grad_screen) {                                                                                 \
                const ScreenGrad& s = sg[size_t(i)];                                                           \
                const double v10[10] = {s.mx, s.my, s.a, s.b, s.c, s.o, s.r, s.g, s.bl, s.d};                  \
                for (int k = 0; k < 10; ++k) grad_screen[k * n + i] = v10[k];                                  \
            }                                                                                                  \
        }                                                                                                      \
        double W[3][3];                                                                                        \
        for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) W[a][b] = double(view[a * 4 + b]);            \
        for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b)                                                \
            A[a][b] = W[a][0] * dWsum[b][0] + W[a][1] * dWsum[b][1] + W[a][2] * dWsum[b][2];                   \
        /* SH colour through the camera centre c = -W^T t (C29): dL/dc = -Gdir, so the twist gains        \
           rho += W Gdir and phi gains nothing (first order); the paper's mode drops it (C8) */     \
        double WG[3];                                                                                          \
        for (int a = 0; a < 3; ++a) WG[a] = W[a][0] * Gdir[0] + W[a][1] * Gdir[1] + W[a][2] * Gdir[2];        \
        if (pose_twist) {                                                                                      \
            for (int a = 0; a < 3; ++a) pose_twist[a] = rho[a] + WG[a];                                        \
            pose_twist[3] = phi[0] + (A[1][2] - A[2][1]);                                                      \
            pose_twist[4] = phi[1] + (A[2][0] - A[0][2]);                                                      \
            pose_twist[5] = phi[2] + (A[0][1] - A[1][0]);                                                      \
        }                                                                                                      \
        if (pose_twist_paper) {                                                                                \
            for (int a = 0; a < 3; ++a) { pose_twist_paper[a] = rho_p[a]; pose_twist_paper[3 + a] = phi_p[a]; } \
        }                                                                                                      \
        if (pose_qt) {                                                                                         \
            /* covariance path to q through Eq. S1: dL/dq += sum_ab dW_ab dR_ab/dq */                         \
            double dR[3][3][4];                                                                                \
            dR_dq(qp, dR);                                                                                     \
            for (int m = 0; m < 4; ++m) {                                                                      \
                double acc = dqS3[m];                                                                          \
                if (qt_cov) for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b) acc += dWsum[a][b] * dR[a][b][m]; \
                /* colour path: c_k = -sum_a R_ak t_a, so dL/dR_ak = t_a Gdir_k */                          \
                if (qt_cov) for (int a = 0; a < 3; ++a) for (int b = 0; b < 3; ++b)                           \
                    acc += double(view[a * 4 + 3]) * Gdir[b] * dR[a][b][m];                                    \
                pose_qt[m] = acc;                                                                              \
            }                                                                                                  \
            for (int a = 0; a < 3; ++a) pose_qt[4 + a] = qt_cov ? rho[a] + WG[a] : rho_p[a];                   \
            pose_qt[7] = qp[0]; pose_qt[8] = qp[1]; pose_qt[9] = qp[2]; pose_qt[10] = qp[3];                   \
        }                                                                                                      \
        return 0;                                                                                              \
    }
ORACLE_BACKWARD(f32, float)
ORACLE_BACKWARD(f64, double)

}  // extern "C"
