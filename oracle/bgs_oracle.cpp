// bgs_oracle.cpp -- CPU ORACLE for the BalanceGS (arXiv 2510.14564) hot path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and bench.py's
// cpu_baseline / --impl reference legs may load this library.  It shares no
// code, header, table or constant generator with the CUDA path under
// paper_2510_14564_b200/csrc/, and neither includes nor links the other.
//
// What it computes (citations: P:L = /root/reference/PAPER.md line L; S:L =
// SPEC.md line L; R# = the readings listed in DESIGN.md §3 / SURVEY.md §8(c)):
//   O1  activations s = exp(ls), o = sigmoid(ol), q = q^/|q^|            (R5)
//   O2  camera-space t = V [mu,1]; cull t_z <= near                     (R3)
//   O3  clip = P [mu,1]; ndc = clip/clip.w; pixel = ((ndc+1) W - 1)/2   (R1, R4)
//   O4  Sigma = R S S^T R^T                                             (R6)
//   O5  Sigma' = J W Sigma W^T J^T (+0.3 I)                             (R7, R8)
//   O6  det, conic = Sigma'^-1                                          (R9)
//   O7  radius = ceil(3 sqrt(lambda_1))                                 (R10)
//   O8  16x16 tile rect: the tiles the alpha >= 1/255 level set's
//       conservative box reaches (R11'; R10's square rect: SQUARE_RECT)  (R11)
//   O9  SH degree <= 3 colour                                           (R12)
//   O10 offsets = exclusive scan of tiles_touched                       (R13)
//   O11 (tile | depth) keys, O12 std::stable_sort, O13 tile ranges      (R13)
//   O14 front-to-back alpha blend  C = sum c_i a_i prod_{j<i}(1 - a_j)  (R14-R17)
//   O15 blend backward, O16 preprocess backward (decisions frozen)      (R18)
//   O17 Adam                                                            (R21)
//
// Float path: every decision-bearing quantity follows the canonical expression
// tree of SURVEY.md §8(c) (R22): fma() is a single-rounding fused multiply-add,
// every other op a separately rounded binary32 op.  Build with
// -ffp-contract=off and without -ffast-math.  Gradients are evaluated in
// double with every discrete decision of the float forward frozen (R18), and
// summed over pixels in double (R24).
//
// Pinned by tests/test_oracle_*.py (closed forms, brute force, P:146 evaluated
// literally, orthonormality quadrature, central finite differences, torch Adam).
//
// Threading (SURVEY.md §8(d) "std::thread over all host cores ... fixed-order reductions"):
// OpenMP over independent units only -- Gaussians (preprocess, key emission, chain rule),
// pixel rows (blend forward), sorted chunks (stable sort = chunk std::stable_sort + stable
// std::merge rounds), tiles (blend backward).  The per-unit arithmetic is unchanged, and the
// one cross-unit sum (the blend backward's per-Gaussian sums over pixels) is reduced in a
// fixed order -- per tile, then tiles in index order -- so results do not depend on the
// thread count.  orc_set_threads(k) fixes k (1 = the plain serial program).

#include <omp.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

namespace {

constexpr int TILE = 16;  // "16 x 16 pixel blocks"

// mode bits: switch readings off (the "plain mode" evaluator)
enum : uint32_t {
  ORC_NO_LOWPASS = 1u,       // R8
  ORC_NO_JCLAMP = 2u,        // R7
  ORC_FULL_RECT = 4u,        // R10/R11: every Gaussian covers every tile
  ORC_NO_ALPHA_CLAMP = 8u,   // R14 clamp at 0.99
  ORC_NO_ALPHA_CUTOFF = 16u, // R14 skip alpha < 1/255
  ORC_NO_EARLY_STOP = 32u,   // R15
  ORC_NO_POWER_GUARD = 64u,  // R14 skip power > 0
  ORC_CANON_EXP = 128u,      // R23 parity mode: G from canon_exp instead of std::exp
  ORC_SQUARE_RECT = 256u,    // R10/R11: 3DGS's square rect of half-width radius (else R11')
};

// R23's optional parity mode: a canonical exponential both sides evaluate
// with the same IEEE binary32 operations -- x = power * log2(e); n = floor(x); f = x - n
// (exact); 2^f from the degree-8 Taylor polynomial of e^(f ln 2) in Horner form with fused
// multiply-adds; times 2^n (exact) -- so alpha, and every blend decision, is reproducible
// bit for bit.
float canon_exp(float power) {
  const float x = power * 1.4426950408889634f;
  const float n = std::floor(x);
  const float f = x - n;
  const float c[9] = {1.0f, 6.9314718e-1f, 2.4022651e-1f, 5.5504109e-2f, 9.6181291e-3f, 1.3333558e-3f,
                      1.5403530e-4f, 1.5252734e-5f, 1.3215487e-6f};  // (ln 2)^k / k!
  float p = c[8];
  for (int k = 7; k >= 0; --k) p = std::fma(p, f, c[k]);
  return std::ldexp(p, (int)n);
}

// clamp bits per Gaussian (decisions frozen for the backward, R18)
enum : uint8_t {
  CB_R = 1, CB_G = 2, CB_B = 4,     // rgb clamped below at 0 (R12)
  CB_JX = 8, CB_JX_NEG = 16,        // J clamp active on x (and its side) (R7)
  CB_JY = 32, CB_JY_NEG = 64,
};

// Real SH constants (R12).
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};

}  // namespace

extern "C" {

typedef struct {
  float view[16];    // world -> camera, column-major: t_r = sum_k view[r+4k] mu_k + view[12+r]
  float proj[16];    // world -> clip, column-major
  float campos[3];
  float tan_fovx, tan_fovy;
  int32_t width, height;
  float bg[3];
  float near_plane;
} orc_camera;

}  // extern "C"

namespace {

struct Theta {  // views into theta[59n] (layout: SURVEY §8.0)
  int64_t n;
  const float* f;
  const float* mean(int64_t i) const { return f + 3 * i; }
  const float* lscale(int64_t i) const { return f + 3 * n + 3 * i; }
  const float* quat(int64_t i) const { return f + 6 * n + 4 * i; }
  float ologit(int64_t i) const { return f[10 * n + i]; }
  const float* sh(int64_t i) const { return f + 11 * n + 48 * i; }
};

struct ThetaD {
  int64_t n;
  const double* f;
  const double* mean(int64_t i) const { return f + 3 * i; }
  const double* lscale(int64_t i) const { return f + 3 * n + 3 * i; }
  const double* quat(int64_t i) const { return f + 6 * n + 4 * i; }
  double ologit(int64_t i) const { return f[10 * n + i]; }
  const double* sh(int64_t i) const { return f + 11 * n + 48 * i; }
};

inline uint32_t float_bits(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  return u;
}

// SH basis Y_k(d) and dY_k/dd (d = unit view direction), [3DGS] sign convention (R12).
template <typename S>
void sh_basis(S x, S y, S z, S Y[16], S dY[16][3]) {
  const S c0 = (S)SH_C0, c1 = (S)SH_C1;
  S c2[5], c3[7];
  for (int i = 0; i < 5; ++i) c2[i] = (S)SH_C2[i];
  for (int i = 0; i < 7; ++i) c3[i] = (S)SH_C3[i];
  const S xx = x * x, yy = y * y, zz = z * z;
  Y[0] = c0;
  Y[1] = -c1 * y;
  Y[2] = c1 * z;
  Y[3] = -c1 * x;
  Y[4] = c2[0] * x * y;
  Y[5] = c2[1] * y * z;
  Y[6] = c2[2] * (2 * zz - xx - yy);
  Y[7] = c2[3] * x * z;
  Y[8] = c2[4] * (xx - yy);
  Y[9] = c3[0] * y * (3 * xx - yy);
  Y[10] = c3[1] * x * y * z;
  Y[11] = c3[2] * y * (4 * zz - xx - yy);
  Y[12] = c3[3] * z * (2 * zz - 3 * xx - 3 * yy);
  Y[13] = c3[4] * x * (4 * zz - xx - yy);
  Y[14] = c3[5] * z * (xx - yy);
  Y[15] = c3[6] * x * (xx - 3 * yy);
  if (!dY) return;
  const S zero = 0;
  auto set = [&](int k, S a, S b, S c) { dY[k][0] = a; dY[k][1] = b; dY[k][2] = c; };
  set(0, zero, zero, zero);
  set(1, zero, -c1, zero);
  set(2, zero, zero, c1);
  set(3, -c1, zero, zero);
  set(4, c2[0] * y, c2[0] * x, zero);
  set(5, zero, c2[1] * z, c2[1] * y);
  set(6, -2 * c2[2] * x, -2 * c2[2] * y, 4 * c2[2] * z);
  set(7, c2[3] * z, zero, c2[3] * x);
  set(8, 2 * c2[4] * x, -2 * c2[4] * y, zero);
  set(9, 6 * c3[0] * x * y, c3[0] * (3 * xx - 3 * yy), zero);
  set(10, c3[1] * y * z, c3[1] * x * z, c3[1] * x * y);
  set(11, -2 * c3[2] * x * y, c3[2] * (4 * zz - xx - 3 * yy), 8 * c3[2] * y * z);
  set(12, -6 * c3[3] * x * z, -6 * c3[3] * y * z, c3[3] * (6 * zz - 3 * xx - 3 * yy));
  set(13, c3[4] * (4 * zz - 3 * xx - yy), -2 * c3[4] * x * y, 8 * c3[4] * x * z);
  set(14, 2 * c3[5] * x * z, -2 * c3[5] * y * z, c3[5] * (xx - yy));
  set(15, c3[6] * (3 * xx - 3 * yy), -6 * c3[6] * x * y, zero);
}

inline int n_coeffs(int deg) { return (deg + 1) * (deg + 1); }

// ---------------------------------------------------------------------------
// O1-O9 in float, canonical expression tree (R22)
// ---------------------------------------------------------------------------
struct PreF {
  bool visible;
  int32_t radius;
  float depth, x, y, conic[3], opacity, rgb[3];
  uint8_t cbits;
  int32_t rect[4];  // x0, y0, x1, y1 (tiles, half-open)
};

PreF preprocess_one(const Theta& th, int64_t i, int deg, const orc_camera& cam, uint32_t mode) {
  PreF p;
  std::memset(&p, 0, sizeof(p));
  const float* V = cam.view;
  const float* P = cam.proj;
  const float mx = th.mean(i)[0], my = th.mean(i)[1], mz = th.mean(i)[2];
  // O2: camera space, near cull (R3)
  float t[3];
  for (int r = 0; r < 3; ++r) t[r] = std::fma(V[8 + r], mz, std::fma(V[4 + r], my, std::fma(V[r], mx, V[12 + r])));
  if (t[2] <= cam.near_plane) return p;
  // O3: clip, perspective divide (R4), pixel coordinates (R1)
  float c[4];
  for (int r = 0; r < 4; ++r) c[r] = std::fma(P[8 + r], mz, std::fma(P[4 + r], my, std::fma(P[r], mx, P[12 + r])));
  const float ndc_x = c[0] / c[3], ndc_y = c[1] / c[3];
  const float px = 0.5f * std::fma(ndc_x + 1.0f, (float)cam.width, -1.0f);
  const float py = 0.5f * std::fma(ndc_y + 1.0f, (float)cam.height, -1.0f);
  // O1: activations (R5): transcendentals in double, rounded once
  float s[3];
  for (int k = 0; k < 3; ++k) s[k] = (float)std::exp((double)th.lscale(i)[k]);
  float qw = th.quat(i)[0], qx = th.quat(i)[1], qy = th.quat(i)[2], qz = th.quat(i)[3];
  const float n2 = std::fma(qw, qw, std::fma(qx, qx, std::fma(qy, qy, qz * qz)));
  const float inv = 1.0f / std::sqrt(n2);
  qw *= inv; qx *= inv; qy *= inv; qz *= inv;
  // O4: Sigma = (R diag s)(R diag s)^T (R6)
  const float xx = qx * qx, yy = qy * qy, zz = qz * qz, xy = qx * qy, xz = qx * qz, yz = qy * qz;
  const float wx = qw * qx, wy = qw * qy, wz = qw * qz;
  float R[3][3];
  R[0][0] = 1.0f - 2.0f * (yy + zz); R[0][1] = 2.0f * (xy - wz);        R[0][2] = 2.0f * (xz + wy);
  R[1][0] = 2.0f * (xy + wz);        R[1][1] = 1.0f - 2.0f * (xx + zz); R[1][2] = 2.0f * (yz - wx);
  R[2][0] = 2.0f * (xz - wy);        R[2][1] = 2.0f * (yz + wx);        R[2][2] = 1.0f - 2.0f * (xx + yy);
  float M[3][3];
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 3; ++k) M[a][k] = R[a][k] * s[k];
  float Sg[3][3];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) Sg[a][b] = std::fma(M[a][2], M[b][2], std::fma(M[a][1], M[b][1], M[a][0] * M[b][0]));
  // O5: J W Sigma W^T J^T + 0.3 I (R7 clamp, R8 low-pass)
  const float fx = (float)cam.width / (2.0f * cam.tan_fovx);
  const float fy = (float)cam.height / (2.0f * cam.tan_fovy);
  const float limx = 1.3f * cam.tan_fovx, limy = 1.3f * cam.tan_fovy;
  float u = t[0] / t[2], v = t[1] / t[2];
  if (!(mode & ORC_NO_JCLAMP)) {
    if (u > limx) p.cbits |= CB_JX;
    if (u < -limx) p.cbits |= CB_JX | CB_JX_NEG;
    if (v > limy) p.cbits |= CB_JY;
    if (v < -limy) p.cbits |= CB_JY | CB_JY_NEG;
    u = std::fmin(limx, std::fmax(-limx, u));
    v = std::fmin(limy, std::fmax(-limy, v));
  }
  const float tpx = u * t[2], tpy = v * t[2];
  const float j00 = fx / t[2], j02 = -(fx * tpx) / (t[2] * t[2]);
  const float j11 = fy / t[2], j12 = -(fy * tpy) / (t[2] * t[2]);
  float T[2][3];
  for (int k = 0; k < 3; ++k) {
    const float W0k = V[0 + 4 * k], W1k = V[1 + 4 * k], W2k = V[2 + 4 * k];
    T[0][k] = std::fma(j02, W2k, j00 * W0k);
    T[1][k] = std::fma(j12, W2k, j11 * W1k);
  }
  float L[2][3];
  for (int a = 0; a < 2; ++a)
    for (int k = 0; k < 3; ++k) L[a][k] = std::fma(T[a][2], Sg[2][k], std::fma(T[a][1], Sg[1][k], T[a][0] * Sg[0][k]));
  const float lp = (mode & ORC_NO_LOWPASS) ? 0.0f : 0.3f;
  const float ca = std::fma(L[0][2], T[0][2], std::fma(L[0][1], T[0][1], L[0][0] * T[0][0])) + lp;
  const float cb = std::fma(L[0][2], T[1][2], std::fma(L[0][1], T[1][1], L[0][0] * T[1][0]));
  const float cc = std::fma(L[1][2], T[1][2], std::fma(L[1][1], T[1][1], L[1][0] * T[1][0])) + lp;
  // O6: det, conic (R9)
  const float det = std::fma(ca, cc, -(cb * cb));
  if (det <= 0.0f) return p;
  const float idet = 1.0f / det;
  const float conic[3] = {cc * idet, -(cb * idet), ca * idet};
  // O7: radius (R10)
  const float mid = 0.5f * (ca + cc);
  const float lam = mid + std::sqrt(std::fmax(0.1f, mid * mid - det));
  const int32_t rad = (int32_t)std::ceil(3.0f * std::sqrt(lam));
  // O1 (opacity): o = sigmoid(ol), the transcendental in double, rounded once (R5)
  const float o = (float)(1.0 / (1.0 + std::exp(-(double)th.ologit(i))));
  // O8: tile rect (R11').  A pixel d away from the centre blends the Gaussian only if
  // o exp(-d^T conic d / 2) >= 1/255 (R14), i.e. d^T Sigma'^-1 d <= 2 tau, tau = ln(255 o):
  // inside the ellipse whose bounding box has half-widths sqrt(2 tau a), sqrt(2 tau c).  The
  // extents e carry margins (tau + 1e-3, x 1.001, + 1e-3 px) for the float error of the
  // blend's own power and alpha, so every pixel outside the box takes alpha < 1/255; the rect
  // is the 16x16 tiles the box reaches (floor then clamp, as R11).  Tiles outside it never
  // blend the Gaussian: the images, final T and every decision are R10's; the lists are
  // shorter, so n_contrib (a list position, R16) is counted in them.  tau in double, rounded
  // once (R5); a Gaussian with tau <= 0 (o < 1/255) blends nowhere and is culled.
  const int tiles_x = (cam.width + TILE - 1) / TILE, tiles_y = (cam.height + TILE - 1) / TILE;
  int32_t rect[4];
  auto clampt = [](float f, int hi) { return (int32_t)std::fmin((float)hi, std::fmax(0.0f, f)); };
  if (mode & ORC_FULL_RECT) {
    rect[0] = 0; rect[1] = 0; rect[2] = tiles_x; rect[3] = tiles_y;
  } else if ((mode & ORC_SQUARE_RECT) || (mode & ORC_NO_ALPHA_CUTOFF)) {  // R10 / R11
    rect[0] = clampt(std::floor((px - (float)rad) * 0.0625f), tiles_x);
    rect[1] = clampt(std::floor((py - (float)rad) * 0.0625f), tiles_y);
    rect[2] = clampt(std::floor((px + (float)(rad + 15)) * 0.0625f), tiles_x);
    rect[3] = clampt(std::floor((py + (float)(rad + 15)) * 0.0625f), tiles_y);
  } else {
    const float tau = (float)std::log((double)(255.0f * o)) + 1e-3f;
    if (!(tau > 0.0f)) return p;
    const float ex = std::sqrt(2.0f * tau * ca) * 1.001f + 1e-3f;
    const float ey = std::sqrt(2.0f * tau * cc) * 1.001f + 1e-3f;
    rect[0] = clampt(std::floor((px - ex) * 0.0625f), tiles_x);
    rect[1] = clampt(std::floor((py - ey) * 0.0625f), tiles_y);
    rect[2] = clampt(std::floor((px + ex) * 0.0625f) + 1.0f, tiles_x);
    rect[3] = clampt(std::floor((py + ey) * 0.0625f) + 1.0f, tiles_y);
  }
  if ((int64_t)(rect[2] - rect[0]) * (rect[3] - rect[1]) == 0) return p;
  // O9: SH colour (R12) -- free evaluation order (float)
  float dir[3] = {mx - cam.campos[0], my - cam.campos[1], mz - cam.campos[2]};
  const float dl = std::sqrt(dir[0] * dir[0] + dir[1] * dir[1] + dir[2] * dir[2]);
  float Y[16];
  sh_basis<float>(dir[0] / dl, dir[1] / dl, dir[2] / dl, Y, nullptr);
  const float* sh = th.sh(i);
  for (int ch = 0; ch < 3; ++ch) {
    float acc = 0.0f;
    for (int k = 0; k < n_coeffs(deg); ++k) acc += Y[k] * sh[3 * k + ch];
    acc += 0.5f;
    if (acc < 0.0f) {
      p.cbits |= (uint8_t)(1u << ch);
      acc = 0.0f;
    }
    p.rgb[ch] = acc;
  }
  p.visible = true;
  p.radius = rad;
  p.depth = t[2];
  p.x = px;
  p.y = py;
  for (int k = 0; k < 3; ++k) p.conic[k] = conic[k];
  p.opacity = o;
  std::memcpy(p.rect, rect, sizeof(rect));
  return p;
}

// ---------------------------------------------------------------------------
// O14 per-pixel walk (float, canonical; R14-R16) with R23 near-tie flags
// ---------------------------------------------------------------------------
struct Gauss2D {  // what the walk reads per list entry
  const float *xy, *conic, *opacity, *rgb;
};

struct WalkOut {
  float C[3];
  float T;
  int32_t last;      // 1-based list position of the last blended Gaussian (R16)
  int32_t walked;    // list entries visited (E_f)
  int32_t blended;   // Gaussians blended (SPEC's per-pixel count, diagnostic)
  bool flagged;      // some decision within delta of its threshold (R23)
};

template <typename F>
WalkOut walk_pixel(const Gauss2D& g, const uint32_t* values, uint32_t start, uint32_t end, float pxf, float pyf,
                   uint32_t mode, double da, double dT, F&& on_blend) {
  WalkOut w;
  w.C[0] = w.C[1] = w.C[2] = 0.0f;
  w.T = 1.0f;
  w.last = 0;
  w.walked = 0;
  w.blended = 0;
  w.flagged = false;
  for (uint32_t pos = start; pos < end; ++pos) {
    const uint32_t id = values[pos];
    ++w.walked;
    const float A = -0.5f * g.conic[3 * id + 0];
    const float B = -g.conic[3 * id + 1];
    const float Cc = -0.5f * g.conic[3 * id + 2];
    const float dx = g.xy[2 * id + 0] - pxf;
    const float dy = g.xy[2 * id + 1] - pyf;
    const float power = std::fma(A, dx * dx, std::fma(Cc, dy * dy, B * (dx * dy)));
    if (!(mode & ORC_NO_POWER_GUARD) && power > 0.0f) continue;
    const float G = (mode & ORC_CANON_EXP) ? canon_exp(power) : std::exp(power);
    const float og = g.opacity[id] * G;
    bool aclamp = false;
    float alpha = og;
    if (!(mode & ORC_NO_ALPHA_CLAMP) && og > 0.99f) {
      alpha = 0.99f;
      aclamp = true;
    }
    if (!(mode & ORC_NO_ALPHA_CUTOFF)) {
      const double ad = (double)g.opacity[id] * std::exp((double)power);
      if (std::fabs(ad - 1.0 / 255.0) <= da * (1.0 / 255.0)) w.flagged = true;
      if (alpha < (1.0f / 255.0f)) continue;
    }
    const float tT = w.T * (1.0f - alpha);
    if (!(mode & ORC_NO_EARLY_STOP)) {
      if (std::fabs((double)tT - 1e-4) <= dT * 1e-4) w.flagged = true;
      if (tT < 1e-4f) break;
    }
    for (int ch = 0; ch < 3; ++ch) w.C[ch] = std::fma(g.rgb[3 * id + ch], alpha * w.T, w.C[ch]);
    w.T = tT;
    w.last = (int32_t)(pos - start + 1);
    ++w.blended;
    on_blend(id, aclamp, pos);
  }
  return w;
}

// ---------------------------------------------------------------------------
// double-precision forward with decisions frozen (R18) -- used by the backward
// and by the finite-difference pin
// ---------------------------------------------------------------------------
struct PreD {
  double s[3], qh[4], qn, q[4], o, R[3][3], M[3][3], Sg[3][3];
  double t[3], u, v, j00, j02, j11, j12, fx, fy, T[2][3], a, b, c, det, conic[3];
  double clip[4], xy[2];
  double dir[3], dl, d[3], Y[16], dY[16][3], rgb[3];
};

void preprocess_double(const ThetaD& th, int64_t i, int deg, const orc_camera& cam, uint32_t mode, uint8_t cbits,
                       PreD& p) {
  double V[16], P[16];
  for (int k = 0; k < 16; ++k) { V[k] = cam.view[k]; P[k] = cam.proj[k]; }
  const double* mu = th.mean(i);
  for (int r = 0; r < 3; ++r) p.t[r] = V[r] * mu[0] + V[4 + r] * mu[1] + V[8 + r] * mu[2] + V[12 + r];
  for (int r = 0; r < 4; ++r) p.clip[r] = P[r] * mu[0] + P[4 + r] * mu[1] + P[8 + r] * mu[2] + P[12 + r];
  p.xy[0] = 0.5 * ((p.clip[0] / p.clip[3] + 1.0) * cam.width - 1.0);
  p.xy[1] = 0.5 * ((p.clip[1] / p.clip[3] + 1.0) * cam.height - 1.0);
  for (int k = 0; k < 3; ++k) p.s[k] = std::exp(th.lscale(i)[k]);
  p.o = 1.0 / (1.0 + std::exp(-th.ologit(i)));
  for (int k = 0; k < 4; ++k) p.qh[k] = th.quat(i)[k];
  p.qn = std::sqrt(p.qh[0] * p.qh[0] + p.qh[1] * p.qh[1] + p.qh[2] * p.qh[2] + p.qh[3] * p.qh[3]);
  for (int k = 0; k < 4; ++k) p.q[k] = p.qh[k] / p.qn;
  const double w = p.q[0], x = p.q[1], y = p.q[2], z = p.q[3];
  p.R[0][0] = 1 - 2 * (y * y + z * z); p.R[0][1] = 2 * (x * y - w * z);     p.R[0][2] = 2 * (x * z + w * y);
  p.R[1][0] = 2 * (x * y + w * z);     p.R[1][1] = 1 - 2 * (x * x + z * z); p.R[1][2] = 2 * (y * z - w * x);
  p.R[2][0] = 2 * (x * z - w * y);     p.R[2][1] = 2 * (y * z + w * x);     p.R[2][2] = 1 - 2 * (x * x + y * y);
  for (int a = 0; a < 3; ++a)
    for (int k = 0; k < 3; ++k) p.M[a][k] = p.R[a][k] * p.s[k];
  for (int a = 0; a < 3; ++a)
    for (int b = 0; b < 3; ++b) {
      double acc = 0;
      for (int k = 0; k < 3; ++k) acc += p.M[a][k] * p.M[b][k];
      p.Sg[a][b] = acc;
    }
  p.fx = cam.width / (2.0 * (double)cam.tan_fovx);
  p.fy = cam.height / (2.0 * (double)cam.tan_fovy);
  const double limx = (double)(1.3f * cam.tan_fovx), limy = (double)(1.3f * cam.tan_fovy);
  p.u = p.t[0] / p.t[2];
  p.v = p.t[1] / p.t[2];
  if (cbits & CB_JX) p.u = (cbits & CB_JX_NEG) ? -limx : limx;
  if (cbits & CB_JY) p.v = (cbits & CB_JY_NEG) ? -limy : limy;
  p.j00 = p.fx / p.t[2];
  p.j02 = -p.fx * p.u / p.t[2];
  p.j11 = p.fy / p.t[2];
  p.j12 = -p.fy * p.v / p.t[2];
  for (int k = 0; k < 3; ++k) {
    p.T[0][k] = p.j00 * V[0 + 4 * k] + p.j02 * V[2 + 4 * k];
    p.T[1][k] = p.j11 * V[1 + 4 * k] + p.j12 * V[2 + 4 * k];
  }
  double TS[2][3];
  for (int a = 0; a < 2; ++a)
    for (int k = 0; k < 3; ++k) TS[a][k] = p.T[a][0] * p.Sg[0][k] + p.T[a][1] * p.Sg[1][k] + p.T[a][2] * p.Sg[2][k];
  const double lp = (mode & ORC_NO_LOWPASS) ? 0.0 : 0.3;
  p.a = TS[0][0] * p.T[0][0] + TS[0][1] * p.T[0][1] + TS[0][2] * p.T[0][2] + lp;
  p.b = TS[0][0] * p.T[1][0] + TS[0][1] * p.T[1][1] + TS[0][2] * p.T[1][2];
  p.c = TS[1][0] * p.T[1][0] + TS[1][1] * p.T[1][1] + TS[1][2] * p.T[1][2] + lp;
  p.det = p.a * p.c - p.b * p.b;
  p.conic[0] = p.c / p.det;
  p.conic[1] = -p.b / p.det;
  p.conic[2] = p.a / p.det;
  for (int k = 0; k < 3; ++k) p.dir[k] = mu[k] - (double)cam.campos[k];
  p.dl = std::sqrt(p.dir[0] * p.dir[0] + p.dir[1] * p.dir[1] + p.dir[2] * p.dir[2]);
  for (int k = 0; k < 3; ++k) p.d[k] = p.dir[k] / p.dl;
  sh_basis<double>(p.d[0], p.d[1], p.d[2], p.Y, p.dY);
  const double* sh = th.sh(i);
  for (int ch = 0; ch < 3; ++ch) {
    double acc = 0.0;
    for (int k = 0; k < n_coeffs(deg); ++k) acc += p.Y[k] * sh[3 * k + ch];
    acc += 0.5;
    p.rgb[ch] = (cbits & (1u << ch)) ? 0.0 : acc;
  }
}

struct PixelList {  // frozen per-pixel decisions: blended Gaussians in order, alpha clamp flags
  const int64_t* ptr;
  const int32_t* gid;
  const uint8_t* aclamp;
};

}  // namespace

// ===========================================================================
// C ABI of the oracle (ctypes from oracle/__init__.py)
// ===========================================================================
extern "C" {

int32_t orc_version(void) { return 2; }

// Threads used by the parallel loops (k <= 0: all host cores); returns the count in effect.
int32_t orc_set_threads(int32_t k) {
  omp_set_num_threads(k > 0 ? k : omp_get_num_procs());
  return omp_get_max_threads();
}

// O1-O9 for every Gaussian.  Outputs for culled Gaussians: radius 0, tiles 0, rest 0.
void orc_preprocess(int64_t n, int32_t deg, const float* theta, const orc_camera* cam, uint32_t mode,
                    int32_t* radius, float* depth, float* xy, float* conic, float* opacity, float* rgb,
                    uint8_t* cbits, int32_t* rect, uint32_t* tiles_touched) {
  Theta th{n, theta};
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    const PreF p = preprocess_one(th, i, deg, *cam, mode);
    radius[i] = p.visible ? p.radius : 0;
    depth[i] = p.depth;
    xy[2 * i] = p.x;
    xy[2 * i + 1] = p.y;
    for (int k = 0; k < 3; ++k) {
      conic[3 * i + k] = p.conic[k];
      rgb[3 * i + k] = p.rgb[k];
    }
    opacity[i] = p.opacity;
    cbits[i] = p.cbits;
    for (int k = 0; k < 4; ++k) rect[4 * i + k] = p.rect[k];
    tiles_touched[i] = p.visible ? (uint32_t)((p.rect[2] - p.rect[0]) * (p.rect[3] - p.rect[1])) : 0u;
  }
}

// O10: exclusive scan in index order; returns K.
int64_t orc_scan(int64_t n, const uint32_t* tiles_touched, uint64_t* offsets) {
  uint64_t acc = 0;
  for (int64_t i = 0; i < n; ++i) {
    offsets[i] = acc;
    acc += tiles_touched[i];
  }
  return (int64_t)acc;
}

// O11: keys in index order, each rect ty-major (R13).
void orc_duplicate(int64_t n, const uint32_t* tiles_touched, const float* depth, const int32_t* rect,
                   const uint64_t* offsets, int32_t tiles_x, uint64_t* keys, uint32_t* values) {
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    if (tiles_touched[i] == 0) continue;
    uint64_t o = offsets[i];
    for (int32_t ty = rect[4 * i + 1]; ty < rect[4 * i + 3]; ++ty)
      for (int32_t tx = rect[4 * i + 0]; tx < rect[4 * i + 2]; ++tx) {
        keys[o] = ((uint64_t)(uint32_t)(ty * tiles_x + tx) << 32) | (uint64_t)float_bits(depth[i]);
        values[o] = (uint32_t)i;
        ++o;
      }
  }
}

// O12: stable ascending sort by the 64-bit key (library routines: std::stable_sort on
// contiguous chunks, then rounds of std::merge of neighbouring sorted runs -- std::merge
// takes the left run's element first on equal keys, so the result is the stable order).
void orc_sort(int64_t k, uint64_t* keys, uint32_t* values) {
  typedef std::pair<uint64_t, uint32_t> KV;
  auto by_key = [](const KV& a, const KV& b) { return a.first < b.first; };
  std::vector<KV> kv((size_t)k), tmp;
#pragma omp parallel for schedule(static, 65536)
  for (int64_t i = 0; i < k; ++i) kv[i] = {keys[i], values[i]};
  const int64_t chunks = k < (1 << 16) ? 1 : std::max<int64_t>(1, omp_get_max_threads());
  const int64_t len = (k + chunks - 1) / std::max<int64_t>(1, chunks);
#pragma omp parallel for schedule(static, 1)
  for (int64_t c = 0; c < chunks; ++c) {
    const int64_t lo = std::min(k, c * len), hi = std::min(k, lo + len);
    std::stable_sort(kv.begin() + lo, kv.begin() + hi, by_key);
  }
  if (chunks > 1) tmp.resize((size_t)k);
  for (int64_t w = len; w < k; w *= 2) {  // merge runs [lo, lo+w) and [lo+w, lo+2w)
    const int64_t pairs = (k + 2 * w - 1) / (2 * w);
#pragma omp parallel for schedule(static, 1)
    for (int64_t pi = 0; pi < pairs; ++pi) {
      const int64_t lo = pi * 2 * w, mid = std::min(k, lo + w), hi = std::min(k, lo + 2 * w);
      std::merge(kv.begin() + lo, kv.begin() + mid, kv.begin() + mid, kv.begin() + hi, tmp.begin() + lo, by_key);
    }
    kv.swap(tmp);
  }
#pragma omp parallel for schedule(static, 65536)
  for (int64_t i = 0; i < k; ++i) {
    keys[i] = kv[i].first;
    values[i] = kv[i].second;
  }
}

// O13: ranges[2t], ranges[2t+1] = [start, end) of tile t; (0, 0) if empty.
void orc_ranges(int64_t k, const uint64_t* keys, int32_t num_tiles, uint32_t* ranges) {
  std::memset(ranges, 0, sizeof(uint32_t) * 2 * (size_t)num_tiles);
  for (int64_t i = 0; i < k; ++i) {
    const uint32_t t = (uint32_t)(keys[i] >> 32);
    if (i == 0 || (uint32_t)(keys[i - 1] >> 32) != t) ranges[2 * t] = (uint32_t)i;
    if (i == k - 1 || (uint32_t)(keys[i + 1] >> 32) != t) ranges[2 * t + 1] = (uint32_t)(i + 1);
  }
}

// O14: blend forward per pixel.  Optional list outputs (frozen decisions) when
// list_ptr != NULL: list_ptr[P+1] (CSR over pixels, row-major), list_gid, list_aclamp
// sized by the caller to the sum of the pixels' tile-list lengths.
void orc_render_fwd(const orc_camera* cam, uint32_t mode, const uint32_t* ranges, const uint32_t* values,
                    const float* xy, const float* conic, const float* opacity, const float* rgb,
                    float* image, float* final_T, uint32_t* n_contrib, uint32_t* walked, uint32_t* blended,
                    uint8_t* flags, double delta_alpha, double delta_T,
                    int64_t* list_ptr, int32_t* list_gid, uint8_t* list_aclamp) {
  const int W = cam->width, H = cam->height;
  const int tiles_x = (W + TILE - 1) / TILE;
  const Gauss2D g{xy, conic, opacity, rgb};
  int64_t cursor = 0;  // list outputs (frozen decisions) are written in pixel order: serial
  auto pixel = [&](int px, int py) {
    const int t = (py / TILE) * tiles_x + (px / TILE);
    const int64_t pix = (int64_t)py * W + px;
    if (list_ptr) list_ptr[pix] = cursor;
    const WalkOut w = walk_pixel(g, values, ranges[2 * t], ranges[2 * t + 1], (float)px, (float)py, mode,
                                 delta_alpha, delta_T, [&](uint32_t id, bool ac, uint32_t) {
                                   if (list_ptr) {
                                     list_gid[cursor] = (int32_t)id;
                                     list_aclamp[cursor] = ac ? 1 : 0;
                                     ++cursor;
                                   }
                                 });
    for (int ch = 0; ch < 3; ++ch) image[(int64_t)ch * H * W + pix] = std::fma(w.T, cam->bg[ch], w.C[ch]);
    final_T[pix] = w.T;
    n_contrib[pix] = (uint32_t)w.last;
    if (walked) walked[pix] = (uint32_t)w.walked;
    if (blended) blended[pix] = (uint32_t)w.blended;
    if (flags) flags[pix] = w.flagged ? 1 : 0;
  };
  if (list_ptr) {
    for (int py = 0; py < H; ++py)
      for (int px = 0; px < W; ++px) pixel(px, py);
  } else {
#pragma omp parallel for schedule(dynamic, 1)
    for (int py = 0; py < H; ++py)
      for (int px = 0; px < W; ++px) pixel(px, py);
  }
  if (list_ptr) list_ptr[(int64_t)H * W] = cursor;
}

// Brute-force evaluator: per pixel, every visible Gaussian whose
// rect contains the pixel's tile, std::sort by (depth bits, index), same walk.
void orc_render_bruteforce(const orc_camera* cam, uint32_t mode, int64_t n, const uint32_t* tiles_touched,
                           const int32_t* rect, const float* depth, const float* xy, const float* conic,
                           const float* opacity, const float* rgb, float* image, float* final_T,
                           uint32_t* n_contrib) {
  const int W = cam->width, H = cam->height;
  const Gauss2D g{xy, conic, opacity, rgb};
  std::vector<uint32_t> lst;
  for (int py = 0; py < H; ++py)
    for (int px = 0; px < W; ++px) {
      const int tx = px / TILE, ty = py / TILE;
      lst.clear();
      for (int64_t i = 0; i < n; ++i)
        if (tiles_touched[i] && rect[4 * i] <= tx && tx < rect[4 * i + 2] && rect[4 * i + 1] <= ty &&
            ty < rect[4 * i + 3])
          lst.push_back((uint32_t)i);
      std::sort(lst.begin(), lst.end(), [&](uint32_t a, uint32_t b) {
        const uint32_t da = float_bits(depth[a]), db = float_bits(depth[b]);
        return da != db ? da < db : a < b;
      });
      const WalkOut w = walk_pixel(g, lst.data(), 0, (uint32_t)lst.size(), (float)px, (float)py, mode, 0.0, 0.0,
                                   [](uint32_t, bool, uint32_t) {});
      const int64_t pix = (int64_t)py * W + px;
      for (int ch = 0; ch < 3; ++ch) image[(int64_t)ch * H * W + pix] = std::fma(w.T, cam->bg[ch], w.C[ch]);
      final_T[pix] = w.T;
      n_contrib[pix] = (uint32_t)w.last;
    }
}

// Frozen-decision forward in double (R18): the function whose derivative
// orc_render_bwd + orc_preprocess_bwd compute.  theta_d is double[59n].
void orc_render_frozen(int64_t n, int32_t deg, const double* theta_d, const orc_camera* cam, uint32_t mode,
                       const int32_t* radius, const uint8_t* cbits, const int64_t* list_ptr,
                       const int32_t* list_gid, const uint8_t* list_aclamp, double* image) {
  ThetaD th{n, theta_d};
  std::vector<PreD> pre((size_t)n);
  for (int64_t i = 0; i < n; ++i)
    if (radius[i] > 0) preprocess_double(th, i, deg, *cam, mode, cbits[i], pre[i]);
  const int W = cam->width, H = cam->height;
  for (int64_t pix = 0; pix < (int64_t)W * H; ++pix) {
    const double pxf = (double)(pix % W), pyf = (double)(pix / W);
    double C[3] = {0, 0, 0}, T = 1.0;
    for (int64_t e = list_ptr[pix]; e < list_ptr[pix + 1]; ++e) {
      const PreD& p = pre[list_gid[e]];
      const double dx = p.xy[0] - pxf, dy = p.xy[1] - pyf;
      const double power = -0.5 * (p.conic[0] * dx * dx + p.conic[2] * dy * dy) - p.conic[1] * dx * dy;
      const double alpha = list_aclamp[e] ? 0.99 : p.o * std::exp(power);
      for (int ch = 0; ch < 3; ++ch) C[ch] += p.rgb[ch] * alpha * T;
      T *= (1.0 - alpha);
    }
    for (int ch = 0; ch < 3; ++ch) image[(int64_t)ch * H * W + pix] = C[ch] + T * (double)cam->bg[ch];
  }
}

// O15: blend backward per pixel (double, decisions frozen from the float walk).
// Outputs per-Gaussian sums (double, +=): g_xy[2n] (pixel units), g_conic[3n]
// (w.r.t. conic = Sigma'^-1 entries (xx, xy, yy)), g_opac[n], g_rgb[3n].
// Sum order (fixed, thread-count independent): within a tile over its pixels in row-major
// order into per-list-position partials, then the tiles' partials in tile index order.
namespace {
struct Blend2D {  // what the double backward reads per Gaussian (from preprocess_double)
  double xy[2], conic[3], o, rgb[3];
};
}  // namespace

void orc_render_bwd(int64_t n, int32_t deg, const float* theta, const orc_camera* cam, uint32_t mode,
                    const int32_t* radius, const uint8_t* cbits, const uint32_t* ranges, const uint32_t* values,
                    const float* xy, const float* conic, const float* opacity, const float* rgb,
                    const float* dl_dimage, double* g_xy, double* g_conic, double* g_opac, double* g_rgb) {
  std::vector<double> thd((size_t)59 * n);
#pragma omp parallel for schedule(static, 65536)
  for (int64_t k = 0; k < 59 * n; ++k) thd[k] = theta[k];
  ThetaD th{n, thd.data()};
  std::vector<Blend2D> pre((size_t)n);
#pragma omp parallel for schedule(static, 4096)
  for (int64_t i = 0; i < n; ++i) {
    if (radius[i] <= 0) continue;
    PreD p;
    preprocess_double(th, i, deg, *cam, mode, cbits[i], p);
    Blend2D& b = pre[i];
    for (int k = 0; k < 2; ++k) b.xy[k] = p.xy[k];
    for (int k = 0; k < 3; ++k) { b.conic[k] = p.conic[k]; b.rgb[k] = p.rgb[k]; }
    b.o = p.o;
  }
  const int W = cam->width, H = cam->height;
  const int tiles_x = (W + TILE - 1) / TILE, tiles_y = (H + TILE - 1) / TILE;
  const int num_tiles = tiles_x * tiles_y;
  const Gauss2D g{xy, conic, opacity, rgb};
  enum { NACC = 9 };  // per list position: xy 2, conic 3, opacity 1, rgb 3
  // one tile: every pixel's walk and double backward, partials per list position
  auto tile_partials = [&](int t, std::vector<double>& acc) {
    const uint32_t start = ranges[2 * t], end = ranges[2 * t + 1];
    acc.assign((size_t)(end - start) * NACC, 0.0);
    std::vector<uint32_t> ids, pos;
    std::vector<uint8_t> acl;
    std::vector<double> al, Tb, Gv;
    const int ty = t / tiles_x, tx = t % tiles_x;
    for (int py = ty * TILE; py < std::min(H, ty * TILE + TILE); ++py)
      for (int px = tx * TILE; px < std::min(W, tx * TILE + TILE); ++px) {
        ids.clear();
        pos.clear();
        acl.clear();
        walk_pixel(g, values, start, end, (float)px, (float)py, mode, 0.0, 0.0,
                   [&](uint32_t id, bool ac, uint32_t ps) {
                     ids.push_back(id);
                     pos.push_back(ps - start);
                     acl.push_back(ac ? 1 : 0);
                   });
        const int m = (int)ids.size();
        if (m == 0) continue;
        const int64_t pix = (int64_t)py * W + px;
        double dLdC[3];
        for (int ch = 0; ch < 3; ++ch) dLdC[ch] = dl_dimage[(int64_t)ch * H * W + pix];
        al.assign(m, 0.0);
        Tb.assign(m + 1, 0.0);
        Gv.assign(m, 0.0);
        Tb[0] = 1.0;
        for (int j = 0; j < m; ++j) {
          const Blend2D& p = pre[ids[j]];
          const double dx = p.xy[0] - px, dy = p.xy[1] - py;
          const double power = -0.5 * (p.conic[0] * dx * dx + p.conic[2] * dy * dy) - p.conic[1] * dx * dy;
          Gv[j] = std::exp(power);
          al[j] = acl[j] ? 0.99 : p.o * Gv[j];
          Tb[j + 1] = Tb[j] * (1.0 - al[j]);
        }
        double S[3];
        for (int ch = 0; ch < 3; ++ch) S[ch] = Tb[m] * (double)cam->bg[ch];
        for (int j = m - 1; j >= 0; --j) {
          const Blend2D& p = pre[ids[j]];
          double* a = acc.data() + (size_t)pos[j] * NACC;  // [xy 0-1 | conic 2-4 | opac 5 | rgb 6-8]
          double dLda = 0.0;
          for (int ch = 0; ch < 3; ++ch) {
            a[6 + ch] += dLdC[ch] * al[j] * Tb[j];
            dLda += dLdC[ch] * (p.rgb[ch] * Tb[j] - S[ch] / (1.0 - al[j]));
            S[ch] += p.rgb[ch] * al[j] * Tb[j];
          }
          if (acl[j]) continue;  // clamped alpha: zero gradient to o and G (R18)
          const double dx = p.xy[0] - px, dy = p.xy[1] - py;
          a[5] += dLda * Gv[j];
          const double dLdp = dLda * p.o * Gv[j];
          a[0] += dLdp * (-p.conic[0] * dx - p.conic[1] * dy);
          a[1] += dLdp * (-p.conic[2] * dy - p.conic[1] * dx);
          a[2] += dLdp * (-0.5 * dx * dx);
          a[3] += dLdp * (-dx * dy);
          a[4] += dLdp * (-0.5 * dy * dy);
        }
      }
  };
  const int batch = std::max(1, 8 * omp_get_max_threads());
  std::vector<std::vector<double>> accs((size_t)batch);
  for (int t0 = 0; t0 < num_tiles; t0 += batch) {
    const int t1 = std::min(num_tiles, t0 + batch);
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = t0; t < t1; ++t) tile_partials(t, accs[t - t0]);
    for (int t = t0; t < t1; ++t) {  // fixed order: tiles in index order, positions in list order
      const std::vector<double>& acc = accs[t - t0];
      const uint32_t start = ranges[2 * t];
      for (size_t q = 0; q < acc.size() / NACC; ++q) {
        const uint32_t id = values[start + q];
        const double* a = acc.data() + q * NACC;
        g_xy[2 * id] += a[0];
        g_xy[2 * id + 1] += a[1];
        for (int k = 0; k < 3; ++k) g_conic[3 * id + k] += a[2 + k];
        g_opac[id] += a[5];
        for (int k = 0; k < 3; ++k) g_rgb[3 * id + k] += a[6 + k];
      }
    }
  }
}

// O16: preprocess backward (double, decisions frozen), grad59[59n] +=.
void orc_preprocess_bwd(int64_t n, int32_t deg, const float* theta, const orc_camera* cam, uint32_t mode,
                        const int32_t* radius, const uint8_t* cbits, const double* g_xy, const double* g_conic,
                        const double* g_opac, const double* g_rgb, double* grad) {
  std::vector<double> thd((size_t)59 * n);
#pragma omp parallel for schedule(static, 65536)
  for (int64_t k = 0; k < 59 * n; ++k) thd[k] = theta[k];
  ThetaD th{n, thd.data()};
  double V[16], P[16];
  for (int k = 0; k < 16; ++k) { V[k] = cam->view[k]; P[k] = cam->proj[k]; }
  const int ncf = n_coeffs(deg);
#pragma omp parallel for schedule(static, 1024)
  for (int64_t i = 0; i < n; ++i) {
    if (radius[i] <= 0) continue;
    PreD p;
    preprocess_double(th, i, deg, *cam, mode, cbits[i], p);
    double* gm = grad + 3 * i;
    double* gls = grad + 3 * n + 3 * i;
    double* gq = grad + 6 * n + 4 * i;
    double* go = grad + 10 * n + i;
    double* gsh = grad + 11 * n + 48 * i;
    double dmu[3] = {0, 0, 0};
    // colour (R12): masked by the frozen clamp, SH coefficients and view direction
    double gr[3];
    for (int ch = 0; ch < 3; ++ch) gr[ch] = (cbits[i] & (1u << ch)) ? 0.0 : g_rgb[3 * i + ch];
    const double* sh = th.sh(i);
    double dLdd[3] = {0, 0, 0};
    for (int k = 0; k < ncf; ++k) {
      double shg = 0.0;
      for (int ch = 0; ch < 3; ++ch) {
        gsh[3 * k + ch] += p.Y[k] * gr[ch];
        shg += sh[3 * k + ch] * gr[ch];
      }
      for (int j = 0; j < 3; ++j) dLdd[j] += p.dY[k][j] * shg;
    }
    const double ddot = dLdd[0] * p.d[0] + dLdd[1] * p.d[1] + dLdd[2] * p.d[2];
    for (int j = 0; j < 3; ++j) dmu[j] += (dLdd[j] - p.d[j] * ddot) / p.dl;
    // opacity
    *go += g_opac[i] * p.o * (1.0 - p.o);
    // conic -> (a, b, c) of Sigma'
    const double gx = g_conic[3 * i], gy = g_conic[3 * i + 1], gz = g_conic[3 * i + 2];
    const double a = p.a, b = p.b, c = p.c, d2 = p.det * p.det;
    const double ga = (-c * c * gx + b * c * gy - b * b * gz) / d2;
    const double gb = (2 * b * c * gx - (a * c + b * b) * gy + 2 * a * b * gz) / d2;
    const double gc = (-b * b * gx + a * b * gy - a * a * gz) / d2;
    const double Gp[2][2] = {{ga, 0.5 * gb}, {0.5 * gb, gc}};
    // Sigma' = T Sigma T^T: dL/dSigma = T^T G' T,  dL/dT = 2 G' T Sigma
    double GS[3][3];
    for (int r = 0; r < 3; ++r)
      for (int s = 0; s < 3; ++s) {
        double acc = 0;
        for (int u = 0; u < 2; ++u)
          for (int v = 0; v < 2; ++v) acc += p.T[u][r] * Gp[u][v] * p.T[v][s];
        GS[r][s] = acc;
      }
    double TS[2][3];
    for (int u = 0; u < 2; ++u)
      for (int k = 0; k < 3; ++k) TS[u][k] = p.T[u][0] * p.Sg[0][k] + p.T[u][1] * p.Sg[1][k] + p.T[u][2] * p.Sg[2][k];
    double gT[2][3];
    for (int u = 0; u < 2; ++u)
      for (int k = 0; k < 3; ++k) gT[u][k] = 2.0 * (Gp[u][0] * TS[0][k] + Gp[u][1] * TS[1][k]);
    // T = J W3
    double gj00 = 0, gj02 = 0, gj11 = 0, gj12 = 0;
    for (int k = 0; k < 3; ++k) {
      gj00 += gT[0][k] * V[0 + 4 * k];
      gj02 += gT[0][k] * V[2 + 4 * k];
      gj11 += gT[1][k] * V[1 + 4 * k];
      gj12 += gT[1][k] * V[2 + 4 * k];
    }
    // J(t) with the frozen clamp branch (R7, R18)
    const double tz = p.t[2], tz2 = tz * tz;
    double gt[3] = {0, 0, 0};
    gt[2] += gj00 * (-p.fx / tz2) + gj11 * (-p.fy / tz2);
    if (cbits[i] & CB_JX) {
      gt[2] += gj02 * (p.fx * p.u / tz2);
    } else {
      gt[0] += gj02 * (-p.fx / tz2);
      gt[2] += gj02 * (2.0 * p.fx * p.t[0] / (tz2 * tz));
    }
    if (cbits[i] & CB_JY) {
      gt[2] += gj12 * (p.fy * p.v / tz2);
    } else {
      gt[1] += gj12 * (-p.fy / tz2);
      gt[2] += gj12 * (2.0 * p.fy * p.t[1] / (tz2 * tz));
    }
    for (int k = 0; k < 3; ++k) dmu[k] += V[0 + 4 * k] * gt[0] + V[1 + 4 * k] * gt[1] + V[2 + 4 * k] * gt[2];
    // projected mean (O3)
    const double c0 = p.clip[0], c1 = p.clip[1], c3 = p.clip[3];
    for (int k = 0; k < 3; ++k) {
      dmu[k] += g_xy[2 * i] * 0.5 * cam->width * (P[0 + 4 * k] * c3 - P[3 + 4 * k] * c0) / (c3 * c3);
      dmu[k] += g_xy[2 * i + 1] * 0.5 * cam->height * (P[1 + 4 * k] * c3 - P[3 + 4 * k] * c1) / (c3 * c3);
    }
    for (int k = 0; k < 3; ++k) gm[k] += dmu[k];
    // Sigma = M M^T, M = R diag(s)
    double gM[3][3];
    for (int r = 0; r < 3; ++r)
      for (int k = 0; k < 3; ++k) gM[r][k] = 2.0 * (GS[r][0] * p.M[0][k] + GS[r][1] * p.M[1][k] + GS[r][2] * p.M[2][k]);
    double gR[3][3];
    for (int k = 0; k < 3; ++k) {
      double gs = 0;
      for (int r = 0; r < 3; ++r) {
        gs += gM[r][k] * p.R[r][k];
        gR[r][k] = gM[r][k] * p.s[k];
      }
      gls[k] += gs * p.s[k];
    }
    const double w = p.q[0], x = p.q[1], y = p.q[2], z = p.q[3];
    double gqn[4];
    gqn[0] = 2 * (-z * gR[0][1] + y * gR[0][2] + z * gR[1][0] - x * gR[1][2] - y * gR[2][0] + x * gR[2][1]);
    gqn[1] = 2 * (y * gR[0][1] + z * gR[0][2] + y * gR[1][0] - 2 * x * gR[1][1] - w * gR[1][2] + z * gR[2][0] +
                  w * gR[2][1] - 2 * x * gR[2][2]);
    gqn[2] = 2 * (-2 * y * gR[0][0] + x * gR[0][1] + w * gR[0][2] + x * gR[1][0] + z * gR[1][2] - w * gR[2][0] +
                  z * gR[2][1] - 2 * y * gR[2][2]);
    gqn[3] = 2 * (-2 * z * gR[0][0] - w * gR[0][1] + x * gR[0][2] + w * gR[1][0] - 2 * z * gR[1][1] + y * gR[1][2] +
                  x * gR[2][0] + y * gR[2][1]);
    const double qd = gqn[0] * p.q[0] + gqn[1] * p.q[1] + gqn[2] * p.q[2] + gqn[3] * p.q[3];
    for (int k = 0; k < 4; ++k) gq[k] += (gqn[k] - p.q[k] * qd) / p.qn;
  }
}

// NEXT-1, T1 statistical density thresholding (§III-C1 l.181-186): "the local
// density rho is determined as the number of neighboring points within a fixed radius r".
// Plain O(n^2) definition: rho(p) = #{q != p : |q - p| <= r}, with the squared distance
// evaluated as ((dx*dx + dy*dy) + dz*dz) in float (separately rounded) and compared with
// r*r in float -- the same decision the GPU grid kernel takes.
void orc_local_density(int64_t n, const float* means, float r, uint32_t* counts) {
  const float r2 = r * r;
  for (int64_t i = 0; i < n; ++i) {
    uint32_t c = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const float dx = means[3 * j] - means[3 * i];
      const float dy = means[3 * j + 1] - means[3 * i + 1];
      const float dz = means[3 * j + 2] - means[3 * i + 2];
      const float d2 = (dx * dx + dy * dy) + dz * dz;
      if (d2 <= r2) ++c;
    }
    counts[i] = c;
  }
}

// §III-C2 l.190: mean distance to the k nearest neighbours, d_p = (1/k) sum_i d(p, p_i)
// (double, brute force with std::partial_sort).
void orc_knn_mean(int64_t n, const float* means, int32_t k, double* out) {
  std::vector<double> d((size_t)(n > 0 ? n - 1 : 0));
  for (int64_t i = 0; i < n; ++i) {
    size_t m = 0;
    for (int64_t j = 0; j < n; ++j) {
      if (j == i) continue;
      const double dx = (double)means[3 * j] - means[3 * i];
      const double dy = (double)means[3 * j + 1] - means[3 * i + 1];
      const double dz = (double)means[3 * j + 2] - means[3 * i + 2];
      d[m++] = std::sqrt(dx * dx + dy * dy + dz * dz);
    }
    const size_t kk = std::min<size_t>((size_t)k, m);
    std::partial_sort(d.begin(), d.begin() + kk, d.begin() + m);
    double acc = 0.0;
    for (size_t t = 0; t < kk; ++t) acc += d[t];
    out[i] = kk ? acc / (double)kk : 0.0;
  }
}

// R23 parity mode's exponential, exposed for its pin (tests/test_oracle_blend.py)
void orc_canon_exp(int64_t n, const float* x, float* out) {
  for (int64_t i = 0; i < n; ++i) out[i] = canon_exp(x[i]);
}

// O17: Adam (R21), PyTorch semantics, in double.  lr[6] = means, log_scales,
// quats, opacity, sh_dc, sh_rest.  grad is zeroed on exit.
void orc_adam(int64_t n, double* theta, double* grad, double* m, double* v, const double* lr, double b1, double b2,
              double eps, int64_t step) {
  const double bc1 = 1.0 - std::pow(b1, (double)step), bc2 = 1.0 - std::pow(b2, (double)step);
#pragma omp parallel for schedule(static, 65536)
  for (int64_t e = 0; e < 59 * n; ++e) {
    int grp;
    if (e < 3 * n) grp = 0;
    else if (e < 6 * n) grp = 1;
    else if (e < 10 * n) grp = 2;
    else if (e < 11 * n) grp = 3;
    else grp = ((e - 11 * n) % 48) < 3 ? 4 : 5;
    const double g = grad[e];
    m[e] = b1 * m[e] + (1.0 - b1) * g;
    v[e] = b2 * v[e] + (1.0 - b2) * g * g;
    theta[e] -= lr[grp] * (m[e] / bc1) / (std::sqrt(v[e] / bc2) + eps);
    grad[e] = 0.0;
  }
}

}  // extern "C"
