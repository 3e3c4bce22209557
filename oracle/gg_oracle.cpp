// gg_oracle.cpp — plain, slow, CPU oracle for the batched 3DGS render path.
//
// TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header, table or constant generator with
// paper_2510_15352_b200/ (the CUDA product path), and never reads anything
// that path produced.
//
// What it computes (DESIGN.md §2 "Definition"):
//   the 3D Gaussian Splatting forward pass that GaussGym uses as its renderer
//   (§3.2 "3D Gaussian Splatting as a Drop-in Renderer",
//   PAPER.md:184 Fig.4 "depth is a by-product"), with the constants SPEC.md
//   fixes (SPEC.md:117-153 rasterizer types/ops, SPEC.md:183 design decisions).
//
//   O1  per Gaussian      : normalise q, R(q), Sigma3 = R diag(s)^2 R^T, DC colour
//                           (SPEC.md:28-34 SplatPrimitive, SPEC.md:130 project_gaussian)
//   O2  per env x Gaussian: world->camera, near/far cull, clamped EWA Jacobian,
//                           Sigma2 + 0.3 I, conic, r = ceil(3 sqrt(lambda1)), tile
//                           rect, SH colour   (readings R3-R8, R16-R17)
//   O3  per env           : per-tile lists sorted by (tile, depth bits, gid)
//                           (SPEC.md:136-144 bin_and_sort)
//   O4  per pixel         : front-to-back compositing, alpha clamp 0.99, 1/255
//                           cutoff, stop when T(1-alpha) < 1e-4
//   O5  outputs           : rgb = C + T bg, depth = sum(w z)/sum(w), alpha = sum(w),
//                           u8 = round-half-even(clamp(rgb)*255)
//
// Precision (DESIGN.md §2.2 "precision modes"):
//   mode A (default): O1-O3 in float32 following the canonical operation order
//     written in DESIGN.md §2.1 (each op correctly rounded, no contraction:
//     this file MUST be compiled with -ffp-contract=off and without
//     -ffast-math); O4-O5 in float64 over the f32 records.  Integer artefacts
//     (tile counts, sorted lists, ranges) are defined by this mode.
//   mode B (diagnostic): O1-O2 in float64 as well.
//
// Drivers: "binned" composites each pixel over its tile's sorted list;
// "plain" composites each pixel over ALL visible Gaussians in global
// (depth bits, gid) order, keeping those whose tile rect contains the pixel's
// tile.  They visit the same sequence, so they agree bit-for-bit in f64.
//
// Built by oracle/build.sh (g++ -O2 -fopenmp -ffp-contract=off -std=c++17).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <vector>

#ifdef _OPENMP
#include <omp.h>
#endif

namespace {

// ---- constants fixed by SPEC.md / the 3DGS definition --------------------
// SH basis constants: real spherical harmonics with the (-1)^m phase used by
// 3DGS (pinned in tests by quadrature + scipy).
const double SH_C0 = 0.28209479177387814;
const double SH_C1 = 0.4886025119029199;
const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                         -1.0925484305920792, 0.5462742152960396};
const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                         0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                         -0.5900435899266435};
const int TILE = 16;                      // SPEC.md:183 "Tile size 16x16"

struct Scene {
  int64_t n = 0;
  int d = 0;
  std::vector<float> means, scales, quats, opac, sh;   // inputs (copied)
  std::vector<float> cov32;     // [n*6] O1 in f32 canonical order
  std::vector<double> cov64;    // [n*6] O1 in f64 (mode B)
};

// O1 — DESIGN.md §2.1 "O1": q <- q/|q|; R(q); M = R diag(s); Sigma3 = M M^T.
template <typename T>
void cov3_of(const float* qin, const float* sin, T out[6]) {
  T w = (T)qin[0], x = (T)qin[1], y = (T)qin[2], z = (T)qin[3];
  T nrm = std::sqrt(((w * w + x * x) + y * y) + z * z);
  w = w / nrm; x = x / nrm; y = y / nrm; z = z / nrm;
  const T one = (T)1, two = (T)2;
  T R[3][3];
  R[0][0] = one - two * (y * y + z * z);
  R[0][1] = two * (x * y - w * z);
  R[0][2] = two * (x * z + w * y);
  R[1][0] = two * (x * y + w * z);
  R[1][1] = one - two * (x * x + z * z);
  R[1][2] = two * (y * z - w * x);
  R[2][0] = two * (x * z - w * y);
  R[2][1] = two * (y * z + w * x);
  R[2][2] = one - two * (x * x + y * y);
  T M[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) M[i][j] = R[i][j] * (T)sin[j];
  auto S = [&](int i, int j) { return (M[i][0] * M[j][0] + M[i][1] * M[j][1]) + M[i][2] * M[j][2]; };
  out[0] = S(0, 0); out[1] = S(0, 1); out[2] = S(0, 2);
  out[3] = S(1, 1); out[4] = S(1, 2); out[5] = S(2, 2);
}

// SH basis values Y_k(dir), k < (d+1)^2, 3DGS real-SH convention.
void sh_basis(int d, double x, double y, double z, double* Y) {
  Y[0] = SH_C0;
  if (d < 1) return;
  Y[1] = -SH_C1 * y;
  Y[2] = SH_C1 * z;
  Y[3] = -SH_C1 * x;
  if (d < 2) return;
  double xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
  Y[4] = SH_C2[0] * xy;
  Y[5] = SH_C2[1] * yz;
  Y[6] = SH_C2[2] * (2.0 * zz - xx - yy);
  Y[7] = SH_C2[3] * xz;
  Y[8] = SH_C2[4] * (xx - yy);
  if (d < 3) return;
  Y[9] = SH_C3[0] * y * (3.0 * xx - yy);
  Y[10] = SH_C3[1] * xy * z;
  Y[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
  Y[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
  Y[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
  Y[14] = SH_C3[5] * z * (xx - yy);
  Y[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

// One projected Gaussian (the record O4 consumes) + its integer artefacts.
struct Proj {
  bool vis = false;
  double u = 0, v = 0, A = 0, B = 0, C = 0, z = 0, o = 0, col[3] = {0, 0, 0};
  float u32 = 0, v32 = 0, A32 = 0, B32 = 0, C32 = 0, z32 = 0;   // f32 values (mode A dump)
  int r = 0, x0 = 0, x1 = 0, y0 = 0, y1 = 0;
  uint32_t zbits = 0;
  float qm = 0.f;                // R35 cutoff with margin (set by tight_rect)
  uint32_t mask = 0xffffffffu;   // R37: kept tiles of a <= 32-tile rect, row-major bits
};

struct Cam {
  double R[3][3], t[3];      // world->camera, f64 copy of the f32 inputs
  float Rf[3][3], tf[3];
  float fx, fy, cx, cy;
  int W, H, TX, TY;
};

// O2 — DESIGN.md §2.1 "O2": canonical op order.  T = float (mode A) or
// double (mode B).  Returns false if culled (near plane, det<=0,
// 3-sigma footprint misses the image).
template <typename T>
bool project_geom(const float* mu, const T cov[6], const Cam& cam, T near_p, T far_p, Proj& P) {
  T R[3][3], t[3];
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) R[i][j] = (T)cam.Rf[i][j];
    t[i] = (T)cam.tf[i];
  }
  const T fx = (T)cam.fx, fy = (T)cam.fy, cx = (T)cam.cx, cy = (T)cam.cy;
  const T W = (T)cam.W, H = (T)cam.H;
  // camera constants (per env): Jacobian clamp limits (reading R4)
  const T tan_x = ((T)0.5 * W) / fx, tan_y = ((T)0.5 * H) / fy;
  const T lim_xp = (W - cx) / fx + (T)0.3 * tan_x;
  const T lim_xn = cx / fx + (T)0.3 * tan_x;
  const T lim_yp = (H - cy) / fy + (T)0.3 * tan_y;
  const T lim_yn = cy / fy + (T)0.3 * tan_y;
  // 1. p = R mu + t
  T p[3];
  for (int k = 0; k < 3; ++k)
    p[k] = ((R[k][0] * (T)mu[0] + R[k][1] * (T)mu[1]) + R[k][2] * (T)mu[2]) + t[k];
  if (p[2] <= near_p || p[2] > far_p) return false;
  const T rz = (T)1 / p[2];
  // 6. mean in pixels (unclamped p)
  const T u = (fx * p[0]) * rz + cx;
  const T v = (fy * p[1]) * rz + cy;
  // 2. clamped Jacobian
  T txz = p[0] * rz, tyz = p[1] * rz;
  txz = std::min(lim_xp, std::max(-lim_xn, txz));
  tyz = std::min(lim_yp, std::max(-lim_yn, tyz));
  const T xc = p[2] * txz, yc = p[2] * tyz;
  const T J00 = fx * rz, J11 = fy * rz;
  const T J02 = -(((fx * xc) * rz) * rz);
  const T J12 = -(((fy * yc) * rz) * rz);
  // 3. T = J W (2x3), Sigma2 = T Sigma3 T^T + 0.3 I
  T Tm[2][3];
  for (int j = 0; j < 3; ++j) {
    Tm[0][j] = J00 * R[0][j] + J02 * R[2][j];
    Tm[1][j] = J11 * R[1][j] + J12 * R[2][j];
  }
  const T S3[3][3] = {{cov[0], cov[1], cov[2]}, {cov[1], cov[3], cov[4]}, {cov[2], cov[4], cov[5]}};
  T U[2][3];
  for (int i = 0; i < 2; ++i)
    for (int j = 0; j < 3; ++j)
      U[i][j] = (Tm[i][0] * S3[0][j] + Tm[i][1] * S3[1][j]) + Tm[i][2] * S3[2][j];
  auto Sij = [&](int i, int j) { return (U[i][0] * Tm[j][0] + U[i][1] * Tm[j][1]) + U[i][2] * Tm[j][2]; };
  const T a = Sij(0, 0) + (T)0.3;
  const T b = Sij(0, 1);
  const T c = Sij(1, 1) + (T)0.3;
  // 4. determinant, conic
  const T det = a * c - b * b;
  if (!(det > (T)0)) return false;
  const T cA = c / det, cB = -b / det, cC = a / det;
  // 5. radius from the larger eigenvalue (eigenvalue floor 0.1, reading R6)
  const T mid = (T)0.5 * (a + c);
  const T lam1 = mid + std::sqrt(std::max((T)0.1, mid * mid - det));
  const T rr = std::ceil((T)3 * std::sqrt(lam1));
  // 7. tile rect [x0,x1) x [y0,y1), clamped to the grid (reading R8)
  const T inv16 = (T)0.0625;
  auto clampT = [](T x, T hi) { return std::min(std::max(x, (T)0), hi); };
  const T fx0 = clampT(std::floor((u - rr) * inv16), (T)cam.TX);
  const T fx1 = clampT(std::ceil((u + rr) * inv16), (T)cam.TX);
  const T fy0 = clampT(std::floor((v - rr) * inv16), (T)cam.TY);
  const T fy1 = clampT(std::ceil((v + rr) * inv16), (T)cam.TY);
  P.x0 = (int)fx0; P.x1 = (int)fx1; P.y0 = (int)fy0; P.y1 = (int)fy1;
  P.r = (int)rr;
  if (P.x0 >= P.x1 || P.y0 >= P.y1) return false;
  P.u = (double)u; P.v = (double)v; P.A = (double)cA; P.B = (double)cB; P.C = (double)cC;
  P.z = (double)p[2];
  P.u32 = (float)u; P.v32 = (float)v; P.A32 = (float)cA; P.B32 = (float)cB; P.C32 = (float)cC;
  P.z32 = (float)p[2];
  float zf = (float)p[2];
  std::memcpy(&P.zbits, &zf, 4);
  return true;
}

// Work-reduction variant (reading R35): the
// paper rect intersected with the tiles whose pixel centres can lie in the
// axis-aligned box of the alpha >= 1/255 ellipse.  alpha = o exp(-q/2) >=
// 1/255  <=>  q <= qmax = 2 ln(255 o); the ellipse {d : q(d) <= qm} of the
// f32 conic [[A,B],[B,C]] has half extents sqrt(qm C / D), sqrt(qm A / D),
// D = AC - B^2.  Evaluated in f32, each op correctly rounded in this order
// (it decides integers: the lists), with bounds that make every rounding
// conservative: D is replaced by a lower bound, the extents are inflated
// relatively and absolutely, and qm adds a margin over qmax that covers the
// f32 evaluation of every pixel.  So a dropped tile never holds a pixel that
// blends the Gaussian: images are unchanged, only the lists get shorter.
// qmax = f32(2 ln(255 o)) once per Gaussian (f64 log).
void tight_rect(Proj& P, float o) {
  P.qm = INFINITY;                                   // no pruning unless the tight rect is computed
  const float qmax = (float)(2.0 * std::log(255.0 * (double)o));
  if (!(qmax >= 0.0f)) { P.x0 = P.x1 = P.y0 = P.y1 = 0; return; }   // o < 1/255: no pixel blends
  const float A = P.A32, B = P.B32, C = P.C32;
  const float AC = A * C, BB = B * B;
  const float Dlo = (AC - BB) - 9.5367431640625e-07f * (AC + BB);     // 2^-20 (AC + BB): D >= Dlo
  if (!(Dlo > 0.0f) || !(A > 0.0f) || !(C > 0.0f)) return;             // degenerate: keep the paper rect
  const float rD = 1.0f / Dlo;
  // |A| ex0^2 + 2|B| ex0 ey0 + |C| ey0^2 at q = qmax, ex0^2 = qmax C / D, ey0^2 = qmax A / D
  const float mag = ((qmax * rD) * ((2.0f * AC) + (2.0f * std::fabs(B)) * std::sqrt(AC)));
  const float qm = (qmax + 1e-3f) + 1e-5f * mag;
  P.qm = qm;
  const float grow = 1.0000038146972656f;                              // 1 + 2^-18
  const float ex = std::sqrt((qm * C) * rD) * grow, ey = std::sqrt((qm * A) * rD) * grow;
  const float u = P.u32, v = P.v32;
  const float sx = (ex + 0.02f) + 1e-5f * std::fabs(u), sy = (ey + 0.02f) + 1e-5f * std::fabs(v);
  // tile t holds pixel centres 16 t + 0.5 .. 16 t + 15.5
  const float lx = std::ceil(((u - sx) - 15.5f) * 0.0625f), hx = std::floor(((u + sx) - 0.5f) * 0.0625f) + 1.0f;
  const float ly = std::ceil(((v - sy) - 15.5f) * 0.0625f), hy = std::floor(((v + sy) - 0.5f) * 0.0625f) + 1.0f;
  const int x0 = (int)std::max((float)P.x0, std::min((float)P.x1, lx));
  const int x1 = (int)std::max((float)P.x0, std::min((float)P.x1, hx));
  const int y0 = (int)std::max((float)P.y0, std::min((float)P.y1, ly));
  const int y1 = (int)std::max((float)P.y0, std::min((float)P.y1, hy));
  if (x0 >= x1 || y0 >= y1) { P.x0 = P.x1 = P.y0 = P.y1 = 0; return; }
  P.x0 = x0; P.x1 = x1; P.y0 = y0; P.y1 = y1;
}

// Work-reduction variant "ellipse ∩ tile" (DESIGN.md
// reading R37; needs F_TIGHT): a tile of a tight rect of at most 32 tiles is
// kept only if the f32 conic's quadratic q(d) = A dx^2 + 2B dx dy + C dy^2,
// minimised over the tile's rectangle of pixel centres, reaches q_m (R35) plus
// a rounding margin.  The minimum of a convex quadratic over a rectangle is 0
// if the mean lies inside, else on an edge: on the edge dx = e it is at
// dy = clamp(-B e / C) (and symmetrically).  Evaluated in f32 in this order.
bool tile_keeps(const Proj& P, int tx, int ty) {
  const float A = P.A32, B = P.B32, C = P.C32;
  const float dxl = (16.0f * (float)tx + 0.5f) - P.u32, dxh = (16.0f * (float)tx + 15.5f) - P.u32;
  const float dyl = (16.0f * (float)ty + 0.5f) - P.v32, dyh = (16.0f * (float)ty + 15.5f) - P.v32;
  if (dxl <= 0.0f && dxh >= 0.0f && dyl <= 0.0f && dyh >= 0.0f) return true;
  float best = INFINITY, mag = 0.0f;
  auto consider = [&](float dx, float dy) {
    const float q = ((A * dx) * dx + ((2.0f * B) * dx) * dy) + (C * dy) * dy;
    if (q < best) {
      best = q;
      mag = ((std::fabs(A) * dx) * dx + ((2.0f * std::fabs(B)) * std::fabs(dx)) * std::fabs(dy)) + (std::fabs(C) * dy) * dy;
    }
  };
  const float ex[2] = {dxl, dxh}, ey[2] = {dyl, dyh};
  for (int k = 0; k < 2; ++k) {
    consider(ex[k], std::min(std::max((-B * ex[k]) / C, dyl), dyh));
    consider(std::min(std::max((-B * ey[k]) / A, dxl), dxh), ey[k]);
  }
  return best <= (P.qm + 1e-3f) + 1e-5f * mag;
}

void ellipse_mask(Proj& P) {
  const int w = P.x1 - P.x0, h = P.y1 - P.y0;
  if (w * h <= 0 || w * h > 32) return;                  // larger rects are not pruned (R37)
  uint32_t m = 0;
  for (int ty = P.y0; ty < P.y1; ++ty)
    for (int tx = P.x0; tx < P.x1; ++tx)
      if (tile_keeps(P, tx, ty)) m |= 1u << ((ty - P.y0) * w + (tx - P.x0));
  P.mask = m;
}

bool in_list(const Proj& P, int tx, int ty) {
  if (tx < P.x0 || tx >= P.x1 || ty < P.y0 || ty >= P.y1) return false;
  const int w = P.x1 - P.x0, h = P.y1 - P.y0;
  return w * h > 32 || ((P.mask >> ((ty - P.y0) * w + (tx - P.x0))) & 1u);
}

// O2.8 colour (f64): degree 0 from O1, else SH at dir = (mu - C)/|mu - C|.
void colour_of(const Scene& S, int64_t i, int dr, const Cam& cam, double out[3]) {
  const int K = (S.d + 1) * (S.d + 1);
  const float* f = &S.sh[(size_t)i * K * 3];
  double Y[16];
  if (dr == 0) {
    Y[0] = SH_C0;
  } else {
    // camera centre C = -R^T t
    double C[3];
    for (int k = 0; k < 3; ++k)
      C[k] = -(cam.R[0][k] * cam.t[0] + cam.R[1][k] * cam.t[1] + cam.R[2][k] * cam.t[2]);
    double dx = S.means[i * 3 + 0] - C[0], dy = S.means[i * 3 + 1] - C[1], dz = S.means[i * 3 + 2] - C[2];
    double nn = std::sqrt(dx * dx + dy * dy + dz * dz);
    sh_basis(dr, dx / nn, dy / nn, dz / nn, Y);
  }
  const int Kr = (dr + 1) * (dr + 1);
  for (int ch = 0; ch < 3; ++ch) {
    double s = 0;
    for (int k = 0; k < Kr; ++k) s += Y[k] * (double)f[k * 3 + ch];
    s += 0.5;
    out[ch] = std::min(1.0, std::max(0.0, s));
  }
}

struct Item {           // O3 list element
  int t;
  uint32_t zbits;
  int gid;
};

struct Result {
  int W = 0, H = 0, TX = 0, TY = 0;
  int64_t n = 0;
  std::vector<double> rgb, depth, alpha;
  std::vector<int32_t> n_eval, n_contrib;
  std::vector<uint8_t> exempt, rgb8;
  std::vector<int32_t> tile_counts;
  std::vector<int32_t> s_tile, s_gid;
  std::vector<uint32_t> s_zbits;
  std::vector<int32_t> ranges;
  std::vector<float> proj;     // [n*16]
};

enum { F_NO_EARLY_OUT = 1, F_UNTRUNCATED = 2, F_PLAIN = 4, F_TIGHT = 8, F_ELLIPSE = 16, F_INTEGER_ONLY = 32 };

// O4 + O5 for one pixel over an ordered sequence of records.
struct PixelOut {
  double rgb[3], depth, alpha;
  int32_t n_eval, n_contrib;
  bool exempt;
};

// Near-miss flags (reading R28).  The definition is evaluated here
// in f64; an f32 renderer evaluates the same records with rounding, so a
// pixel is flagged ("exempt" candidate) when one of its decisions lies within
// an f32 error bound of its threshold:
//   cutoff  |alpha 255 - 1| < max(1e-4, da),
//   stop    |T' / 1e-4 - 1| < max(1e-4, dT'),
// da = relative error bound of an f32 alpha = ln2 e_x + 2^-21 (ex2 rounding),
// e_x = 2^-21 M the f32 exponent's absolute error, M = the magnitude of the
// exponent's terms expanded about the pixel's tile origin (the form a tiled
// renderer evaluates: (log2 e / 2)(|A| + 2|B| + |C|)(max(|Dx|, |Dy|) + 16)^2
// + |log2 o|, D = mean - the tile's first pixel centre); dT' = the relative
// error bound of an f32 T' = sum over the blended pairs so far (and this one)
// of alpha/(1 - alpha) da + 2^-22 per step (dT/T = sum dalpha/(1 - alpha)).
// The flags mark candidates only; tests/parity.py caps the failures.
template <typename Seq>
PixelOut composite(const Seq& seq, const std::vector<Proj>& P, int px, int py, const double bg[3],
                   int flags) {
  const double cxp = px + 0.5, cyp = py + 0.5;     // pixel centre (reading R1)
  const double tox = TILE * (px / TILE) + 0.5, toy = TILE * (py / TILE) + 0.5;   // tile origin (flags only)
  const double HALF_LOG2E = 0.72134752044448170, LN2 = 0.69314718055994531;
  double T = 1.0, C[3] = {0, 0, 0}, Dn = 0.0, A = 0.0;
  double relT = 0.0;                               // f32 error bound of T, relative (flags only)
  int32_t ne = 0, nc = 0;
  bool ex = false;
  for (int gid : seq) {
    const Proj& g = P[gid];
    ++ne;
    const double dx = g.u - cxp, dy = g.v - cyp;
    double q = g.A * dx * dx + 2.0 * g.B * dx * dy + g.C * dy * dy;
    q = std::max(q, 0.0);                                 // reading R13
    const double alpha = std::min(0.99, g.o * std::exp(-0.5 * q));
    double dal = 1e-4;
    if (g.o > 0.0) {
      const double m = std::max(std::fabs(g.u - tox), std::fabs(g.v - toy)) + TILE;
      const double M = HALF_LOG2E * (std::fabs(g.A) + 2.0 * std::fabs(g.B) + std::fabs(g.C)) * m * m +
                       std::fabs(std::log2(g.o));
      dal = LN2 * (M * 0x1p-21) + 0x1p-21;
    }
    if (std::fabs(alpha * 255.0 - 1.0) < std::max(1e-4, dal)) ex = true;   // cutoff near-miss
    if (alpha < 1.0 / 255.0) continue;                       // skip (reading R11)
    const double Tn = T * (1.0 - alpha);
    const double dTn = relT + alpha / (1.0 - alpha) * dal + 0x1p-22;
    if (std::fabs(Tn / 1e-4 - 1.0) < std::max(1e-4, dTn)) ex = true;   // early-out near-miss
    if (Tn < 1e-4 && !(flags & F_NO_EARLY_OUT)) break;       // stop, i not blended (R12)
    const double w = alpha * T;
    C[0] += w * g.col[0]; C[1] += w * g.col[1]; C[2] += w * g.col[2];
    Dn += w * g.z;
    A += w;
    T = Tn;
    relT = dTn;
    ++nc;
  }
  PixelOut o;
  for (int ch = 0; ch < 3; ++ch) o.rgb[ch] = C[ch] + T * bg[ch];   // O5 (reading R15)
  o.depth = A > 0 ? Dn / A : 0.0;                                   // reading R14
  o.alpha = A;
  o.n_eval = ne; o.n_contrib = nc; o.exempt = ex;
  return o;
}

uint8_t quantize(double x) {               // O5: round-half-even(clamp(x)*255)
  x = std::min(1.0, std::max(0.0, x)) * 255.0;
  return (uint8_t)std::nearbyint(x);       // default rounding mode = to nearest even
}

}  // namespace

extern "C" {

struct OrOpts {
  float near_plane, far_plane;
  double background[3];
  int32_t sh_degree;   // -1: scene degree
  int32_t mode;        // 0 = A (f32 canonical projection), 1 = B (f64 projection)
  int32_t flags;       // F_NO_EARLY_OUT | F_UNTRUNCATED | F_PLAIN | F_TIGHT | F_ELLIPSE | F_INTEGER_ONLY
};

void* or_scene_create(int64_t n, int32_t d, const float* means, const float* scales,
                      const float* quats, const float* opac, const float* sh) {
  if (n < 0 || d < 0 || d > 3) return nullptr;
  Scene* S = new Scene();
  S->n = n; S->d = d;
  const int K = (d + 1) * (d + 1);
  S->means.assign(means, means + n * 3);
  S->scales.assign(scales, scales + n * 3);
  S->quats.assign(quats, quats + n * 4);
  S->opac.assign(opac, opac + n);
  S->sh.assign(sh, sh + n * K * 3);
  S->cov32.resize(n * 6);
  S->cov64.resize(n * 6);
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    cov3_of<float>(&S->quats[i * 4], &S->scales[i * 3], &S->cov32[i * 6]);
    cov3_of<double>(&S->quats[i * 4], &S->scales[i * 3], &S->cov64[i * 6]);
  }
  return S;
}

void or_scene_free(void* s) { delete (Scene*)s; }

void or_scene_cov3(const void* s, float* out32, double* out64) {
  const Scene* S = (const Scene*)s;
  if (out32) std::memcpy(out32, S->cov32.data(), S->cov32.size() * 4);
  if (out64) std::memcpy(out64, S->cov64.data(), S->cov64.size() * 8);
}

void or_sh_basis(int32_t d, const double* dir, double* out) { sh_basis(d, dir[0], dir[1], dir[2], out); }

void or_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
#else
  (void)n;
#endif
}

int or_num_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

void* or_render_env(const void* scene, const float* view, const float* intr, int32_t W, int32_t H,
                    const OrOpts* opt) {
  const Scene& S = *(const Scene*)scene;
  if (W <= 0 || H <= 0) return nullptr;
  // reading R29: opts.sh_degree caps the scene's degree
  const int dr = opt->sh_degree < 0 ? S.d : std::min<int>(opt->sh_degree, S.d);
  Cam cam;
  for (int i = 0; i < 3; ++i) {
    for (int j = 0; j < 3; ++j) { cam.Rf[i][j] = view[i * 4 + j]; cam.R[i][j] = view[i * 4 + j]; }
    cam.tf[i] = view[i * 4 + 3]; cam.t[i] = view[i * 4 + 3];
  }
  cam.fx = intr[0]; cam.fy = intr[1]; cam.cx = intr[2]; cam.cy = intr[3];
  cam.W = W; cam.H = H;
  cam.TX = (W + TILE - 1) / TILE; cam.TY = (H + TILE - 1) / TILE;

  Result* R = new Result();
  R->W = W; R->H = H; R->TX = cam.TX; R->TY = cam.TY; R->n = S.n;
  const int64_t n = S.n;
  std::vector<Proj> P(n);
  R->tile_counts.assign(n, 0);
  R->proj.assign(n * 16, 0.0f);

  // O1-O2 (+ colour) per Gaussian
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < n; ++i) {
    Proj& g = P[i];
    bool vis;
    if (opt->mode == 0)
      vis = project_geom<float>(&S.means[i * 3], &S.cov32[i * 6], cam, opt->near_plane, opt->far_plane, g);
    else
      vis = project_geom<double>(&S.means[i * 3], &S.cov64[i * 6], cam, (double)opt->near_plane,
                                 (double)opt->far_plane, g);
    g.vis = vis;
    if (!vis) continue;
    g.o = (double)S.opac[i];
    colour_of(S, i, dr, cam, g.col);
    if (opt->flags & (F_TIGHT | F_ELLIPSE)) tight_rect(g, S.opac[i]);
    if (opt->flags & F_ELLIPSE) ellipse_mask(g);
    {
      const int area = (g.x1 - g.x0) * (g.y1 - g.y0);
      R->tile_counts[i] = area <= 32 ? __builtin_popcount(g.mask & (area == 32 ? 0xffffffffu : ((1u << area) - 1u)))
                                     : area;
    }
    float* d = &R->proj[i * 16];
    // dump column 0: "has at least one tile"
    d[0] = R->tile_counts[i] > 0 ? 1.0f : 0.0f; d[1] = g.u32; d[2] = g.v32; d[3] = g.A32; d[4] = g.B32; d[5] = g.C32; d[6] = g.z32;
    d[7] = (float)g.r; d[8] = (float)g.x0; d[9] = (float)g.x1; d[10] = (float)g.y0; d[11] = (float)g.y1;
    d[12] = (float)g.col[0]; d[13] = (float)g.col[1]; d[14] = (float)g.col[2]; d[15] = (float)g.o;
  }

  // O3 — emission in ascending gid, tiles row-major, then sort by (t, zbits, gid)
  std::vector<Item> items;
  for (int64_t i = 0; i < n; ++i) {
    const Proj& g = P[i];
    if (!g.vis) continue;
    for (int ty = g.y0; ty < g.y1; ++ty)
      for (int tx = g.x0; tx < g.x1; ++tx)
        if (in_list(g, tx, ty)) items.push_back({ty * cam.TX + tx, g.zbits, (int)i});
  }
  std::stable_sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    if (a.t != b.t) return a.t < b.t;
    return a.zbits < b.zbits;
  });
  const int ntiles = cam.TX * cam.TY;
  R->ranges.assign(ntiles * 2, 0);
  {
    size_t k = 0;
    for (int t = 0; t < ntiles; ++t) {
      R->ranges[t * 2] = (int32_t)k;
      while (k < items.size() && items[k].t == t) ++k;
      R->ranges[t * 2 + 1] = (int32_t)k;
    }
  }
  R->s_tile.resize(items.size());
  R->s_zbits.resize(items.size());
  R->s_gid.resize(items.size());
  for (size_t k = 0; k < items.size(); ++k) {
    R->s_tile[k] = items[k].t; R->s_zbits[k] = items[k].zbits; R->s_gid[k] = items[k].gid;
  }

  // F_INTEGER_ONLY: stop after O3 (the integer artefacts); the image
  // outputs are left empty (a test-time shortcut, no arithmetic changes)
  if (opt->flags & F_INTEGER_ONLY) return R;

  // O4-O5
  const size_t npx = (size_t)W * H;
  R->rgb.assign(npx * 3, 0); R->depth.assign(npx, 0); R->alpha.assign(npx, 0);
  R->n_eval.assign(npx, 0); R->n_contrib.assign(npx, 0); R->exempt.assign(npx, 0);
  R->rgb8.assign(npx * 3, 0);
  const double* bg = opt->background;
  const int flags = opt->flags;

  // global (zbits, gid) order of visible Gaussians: used by the plain and
  // untruncated drivers
  std::vector<int> global;
  if (flags & (F_PLAIN | F_UNTRUNCATED)) {
    for (int64_t i = 0; i < n; ++i)
      if (P[i].vis) global.push_back((int)i);
    std::stable_sort(global.begin(), global.end(),
                     [&](int a, int b) { return P[a].zbits < P[b].zbits; });
  }

  auto store = [&](int px, int py, const PixelOut& o) {
    const size_t p = (size_t)py * W + px;
    for (int ch = 0; ch < 3; ++ch) { R->rgb[p * 3 + ch] = o.rgb[ch]; R->rgb8[p * 3 + ch] = quantize(o.rgb[ch]); }
    R->depth[p] = o.depth; R->alpha[p] = o.alpha;
    R->n_eval[p] = o.n_eval; R->n_contrib[p] = o.n_contrib; R->exempt[p] = o.exempt ? 1 : 0;
  };

#pragma omp parallel for schedule(dynamic, 1)
  for (int t = 0; t < ntiles; ++t) {
    const int tx = t % cam.TX, ty = t / cam.TX;
    std::vector<int> seq;
    if (flags & F_UNTRUNCATED) {
      seq = global;                              // diagnostic: no footprint truncation
    } else if (flags & F_PLAIN) {
      for (int gid : global) {
        const Proj& g = P[gid];
        if (in_list(g, tx, ty)) seq.push_back(gid);
      }
    } else {
      for (int k = R->ranges[t * 2]; k < R->ranges[t * 2 + 1]; ++k) seq.push_back(items[k].gid);
    }
    for (int py = ty * TILE; py < std::min(H, (ty + 1) * TILE); ++py)
      for (int px = tx * TILE; px < std::min(W, (tx + 1) * TILE); ++px)
        store(px, py, composite(seq, P, px, py, bg, flags));
  }
  return R;
}

// kinds for or_result_len / or_result_copy
enum {
  K_RGB = 0, K_DEPTH = 1, K_ALPHA = 2, K_NEVAL = 3, K_NCONTRIB = 4, K_EXEMPT = 5,
  K_TILE_COUNTS = 6, K_SORTED_TILE = 7, K_SORTED_ZBITS = 8, K_SORTED_GID = 9, K_RANGES = 10,
  K_PROJ = 11, K_RGB8 = 12
};

int64_t or_result_len(const void* r, int32_t kind) {
  const Result* R = (const Result*)r;
  switch (kind) {
    case K_RGB: return R->rgb.size();
    case K_DEPTH: return R->depth.size();
    case K_ALPHA: return R->alpha.size();
    case K_NEVAL: return R->n_eval.size();
    case K_NCONTRIB: return R->n_contrib.size();
    case K_EXEMPT: return R->exempt.size();
    case K_TILE_COUNTS: return R->tile_counts.size();
    case K_SORTED_TILE: return R->s_tile.size();
    case K_SORTED_ZBITS: return R->s_zbits.size();
    case K_SORTED_GID: return R->s_gid.size();
    case K_RANGES: return R->ranges.size();
    case K_PROJ: return R->proj.size();
    case K_RGB8: return R->rgb8.size();
  }
  return -1;
}

int or_result_copy(const void* r, int32_t kind, void* dst) {
  const Result* R = (const Result*)r;
  auto cp = [&](const auto& v) { std::memcpy(dst, v.data(), v.size() * sizeof(v[0])); return 0; };
  switch (kind) {
    case K_RGB: return cp(R->rgb);
    case K_DEPTH: return cp(R->depth);
    case K_ALPHA: return cp(R->alpha);
    case K_NEVAL: return cp(R->n_eval);
    case K_NCONTRIB: return cp(R->n_contrib);
    case K_EXEMPT: return cp(R->exempt);
    case K_TILE_COUNTS: return cp(R->tile_counts);
    case K_SORTED_TILE: return cp(R->s_tile);
    case K_SORTED_ZBITS: return cp(R->s_zbits);
    case K_SORTED_GID: return cp(R->s_gid);
    case K_RANGES: return cp(R->ranges);
    case K_PROJ: return cp(R->proj);
    case K_RGB8: return cp(R->rgb8);
  }
  return -1;
}

void or_result_free(void* r) { delete (Result*)r; }

}  // extern "C"
