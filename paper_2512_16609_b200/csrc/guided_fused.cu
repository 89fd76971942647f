// Image mode, wide frames: the whole guided filter + recovery in ONE pass over
// the frame with exact integer box sums (reference estimation.py:110-172,
// pipeline.py:197-215, imageops.py:39-44, recover.py:28-69).
//
// Features of a pixel (R, G, B) with m = min(R, G, B):
//   guide  g = N / 255000,  N = 299 R + 587 G + 114 B        (exact integer N)
//   coarse p = 1 - c m      (c = omega / (255 max(A)))        for m <= m*
//            = t_min                                           for m >  m* (clipped)
// where m* is the largest m the reference's clip(1 - omega (m/255)/max(A), t_min, 1)
// leaves above t_min.  Every box sum the guided filter needs is then a linear
// combination of window sums of the integers N, m, N m, N^2 (and, when some m
// clip, of the clip indicator and N on clipped pixels), which are summed EXACTLY
// in 64-bit integers, packed two fields per word where the window sums fit:
//   Q1 = N m u + (m u) << 42      Q2 = N^2 (+ (1-u) << 50)      Q3 = N (+ (N (1-u)) << 32)
// (u = [m <= m*]).  Integer arithmetic modulo 2^64 is linear, so prefix sums may
// wrap: a window difference is exact whenever the window value fits its field
// (r <= 63).  From the exact sums, var(g) and cov(g, p) come out as exact
// integer numerators (no cancellation, unlike the reference's corr - mean^2), and
//   a = cov / (var + eps),  b = mean_p - a mean_g
// are rounded once to fixed point (a_q = rint(a 2^s), exact int64 sums again).
//
// Exact sums make the result independent of summation order, so one CTA can
// own a column strip and walk its rows with sliding sums and no error growth:
//   lead  = vertical sums of the features over rows [y, y+2r] -> a, b at row y+r
//   trail = the same sums 2r+1 rows behind                     -> a, b at row y-r-1
//   A, B  = vertical sums of a_q, b_q over rows [y-r, y+r] += lead - trail
// The trail RECOMPUTES the a, b that leave the pass-2 window (bit-identical to
// what the lead computed 2r+1 rows earlier, exact sums + the same fp64 code)
// instead of storing them: nothing but the frame is read from HBM and nothing
// but the output (or, with gray-world balance, t~) is written.  Horizontal box
// sums: a per-warp exclusive prefix in shared memory (thread-local sums over 4
// columns + shuffle scan) plus the warp totals; a window spans at most two warps.
//
// Replicate borders: feature rows/columns clamp when the frame is read; a and b
// at virtual columns are the edge column's (computed from its window sums); at
// virtual rows the edge rows' a, b (kept per thread in a small global scratch).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <type_traits>

#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kFMaxWarps = 12;  // up to 384 threads (3 warps per SMSP at 168 registers), 1536 strip columns
constexpr int kFThreads = kFMaxWarps * 32;  // every CTA: 384 threads, 4 strip columns each
constexpr int kFMaxCols = kFMaxWarps * 128;

struct FusedArgs {
  const uint8_t* in;
  int64_t in_fs;
  int H, W, r;
  int ow;        // output columns per strip (multiple of 4)
  int seg_rows;  // output rows per segment
  int nstrips, nsegs;
  const double* airlight;  // [n][3] (batch-relative)
  double omega, t_min;
  double E;                // eps * (kk * 255000)^2
  double qs, rqkk;         // 2^s, 2^-s / kk
  double rkk, r255kk;      // 1/kk, 1/(255000 kk)
  uint64_t kk;
  const double* thr;
  double inv_gamma;
  int gamma_is_one;
  int pow_general;         // 1: pow_tab (inv_gamma outside the series' range)
  int gw_bf;               // k_gw_sums: branch-free series terms (DHZ_GW_BF=0 turns them off for A/B)
  double h[9];             // binomial series coefficients C(inv_gamma, k), k = 1..8
  uint8_t* out;
  int64_t out_fs;
  double* t_out;                  // MODE 1: t~ per pixel [n][H*W]
  unsigned long long* bsum;       // MODE 1: [n][3] fixed-point channel sums (2^38)
  long long* edge;                // [ctas][threads][16] a_q, b_q of rows 0 and H-1
  longlong2* ab;                  // two-pass form: (a_q, b_q) per pixel [n][H*W]
};

struct FusedShared {
  double f255[256];   // v / 255
  double2 thr2[256];  // (thr[k], thr[k+1]) output byte thresholds, thr[0] = -inf, thr[256] = +inf
  double sA[3];
  int mstar;
  };

__device__ __forceinline__ double guide_n(uint32_t N) {
  constexpr double k = 255000.0, rk = 1.0 / 255000.0;
  return div_rb(u32_to_f64(N), k, rk);
}

// The general pow, kept out of line (rare paths; inlined it bloats the hot loops).
__device__ __noinline__ double pow_general_ool(double x, double e) { return pow(x, e); }

// Tables of pow_series (gray-world sums only).
struct SeriesTables {
  double ce[1024];  // c_j^e, c_j = 1 + (j + 0.5)/1024
  double ri[1024];  // RN(1 / c_j)
  double p2[65];    // 2^(-k e)
};

__device__ __forceinline__ void series_tables_init(SeriesTables& T, double e) {
  for (int j = threadIdx.x; j < 1024; j += blockDim.x) {
    const double c = 1.0 + ((double)j + 0.5) / 1024.0;
    T.ce[j] = pow(c, e);
    T.ri[j] = __ddiv_rn(1.0, c);
  }
  for (int k = threadIdx.x; k <= 64; k += blockDim.x) T.p2[k] = exp2(-(double)k * e);
}

// x^e, x in [0, 1] (fixed e = inv_gamma): x = m 2^-k, m in [1, 2), c_j the centre of
// m's 1/1024 interval, m^e = c_j^e (1 + u)^e with |u| < 2^-11 and the binomial series
// to degree 4 (the u^5 term is below |C(e,5)| 2^-55: 3e-19 relative at e = 1/1.2,
// 1e-13 at e = 16).  Gray-world channel sums only (bytes never come from it).
__device__ __forceinline__ double pow_series(double x, const FusedArgs& A, const SeriesTables& S) {
  if (!(x > 0.0)) return 0.0;
  if (x >= 1.0) return 1.0;
  const long long bits = __double_as_longlong(x);
  const int k = 1023 - (int)(bits >> 52);  // x in [2^-k, 2^(1-k))
  if (k > 64) return pow_general_ool(x, A.inv_gamma);  // (never for recovered samples in practice)
  const int j = (int)((bits >> 42) & 1023);
  const double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double u = __fma_rn(m, S.ri[j], -1.0);
  double s = A.h[4];
#pragma unroll
  for (int i = 3; i >= 1; --i) s = __fma_rn(s, u, A.h[i]);
  const double pm = __fma_rn(s, u, 1.0);  // (1 + u)^e
  return __dmul_rn(__dmul_rn(S.ce[j], pm), S.p2[k]);
}

// One sample's gray-world term for the fixed-point channel sums: g = clip(x)^e with
// x = RN(v/255 - A) rt + A (rt = RN(1/t~): one FMA, within 2 ulp of the exact
// recovery, far below the 2^-38 resolution of the sums), returned as the bit pattern
// of RN(g 2^38 + 1.5 2^52), whose low bits minus kGwBias are rint(g 2^38) (no
// conversion instruction).
constexpr unsigned long long kGwBias = 0x4338000000000000ull;
__device__ __forceinline__ unsigned long long gw_term(double f255v, double Ac, double rt, const FusedArgs& A,
                                                      const SeriesTables& PT) {
  const double x = fmin(fmax(__fma_rn(__dsub_rn(f255v, Ac), rt, Ac), 0.0), 1.0);
  const double g = A.gamma_is_one ? x : (A.pow_general ? pow_general_ool(x, A.inv_gamma) : pow_series(x, A, PT));
  return (unsigned long long)__double_as_longlong(__fma_rn(g, 0x1p38, 0x1.8p52));
}

// gw_term without branches, for the streaming sums kernel (series path only: gamma != 1,
// inv_gamma <= 16).  Same operations on the same inputs as gw_term / pow_series, with the
// x <= 0 and x >= 1 exits as selects; a sample in (0, 2^-64) — pow_series hands those to
// the general pow — sets `rare`, and the caller redoes its group with gw_term.
__device__ __forceinline__ unsigned long long gw_term_bf(double f255v, double Ac, double rt, const FusedArgs& A,
                                                         const SeriesTables& S, bool& rare) {
  const double x = fmin(fmax(__fma_rn(__dsub_rn(f255v, Ac), rt, Ac), 0.0), 1.0);
  rare |= (x > 0.0) & (x < 0x1p-64);
  const long long bits = __double_as_longlong(fmax(x, 0x1p-64));  // k in [0, 64]
  const int k = 1023 - (int)(bits >> 52);
  const int j = (int)((bits >> 42) & 1023);
  const double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double u = __fma_rn(m, S.ri[j], -1.0);
  double s = A.h[4];
#pragma unroll
  for (int i = 3; i >= 1; --i) s = __fma_rn(s, u, A.h[i]);
  const double pm = __fma_rn(s, u, 1.0);
  double g = __dmul_rn(__dmul_rn(S.ce[j], pm), S.p2[k]);
  g = x >= 1.0 ? 1.0 : g;
  g = x >= 0x1p-64 ? g : 0.0;
  return (unsigned long long)__double_as_longlong(__fma_rn(g, 0x1p38, 0x1.8p52));
}

// Output byte of a recovered sample x: the k with thr[k] <= x < thr[k+1], walked from a
// guess (one 16-byte shared load when the guess is right).
__device__ __forceinline__ uint32_t quantize_pair(double x, const double2* thr2, int k) {
  double2 p = thr2[k];
  while (!(p.x <= x)) p = thr2[--k];
  while (!(x < p.y)) p = thr2[++k];
  return (uint32_t)k;
}

__device__ __forceinline__ void load_row(uint32_t (&w)[3], const uint8_t* __restrict__ frame, int64_t pitch, int Y,
                                         int x, int W, bool vec) {
  const uint8_t* row = frame + (int64_t)Y * pitch;
  if (vec) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(row + 3 * x);
    w[0] = __ldg(p);
    w[1] = __ldg(p + 1);
    w[2] = __ldg(p + 2);
  } else {
    uint32_t b[12];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int xx = min(max(x + c, 0), W - 1);
      b[3 * c] = __ldg(row + 3 * xx);
      b[3 * c + 1] = __ldg(row + 3 * xx + 1);
      b[3 * c + 2] = __ldg(row + 3 * xx + 2);
    }
#pragma unroll
    for (int q = 0; q < 3; ++q) w[q] = b[4 * q] | (b[4 * q + 1] << 8) | (b[4 * q + 2] << 16) | (b[4 * q + 3] << 24);
  }
}

// R, G, B of pixel c (0..3) of a 12-byte group
__device__ __forceinline__ void rgb_of(const uint32_t (&w)[3], int c, uint32_t& R, uint32_t& G, uint32_t& B) {
  // byte 3c + k of the little-endian 12-byte group
  const int b0 = 3 * c;
  auto byte_at = [&](int i) -> uint32_t { return (w[i >> 2] >> (8 * (i & 3))) & 255u; };
  R = byte_at(b0);
  G = byte_at(b0 + 1);
  B = byte_at(b0 + 2);
}

template <bool CLIP>
struct Feat {
  using Q3T = typename std::conditional<CLIP, uint64_t, uint32_t>::type;
  uint64_t q1[4], q2[4];
  Q3T q3[4];
};

template <bool CLIP>
__device__ __forceinline__ void features(const uint32_t (&w)[3], int mstar, Feat<CLIP>& F) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    uint32_t R, G, B;
    rgb_of(w, c, R, G, B);
    const uint32_t N = 299u * R + 587u * G + 114u * B;
    const uint32_t m = min(min(R, G), B);
    const uint64_t nn = (uint64_t)N * N;
    if (CLIP) {
      const bool u = (int)m <= mstar;
      F.q1[c] = u ? ((uint64_t)(N * m) | ((uint64_t)m << 42)) : 0ull;
      F.q2[c] = nn | (u ? 0ull : (1ull << 50));
      F.q3[c] = (typename Feat<CLIP>::Q3T)((uint64_t)N | (u ? 0ull : ((uint64_t)N << 32)));
    } else {
      F.q1[c] = (uint64_t)(N * m) | ((uint64_t)m << 42);
      F.q2[c] = nn;
      F.q3[c] = (typename Feat<CLIP>::Q3T)N;
    }
  }
}

// sums += add - sub (either may be absent)
template <bool CLIP>
__device__ __forceinline__ void accumulate(Feat<CLIP>& S, const Feat<CLIP>* add, const Feat<CLIP>* sub) {
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    if (add) {
      S.q1[c] += add->q1[c];
      S.q2[c] += add->q2[c];
      S.q3[c] += add->q3[c];
    }
    if (sub) {
      S.q1[c] -= sub->q1[c];
      S.q2[c] -= sub->q2[c];
      S.q3[c] -= sub->q3[c];
    }
  }
}

// Warp-local exclusive prefix of one word over the strip: the thread's 4 columns
// go to E[4t .. 4t+3]; lane 31 leaves the warp total in Tw[warp].
template <typename U>
__device__ __forceinline__ void scan_store(const U (&v)[4], U* __restrict__ E, U* __restrict__ Tw) {
  const int lane = threadIdx.x & 31;
  const U s1 = v[0] + v[1], s2 = s1 + v[2], s3 = s2 + v[3];
  U x = s3;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const U y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  const U o = x - s3;
  U* e = E + 4 * threadIdx.x;
  if (sizeof(U) == 4) {
    *reinterpret_cast<uint4*>(e) = make_uint4((uint32_t)o, (uint32_t)(o + v[0]), (uint32_t)(o + s1),
                                              (uint32_t)(o + s2));
  } else {
    reinterpret_cast<ulonglong2*>(e)[0] = make_ulonglong2((uint64_t)o, (uint64_t)(o + v[0]));
    reinterpret_cast<ulonglong2*>(e)[1] = make_ulonglong2((uint64_t)(o + s1), (uint64_t)(o + s2));
  }
  if (lane == 31) Tw[threadIdx.x >> 5] = x;
}

// Same as scan_store for three words at once (independent shuffle chains interleaved).
template <typename U3>
__device__ __forceinline__ void scan_store3(const uint64_t (&a)[4], const uint64_t (&b)[4], const U3 (&c)[4],
                                            uint64_t* __restrict__ Ea, uint64_t* __restrict__ Eb,
                                            U3* __restrict__ Ec, uint64_t* __restrict__ Ta, uint64_t* __restrict__ Tb,
                                            U3* __restrict__ Tc) {
  const int lane = threadIdx.x & 31;
  const uint64_t a1 = a[0] + a[1], a2 = a1 + a[2], a3 = a2 + a[3];
  const uint64_t b1 = b[0] + b[1], b2 = b1 + b[2], b3 = b2 + b[3];
  const U3 c1 = c[0] + c[1], c2 = c1 + c[2], c3 = c2 + c[3];
  uint64_t xa = a3, xb = b3;
  U3 xc = c3;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint64_t ya = __shfl_up_sync(0xffffffffu, xa, o);
    const uint64_t yb = __shfl_up_sync(0xffffffffu, xb, o);
    const U3 yc = __shfl_up_sync(0xffffffffu, xc, o);
    if (lane >= o) {
      xa += ya;
      xb += yb;
      xc += yc;
    }
  }
  const uint64_t oa = xa - a3, ob = xb - b3;
  const U3 oc = xc - c3;
  const int k = 4 * threadIdx.x;
  reinterpret_cast<ulonglong2*>(Ea + k)[0] = make_ulonglong2(oa, oa + a[0]);
  reinterpret_cast<ulonglong2*>(Ea + k)[1] = make_ulonglong2(oa + a1, oa + a2);
  reinterpret_cast<ulonglong2*>(Eb + k)[0] = make_ulonglong2(ob, ob + b[0]);
  reinterpret_cast<ulonglong2*>(Eb + k)[1] = make_ulonglong2(ob + b1, ob + b2);
  if (sizeof(U3) == 4) {
    *reinterpret_cast<uint4*>(Ec + k) = make_uint4((uint32_t)oc, (uint32_t)(oc + c[0]), (uint32_t)(oc + c1),
                                                   (uint32_t)(oc + c2));
  } else {
    reinterpret_cast<ulonglong2*>(Ec + k)[0] = make_ulonglong2((uint64_t)oc, (uint64_t)(oc + c[0]));
    reinterpret_cast<ulonglong2*>(Ec + k)[1] = make_ulonglong2((uint64_t)(oc + c1), (uint64_t)(oc + c2));
  }
  if (lane == 31) {
    Ta[threadIdx.x >> 5] = xa;
    Tb[threadIdx.x >> 5] = xb;
    Tc[threadIdx.x >> 5] = xc;
  }
}

// 4 consecutive elements starting at k, k = 4t + OFF (OFF = 0..3 at compile time)
template <typename U, int OFF>
__device__ __forceinline__ void load4(const U* __restrict__ E, int k, U (&o)[4]) {
  if (sizeof(U) == 4) {
    const uint32_t* p = reinterpret_cast<const uint32_t*>(E) + k;
    if (OFF == 0) {
      const uint4 v = *reinterpret_cast<const uint4*>(p);
      o[0] = v.x; o[1] = v.y; o[2] = v.z; o[3] = v.w;
    } else if (OFF == 2) {
      const uint2 a = *reinterpret_cast<const uint2*>(p), b = *reinterpret_cast<const uint2*>(p + 2);
      o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    } else if (OFF == 1) {
      const uint2 m = *reinterpret_cast<const uint2*>(p + 1);
      o[0] = p[0]; o[1] = m.x; o[2] = m.y; o[3] = p[3];
    } else {
      const uint2 m = *reinterpret_cast<const uint2*>(p + 1);  // k+1 = 4t+4: 8-aligned
      o[0] = p[0]; o[1] = m.x; o[2] = m.y; o[3] = p[3];
    }
  } else {
    const uint64_t* p = reinterpret_cast<const uint64_t*>(E) + k;
    if ((OFF & 1) == 0) {
      const ulonglong2 a = *reinterpret_cast<const ulonglong2*>(p), b = *reinterpret_cast<const ulonglong2*>(p + 2);
      o[0] = a.x; o[1] = a.y; o[2] = b.x; o[3] = b.y;
    } else {
      const ulonglong2 m = *reinterpret_cast<const ulonglong2*>(p + 1);
      o[0] = p[0]; o[1] = m.x; o[2] = m.y; o[3] = p[3];
    }
  }
}

// Per-thread window geometry of a box of radius r over the thread's 4 columns.
// Window sum of column c = E[hi_c] - E[lo_c] (+ Tw[warp of lo_c] when hi_c lies in the
// next warp), lo_c = src_c - r, hi_c = src_c + r + 1.  `contig`: the 4 source columns
// are the thread's own consecutive columns (lo_0 = 4t - r); otherwise (strip threads
// on a frame edge) the indices are used one by one.
struct WinGeo {
  int lo0;
  int wl0;         // warp of lo_0
  uint32_t xa, xb; // column c crosses into the next warp from warp wl0 / wl0 + 1
  uint32_t valid;  // columns whose window lies inside the strip
  bool contig;
};

__device__ __forceinline__ WinGeo win_geo(const int (&src)[4], int r, int nc) {
  WinGeo g;
  g.valid = 0;
  g.xa = g.xb = 0;
  g.contig = src[1] == src[0] + 1 && src[2] == src[0] + 2 && src[3] == src[0] + 3;
  g.lo0 = src[0] - r;
  g.wl0 = max(g.lo0, 0) >> 7;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int lo = src[c] - r, hi = src[c] + r + 1;
    if (lo >= 0 && hi <= nc - 1) {
      g.valid |= 1u << c;
      const int wl = lo >> 7, wh = hi >> 7;
      if (wh != wl) {
        if (wl == g.wl0) g.xa |= 1u << c;
        else g.xb |= 1u << c;
      }
    }
  }
  g.contig = g.contig && g.valid == 15u;
  return g;
}

template <typename U, int LOFF, int HOFF>
__device__ __forceinline__ void window4(const U* __restrict__ E, const U* __restrict__ Tw, const WinGeo& g,
                                        int s0, int s1, int s2, int s3, int r, U (&o)[4]) {
  U hi[4], lo[4];
  if (g.contig) {
    load4<U, LOFF>(E, g.lo0, lo);
    load4<U, HOFF>(E, g.lo0 + 2 * r + 1, hi);
  } else {
    const int src[4] = {s0, s1, s2, s3};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const bool v = g.valid >> c & 1;
      hi[c] = v ? E[src[c] + r + 1] : (U)0;
      lo[c] = v ? E[src[c] - r] : (U)0;
    }
  }
  const U ta = Tw[g.wl0], tb = Tw[g.wl0 + 1];  // (Tw has kFMaxWarps + 1 slots)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    U v = hi[c] - lo[c];
    if (g.xa >> c & 1) v += ta;
    if (g.xb >> c & 1) v += tb;
    o[c] = v;
  }
}

struct FrameConst {
  double cw;    // omega / (255 max A)
  double omt;   // 1 - t_min
};

// (low 64 bits of) a * b: one IMAD.WIDE.U32 + one IMAD
__device__ __forceinline__ uint64_t mul64x32(uint64_t a, uint32_t b) {
  const uint64_t lo = (uint64_t)(uint32_t)a * b;
  return lo + ((uint64_t)((uint32_t)(a >> 32) * b) << 32);
}

// 1 / d for d >= 1 (here d >= eps (kk 255000)^2): fp32 seed + two Newton steps, a fixed
// instruction sequence (deterministic; error < 2 ulp).
__device__ __forceinline__ double rcp_nr(double d) {
  float xf;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(xf) : "f"(__double2float_rn(d)));
  double x = (double)xf;
  double e = __fma_rn(-d, x, 1.0);
  x = __fma_rn(x, e, x);
  e = __fma_rn(-d, x, 1.0);
  return __fma_rn(x, e, x);
}

// a, b (fixed point) from the exact window sums.  Lead and trail call this on the
// same integers and get the same bits (explicitly rounded fp64 ops only).
template <bool CLIP>
__device__ __forceinline__ void ab_from_sums(uint64_t q1, uint64_t q2, uint64_t q3, const FusedArgs& A,
                                             const FrameConst& K, long long& aq, long long& bq) {
  const uint64_t s_gm = q1 & ((1ull << 42) - 1);
  const uint32_t s_m = (uint32_t)(q1 >> 42);
  const uint64_t s_gg = CLIP ? (q2 & ((1ull << 50) - 1)) : q2;
  const uint32_t s_g = (uint32_t)q3;
  const uint32_t kk = (uint32_t)A.kk;
  const uint64_t vn = mul64x32(s_gg, kk) - (uint64_t)s_g * s_g;                       // kk^2 255000^2 var(g)
  const long long cm = (long long)mul64x32(s_gm, kk) - (long long)((uint64_t)s_g * s_m);  // kk^2 255000 cov(g, m_u)
  double num = __dmul_rn(K.cw, __ll2double_rn(cm));
  double pn = __dmul_rn(K.cw, u32_to_f64(s_m));
  if (CLIP) {
    const uint32_t n_c = (uint32_t)(q2 >> 50), s_gc = (uint32_t)(q3 >> 32);
    const long long cc = (long long)((uint64_t)s_gc * kk) - (long long)((uint64_t)s_g * n_c);
    num = __fma_rn(K.omt, __ll2double_rn(cc), num);
    pn = __fma_rn(K.omt, u32_to_f64(n_c), pn);
  }
  // cov(g, p) = -num / (kk^2 255000);  a = cov / (var + eps) = -255000 num / (vn + E)
  const double a = __dmul_rn(__dmul_rn(-255000.0, num), rcp_nr(__dadd_rn(__ull2double_rn(vn), A.E)));
  const double mp = __dsub_rn(1.0, __dmul_rn(pn, A.rkk));
  const double mi = __dmul_rn(u32_to_f64(s_g), A.r255kk);
  const double b = __fma_rn(-a, mi, mp);
  aq = __double2ll_rn(__dmul_rn(a, A.qs));
  bq = __double2ll_rn(__dmul_rn(b, A.qs));
}

// Shared-memory layout of one CTA (dynamic part): phase A = lead (0) / trail (1)
// window-sum prefixes, phase B = the a, b column sums, the warp totals, then each
// thread's private state (trail sums, a/b column sums; SoA so a warp's accesses are
// contiguous) which would not fit the register file.
constexpr int kTw = kFMaxWarps + 1;
constexpr int kPriv = 20;  // u64 words per thread: trail q1[4] q2[4] q3[4], sa[4], sb[4]

constexpr size_t kFusedSmem = (size_t)64 * kFMaxCols + 8 * 8 * kTw + 8ull * kPriv * kFThreads;

// One segment: output rows [y0, y1) of strip `strip` of frame f.  R4 = r & 3 fixes the
// alignment of the window reads.
template <bool CLIP, int MODE, int R4>
__device__ __noinline__ void fused_segment(const FusedArgs& A, FusedShared& S, const SeriesTables& PT, unsigned char* dyn,
                                           int f, int strip,
                                           int y0, int y1, const FrameConst K, long long* __restrict__ edge,
                                           unsigned long long* __restrict__ bsum3) {
  using Q3T = typename Feat<CLIP>::Q3T;
  constexpr int LOFF = (4 - R4) & 3, HOFF = (R4 + 1) & 3;
  const int r = A.r, H = A.H, W = A.W;
  constexpr int nthr = kFThreads, nc = kFMaxCols;
  const int t = threadIdx.x;
  const int xo0 = strip * A.ow, xo1 = min(W, xo0 + A.ow);
  const int xs = (xo0 - 2 * r) & ~3;  // strip column 0 (multiple of 4, may be < 0)
  const uint8_t* frame = A.in + (int64_t)f * A.in_fs;
  const int64_t pitch = 3LL * W;
  const int xt = xs + 4 * t;  // frame column of the thread's first column
  const bool vec = xt >= 0 && xt + 3 < W && (W & 3) == 0 && ((uintptr_t)frame & 3) == 0;

  unsigned char* d = dyn;
  uint64_t* e1[2];
  uint64_t* e2[2];
  Q3T* e3[2];
  for (int s = 0; s < 2; ++s) {
    e1[s] = reinterpret_cast<uint64_t*>(d); d += 8 * nc;
    e2[s] = reinterpret_cast<uint64_t*>(d); d += 8 * nc;
    e3[s] = reinterpret_cast<Q3T*>(d); d += (CLIP ? 8 : 4) * nc;
  }
  if (!CLIP) d += 8 * nc;  // (same layout size in both modes)
  uint64_t* eA = reinterpret_cast<uint64_t*>(d); d += 8 * nc;
  uint64_t* eB = reinterpret_cast<uint64_t*>(d); d += 8 * nc;
  uint64_t* tw = reinterpret_cast<uint64_t*>(d); d += 8 * 8 * kTw;
  uint64_t* priv = reinterpret_cast<uint64_t*>(d) + t;  // word k of this thread: priv[k * nthr]
  auto P = [&](int k) -> uint64_t& { return priv[k * nthr]; };

  // a, b source columns: own column clamped to the frame (virtual columns copy the edge's)
  const int jc0 = min(max(4 * t, -xs), W - 1 - xs), jc1 = min(max(4 * t + 1, -xs), W - 1 - xs),
            jc2 = min(max(4 * t + 2, -xs), W - 1 - xs), jc3 = min(max(4 * t + 3, -xs), W - 1 - xs);
  WinGeo g1, g2;
  {
    const int jc[4] = {jc0, jc1, jc2, jc3}, jo[4] = {4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3};
    g1 = win_geo(jc, r, nc);  // pass 1 windows (a, b at the thread's columns)
    g2 = win_geo(jo, r, nc);  // pass 2 windows (box of a, b)
  }
  uint32_t outmask = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (xt + c >= xo0 && xt + c < xo1) outmask |= 1u << c;
  const bool vec_out = outmask == 15u && (W & 3) == 0 && ((uintptr_t)A.out & 3) == 0 && (A.out_fs & 3) == 0;

  Feat<CLIP> L;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    L.q1[c] = L.q2[c] = 0;
    L.q3[c] = 0;
    P(12 + c) = 0;
    P(16 + c) = 0;
  }
  int pend = 0;  // lead rows above the frame not added yet (they are row 0's a, b)
  unsigned long long bs0 = 0, bs1 = 0, bs2 = 0;

  const int ystart = y0 - 4 * r;
  const int yP = y0 - 2 * r;  // first lead a, b step
#define CL(y) min(max((y), 0), H - 1)
#define TW1(b) (tw + (3 * (b)) * kTw)
#define TW2(b) (tw + (3 * (b) + 1) * kTw)
#define TW3(b) (reinterpret_cast<Q3T*>(tw + (3 * (b) + 2) * kTw))

  uint32_t wC[3] = {0, 0, 0};
  uint32_t nE[3], nT[3] = {0, 0, 0}, nC[3] = {0, 0, 0};
  // ---- phase F: fill the lead window with rows y0-2r .. y0-1 (steps ystart .. yP-1)
  load_row(nE, frame, pitch, CL(ystart + 2 * r), xt, W, vec);
  for (int y = ystart; y < yP; ++y) {
    const uint32_t wE[3] = {nE[0], nE[1], nE[2]};
    if (y + 1 < yP) load_row(nE, frame, pitch, CL(y + 1 + 2 * r), xt, W, vec);
    Feat<CLIP> fe;
    features<CLIP>(wE, S.mstar, fe);
    accumulate<CLIP>(L, &fe, nullptr);
  }
  load_row(nE, frame, pitch, CL(yP + 2 * r), xt, W, vec);
  load_row(nC, frame, pitch, CL(yP), xt, W, vec);
  // ---- phases P (y < y0: lead only, A/B fill) and O (y >= y0: lead, trail, output)
  for (int y = yP; y < y1; ++y) {
    uint32_t wE[3], wP[3], wT[3];
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      wP[q] = wC[q];
      wE[q] = nE[q];
      wC[q] = nC[q];
      wT[q] = nT[q];
    }
    if (y + 1 < y1) {  // prefetch the next step's rows
      load_row(nE, frame, pitch, CL(y + 1 + 2 * r), xt, W, vec);
      load_row(nC, frame, pitch, CL(y + 1), xt, W, vec);
      if (y + 1 >= y0 + 2) load_row(nT, frame, pitch, CL(y + 1 - 2 * r - 2), xt, W, vec);
    }
    // feature rows: lead += E - P (P absent on the first step); trail (in smem) += P - T
    {
      Feat<CLIP> fe, fl;
      features<CLIP>(wE, S.mstar, fe);
      if (y > yP) {
        features<CLIP>(wP, S.mstar, fl);
        accumulate<CLIP>(L, &fe, &fl);
        if (y >= y0 + 2) {
          Feat<CLIP> ft;
          features<CLIP>(wT, S.mstar, ft);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            P(c) += fl.q1[c] - ft.q1[c];
            P(4 + c) += fl.q2[c] - ft.q2[c];
            P(8 + c) = (uint64_t)(Q3T)((Q3T)P(8 + c) + fl.q3[c] - ft.q3[c]);
          }
        }
      } else {
        accumulate<CLIP>(L, &fe, nullptr);
#pragma unroll
        for (int c = 0; c < 4; ++c) {  // the trail starts on the lead's first window (row y0 - r)
          P(c) = L.q1[c];
          P(4 + c) = L.q2[c];
          P(8 + c) = (uint64_t)L.q3[c];
        }
      }
    }
    const int yl = y + r, ytr = y - r - 1;
    const bool out_phase = y >= y0;
    const bool trail_on = y >= y0 + 1, trail_ab = trail_on && ytr >= 0;
    // lead buffer: 0 from y0 on (trail in 1, two barriers per step); before y0 the lead
    // alternates 0/1 (one barrier per step), ending on 1 at y0 - 1
    const int lb = out_phase ? 0 : ((y0 - y) & 1);
    // ---- phase A: horizontal prefixes of the lead / trail sums
    if (yl >= 0 && yl <= H - 1) scan_store3<Q3T>(L.q1, L.q2, L.q3, e1[lb], e2[lb], e3[lb], TW1(lb), TW2(lb), TW3(lb));
    if (trail_ab) {
      uint64_t v1[4], v2[4];
      Q3T v3[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        v1[c] = P(c);
        v2[c] = P(4 + c);
        v3[c] = (Q3T)P(8 + c);
      }
      scan_store3<Q3T>(v1, v2, v3, e1[1], e2[1], e3[1], TW1(1), TW2(1), TW3(1));
    }
    __syncthreads();
    // ---- lead a, b of row yl -> A, B column sums
    if (g1.valid) {
      long long da[4] = {0, 0, 0, 0}, db[4] = {0, 0, 0, 0};
      if (yl < 0) {
        ++pend;
      } else if (yl > H - 1) {  // below the frame: row H-1 again
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          da[c] = edge[8 + c];
          db[c] = edge[12 + c];
        }
      } else {
        uint64_t w1[4], w2[4];
        Q3T w3[4];
        window4<uint64_t, LOFF, HOFF>(e1[lb], TW1(lb), g1, jc0, jc1, jc2, jc3, r, w1);
        window4<uint64_t, LOFF, HOFF>(e2[lb], TW2(lb), g1, jc0, jc1, jc2, jc3, r, w2);
        window4<Q3T, LOFF, HOFF>(e3[lb], TW3(lb), g1, jc0, jc1, jc2, jc3, r, w3);
#pragma unroll
        for (int c = 0; c < 4; ++c) ab_from_sums<CLIP>(w1[c], w2[c], (uint64_t)w3[c], A, K, da[c], db[c]);
        if (yl == H - 1) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            edge[8 + c] = da[c];
            edge[12 + c] = db[c];
          }
        }
        if (yl == 0) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            edge[c] = da[c];
            edge[4 + c] = db[c];
            da[c] *= (long long)(pend + 1);
            db[c] *= (long long)(pend + 1);
          }
        }
      }
      // ---- trail a, b of row ytr leave the sums
      if (trail_on) {
        if (trail_ab) {
          uint64_t w1[4], w2[4];
          Q3T w3[4];
          window4<uint64_t, LOFF, HOFF>(e1[1], TW1(1), g1, jc0, jc1, jc2, jc3, r, w1);
          window4<uint64_t, LOFF, HOFF>(e2[1], TW2(1), g1, jc0, jc1, jc2, jc3, r, w2);
          window4<Q3T, LOFF, HOFF>(e3[1], TW3(1), g1, jc0, jc1, jc2, jc3, r, w3);
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            long long aq, bq;
            ab_from_sums<CLIP>(w1[c], w2[c], (uint64_t)w3[c], A, K, aq, bq);
            da[c] -= aq;
            db[c] -= bq;
          }
        } else {  // above the frame: row 0
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            da[c] -= edge[c];
            db[c] -= edge[4 + c];
          }
        }
      }
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        if (g1.valid >> c & 1) {
          P(12 + c) += (uint64_t)da[c];
          P(16 + c) += (uint64_t)db[c];
        }
      }
    } else if (yl < 0) {
      ++pend;
    }
    if (!out_phase) continue;
    // ---- phase B: box of the a, b column sums -> t~ -> row y
    {
      uint64_t v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = P(12 + c);
      scan_store<uint64_t>(v, eA, tw + 6 * kTw);
#pragma unroll
      for (int c = 0; c < 4; ++c) v[c] = P(16 + c);
      scan_store<uint64_t>(v, eB, tw + 7 * kTw);
    }
    __syncthreads();
    if (!outmask) continue;
    uint64_t ba[4], bb[4];
    window4<uint64_t, LOFF, HOFF>(eA, tw + 6 * kTw, g2, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, ba);
    window4<uint64_t, LOFF, HOFF>(eB, tw + 7 * kTw, g2, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, bb);
    const double A0 = S.sA[0], A1 = S.sA[1], A2 = S.sA[2];
    uint32_t ob[12];
    const int64_t pix0 = (int64_t)y * W + xt;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ob[3 * c] = ob[3 * c + 1] = ob[3 * c + 2] = 0;
      if (!(outmask >> c & 1)) continue;
      uint32_t R, G, B;
      rgb_of(wC, c, R, G, B);
      const double mab = __dmul_rn(__ll2double_rn((long long)ba[c]), A.rqkk);
      const double mbb = __dmul_rn(__ll2double_rn((long long)bb[c]), A.rqkk);
      const double gg = guide_n(299u * R + 587u * G + 114u * B);
      // q = box(a) g + box(b); clip(q, 0, 1) then max(., t_min) == clip(q, t_min, 1)
      const double tt = fmin(fmax(__dadd_rn(__dmul_rn(mab, gg), mbb), A.t_min), 1.0);
      const double rt = __drcp_rn(tt);
      const double x0 = recover_raw(S.f255[R], A0, tt, rt), x1 = recover_raw(S.f255[G], A1, tt, rt),
                   x2 = recover_raw(S.f255[B], A2, tt, rt);
      if (MODE == 0) {
        const float ig = (float)A.inv_gamma;
        ob[3 * c] = quantize_pair(x0, S.thr2, guess_byte(x0, ig, 1.0f));
        ob[3 * c + 1] = quantize_pair(x1, S.thr2, guess_byte(x1, ig, 1.0f));
        ob[3 * c + 2] = quantize_pair(x2, S.thr2, guess_byte(x2, ig, 1.0f));
      } else {
        A.t_out[(int64_t)f * H * W + pix0 + c] = tt;
        bs0 += gw_term(S.f255[R], A0, rt, A, PT) - kGwBias;
        bs1 += gw_term(S.f255[G], A1, rt, A, PT) - kGwBias;
        bs2 += gw_term(S.f255[B], A2, rt, A, PT) - kGwBias;
      }
    }
    if (MODE == 0) {
      uint8_t* orow = A.out + (int64_t)f * A.out_fs + pix0 * 3;
      if (vec_out) {
        uint32_t* o32 = reinterpret_cast<uint32_t*>(orow);
        o32[0] = ob[0] | (ob[1] << 8) | (ob[2] << 16) | (ob[3] << 24);
        o32[1] = ob[4] | (ob[5] << 8) | (ob[6] << 16) | (ob[7] << 24);
        o32[2] = ob[8] | (ob[9] << 8) | (ob[10] << 16) | (ob[11] << 24);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (outmask >> c & 1) {
            orow[3 * c] = (uint8_t)ob[3 * c];
            orow[3 * c + 1] = (uint8_t)ob[3 * c + 1];
            orow[3 * c + 2] = (uint8_t)ob[3 * c + 2];
          }
      }
    }
  }
#undef CL
#undef TW1
#undef TW2
#undef TW3
  if (MODE == 1) {  // per-frame channel sums (integer: order-free)
    unsigned long long v[3] = {bs0, bs1, bs2};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[ch] += __shfl_xor_sync(0xffffffffu, v[ch], o);
      if ((threadIdx.x & 31) == 0 && v[ch]) atomicAdd(&bsum3[ch], v[ch]);
    }
  }
}

// Persistent CTAs over the flat list of (frame, strip) columns x rows: CTA i takes
// rows [i*total/P, (i+1)*total/P) of the concatenated columns, i.e. one or a few
// segments, each with its own 4r-row warm-up.  Every CTA gets the same number of
// output rows, so no wave tail; results do not depend on the split (exact sums).
template <int MODE>
__global__ void __maxnreg__(168) k_gf_fused(FusedArgs A, int nframes) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ FusedShared S;
  __shared__ SeriesTables PT;
  const double e = A.inv_gamma;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    S.f255[v] = __ddiv_rn((double)v, 255.0);
    S.thr2[v] = make_double2(v == 0 ? -INFINITY : A.thr[v], v == 255 ? INFINITY : A.thr[v + 1]);
  }
  if (MODE == 1 && !A.gamma_is_one) series_tables_init(PT, e);
  const int64_t cols = (int64_t)nframes * A.nstrips;
  const int64_t total = cols * A.H;
  const int64_t b0 = total * blockIdx.x / gridDim.x, b1 = total * (blockIdx.x + 1) / gridDim.x;
  long long* edge = A.edge + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 16;
  for (int64_t b = b0; b < b1;) {
    const int64_t col = b / A.H;
    const int yseg0 = (int)(b - col * A.H);
    const int64_t end = min(b1, (col + 1) * A.H);
    const int yseg1 = yseg0 + (int)(end - b);
    b = end;
    const int f = (int)(col / A.nstrips), strip = (int)(col - (int64_t)f * A.nstrips);
    __syncthreads();  // previous segment's readers of S / the arrays are done
    const double a0 = A.airlight[3 * f], a1 = A.airlight[3 * f + 1], a2 = A.airlight[3 * f + 2];
    const double amax = fmax(fmax(a0, a1), a2);
    if (threadIdx.x == 0) {
      S.sA[0] = a0;
      S.sA[1] = a1;
      S.sA[2] = a2;
      S.mstar = -1;
    }
    __syncthreads();
    // m* = largest m the reference leaves unclipped: 1 - omega*((m/255)/max(A)) > t_min
    for (int m = threadIdx.x; m < 256; m += blockDim.x) {
      const double p = __dsub_rn(1.0, __dmul_rn(A.omega, __ddiv_rn(__ddiv_rn((double)m, 255.0), amax)));
      if (p > A.t_min) atomicMax(&S.mstar, m);
    }
    __syncthreads();
    FrameConst K;
    K.cw = __ddiv_rn(A.omega, __dmul_rn(255.0, amax));
    K.omt = __dsub_rn(1.0, A.t_min);
    const bool clip = S.mstar < 255;
#define DHZ_SEG(R4)                                                                   \
  if (clip) fused_segment<true, MODE, R4>(A, S, PT, dyn, f, strip, yseg0, yseg1, K, edge, A.bsum + 3 * f); \
  else fused_segment<false, MODE, R4>(A, S, PT, dyn, f, strip, yseg0, yseg1, K, edge, A.bsum + 3 * f);
    switch (A.r & 3) {
      case 0: DHZ_SEG(0) break;
      case 1: DHZ_SEG(1) break;
      case 2: DHZ_SEG(2) break;
      default: DHZ_SEG(3) break;
    }
#undef DHZ_SEG
  }
}

__global__ void k_bsum_to_part(const unsigned long long* __restrict__ bsum, int n, double* __restrict__ part) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < 3 * n) part[i] = __dmul_rn(__ull2double_rn(bsum[i]), 0x1p-38);
}

struct FusedPlan {
  int ow, nstrips, threads, ctas;
  size_t smem;
};

FusedPlan fused_plan(int n, int H, int W, int r, int sms) {
  FusedPlan P{};
  const int ow_max = (kFMaxCols - 4 * r - 8) & ~3;
  P.nstrips = (W + ow_max - 1) / ow_max;
  P.ow = (((W + P.nstrips - 1) / P.nstrips) + 3) & ~3;
  const int need = P.ow + 4 * r + 8;
  (void)need;
  P.threads = kFThreads;
  P.smem = kFusedSmem;
  const int64_t rows = (int64_t)n * P.nstrips * H;
  // every CTA pays a ~4r-row warm-up per segment: keep >= 8r output rows per CTA
  const int64_t by_rows = std::max<int64_t>(1, rows / std::max(64, 8 * r));
  P.ctas = (int)std::min<int64_t>(sms, by_rows);
  return P;
}


// ---------------------------------------------------------------------------
// Two-pass form of the same exact filter (the default for r <= kFusedMaxRadius).
// Pass 1 (k_gx_ab) walks a column strip with the lead window only and writes every
// pixel's fixed-point (a_q, b_q) — the very integers the one-pass kernel's lead
// produces (same exact sums, same fp64 code in ab_from_sums) — 16 B/px.  Pass 2
// (k_gx_out) walks a strip of (a_q, b_q) with vertical sliding sums (the leaving row
// is read back instead of recomputed by a trail window) and forms t~ and the output
// exactly as the one-pass kernel does, so both forms give the same bytes.  Compared
// with the one-pass kernel this drops the trail's second horizontal scan and second
// a/b evaluation (about half the instructions) and the per-thread private state in
// shared memory (more warps per SM), for 16 B/px written and 32 B/px read back.
// A pixel's a/b and output do not depend on the strip / segment / CTA split (exact
// integer sums), so the segments are long and the split is by rows of the batch.
constexpr int kXThreads = 256;            // 8 warps, 4 strip columns per thread
constexpr int kXCols = 4 * kXThreads;     // strip columns (prefix window <= 2r+1 <= 127 < 128 per warp)
constexpr int kXTw = kXThreads / 32 + 2;  // warp-total slots (+1: a window's second warp may be past the end; +1: even, keeps 16-B alignment)

// Pass-1 shared memory: double-buffered (by row parity) prefixes of 3 words + warp totals.
constexpr size_t kXSmem1 = 2ull * (3 * 8 * kXCols + 3 * 8 * kXTw);
// Pass-2: double-buffered prefixes of the a, b column sums + warp totals, then the
// cp.async staging of the next step's entering / leaving (a_q, b_q) (2 rows x 4 columns
// x 16 B per thread, one stage: refilled right after it is consumed, so the loads have
// the rest of the step in flight and hold no registers).
constexpr size_t kXStage = 2ull * 4 * 16 * kXThreads;
constexpr size_t kXSmem2 = 2ull * (2 * 8 * kXCols + 2 * 8 * kXTw) + kXStage;

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const uint32_t sa = (uint32_t)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One Kogge-Stone step of a warp inclusive scan: x += (value of lane - o) for lanes
// >= o, as a predicated add on the shuffle's own in-range predicate (no SELs).
__device__ __forceinline__ uint64_t scan_step(uint64_t x, int o) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 l, h, xl, xh;\n\t.reg .b64 y;\n\t"
      "mov.b64 {xl, xh}, %0;\n\t"
      "shfl.sync.up.b32 l|p, xl, %1, 0, -1;\n\t"
      "shfl.sync.up.b32 h, xh, %1, 0, -1;\n\t"
      "mov.b64 y, {l, h};\n\t"
      "@p add.u64 %0, %0, y;\n\t}"
      : "+l"(x)
      : "r"(o));
  return x;
}
__device__ __forceinline__ uint32_t scan_step(uint32_t x, int o) {
  asm("{\n\t.reg .pred p;\n\t.reg .b32 y;\n\t"
      "shfl.sync.up.b32 y|p, %0, %1, 0, -1;\n\t"
      "@p add.u32 %0, %0, y;\n\t}"
      : "+r"(x)
      : "r"(o));
  return x;
}

// Warp-local exclusive prefixes of 2 or 3 words (the thread's 4 columns each) with the
// warp totals, the shuffle chains interleaved.
template <typename U3>
__device__ __forceinline__ void x_scan3(const uint64_t (&a)[4], const uint64_t (&b)[4], const U3 (&c)[4],
                                        uint64_t* __restrict__ Ea, uint64_t* __restrict__ Eb, U3* __restrict__ Ec,
                                        uint64_t* __restrict__ Ta, uint64_t* __restrict__ Tb, U3* __restrict__ Tc) {
  const int lane = threadIdx.x & 31;
  const uint64_t a1 = a[0] + a[1], a2 = a1 + a[2], a3 = a2 + a[3];
  const uint64_t b1 = b[0] + b[1], b2 = b1 + b[2], b3 = b2 + b[3];
  const U3 c1 = c[0] + c[1], c2 = c1 + c[2], c3 = c2 + c[3];
  uint64_t xa = a3, xb = b3;
  U3 xc = c3;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    xa = scan_step(xa, o);
    xb = scan_step(xb, o);
    xc = scan_step(xc, o);
  }
  const uint64_t oa = xa - a3, ob = xb - b3;
  const U3 oc = xc - c3;
  const int k = 4 * threadIdx.x;
  reinterpret_cast<ulonglong2*>(Ea + k)[0] = make_ulonglong2(oa, oa + a[0]);
  reinterpret_cast<ulonglong2*>(Ea + k)[1] = make_ulonglong2(oa + a1, oa + a2);
  reinterpret_cast<ulonglong2*>(Eb + k)[0] = make_ulonglong2(ob, ob + b[0]);
  reinterpret_cast<ulonglong2*>(Eb + k)[1] = make_ulonglong2(ob + b1, ob + b2);
  if (sizeof(U3) == 4) {
    *reinterpret_cast<uint4*>(Ec + k) = make_uint4((uint32_t)oc, (uint32_t)(oc + c[0]), (uint32_t)(oc + c1),
                                                   (uint32_t)(oc + c2));
  } else {
    reinterpret_cast<ulonglong2*>(Ec + k)[0] = make_ulonglong2((uint64_t)oc, (uint64_t)(oc + c[0]));
    reinterpret_cast<ulonglong2*>(Ec + k)[1] = make_ulonglong2((uint64_t)(oc + c1), (uint64_t)(oc + c2));
  }
  if (lane == 31) {
    Ta[threadIdx.x >> 5] = xa;
    Tb[threadIdx.x >> 5] = xb;
    Tc[threadIdx.x >> 5] = xc;
  }
}

__device__ __forceinline__ void scan_store2(const uint64_t (&a)[4], const uint64_t (&b)[4], uint64_t* __restrict__ Ea,
                                            uint64_t* __restrict__ Eb, uint64_t* __restrict__ Ta,
                                            uint64_t* __restrict__ Tb) {
  const int lane = threadIdx.x & 31;
  const uint64_t a1 = a[0] + a[1], a2 = a1 + a[2], a3 = a2 + a[3];
  const uint64_t b1 = b[0] + b[1], b2 = b1 + b[2], b3 = b2 + b[3];
  uint64_t xa = a3, xb = b3;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    xa = scan_step(xa, o);
    xb = scan_step(xb, o);
  }
  const uint64_t oa = xa - a3, ob = xb - b3;
  const int k = 4 * threadIdx.x;
  reinterpret_cast<ulonglong2*>(Ea + k)[0] = make_ulonglong2(oa, oa + a[0]);
  reinterpret_cast<ulonglong2*>(Ea + k)[1] = make_ulonglong2(oa + a1, oa + a2);
  reinterpret_cast<ulonglong2*>(Eb + k)[0] = make_ulonglong2(ob, ob + b[0]);
  reinterpret_cast<ulonglong2*>(Eb + k)[1] = make_ulonglong2(ob + b1, ob + b2);
  if (lane == 31) {
    Ta[threadIdx.x >> 5] = xa;
    Tb[threadIdx.x >> 5] = xb;
  }
}

// Per-segment frame constants of pass 1: m* (largest unclipped m) and c = omega/(255 max A).
__device__ __forceinline__ bool x_frame_setup(const FusedArgs& A, FusedShared& S, int f, FrameConst& K) {
  const double a0 = A.airlight[3 * f], a1 = A.airlight[3 * f + 1], a2 = A.airlight[3 * f + 2];
  const double amax = fmax(fmax(a0, a1), a2);
  if (threadIdx.x == 0) {
    S.sA[0] = a0;
    S.sA[1] = a1;
    S.sA[2] = a2;
    S.mstar = -1;
  }
  __syncthreads();
  for (int m = threadIdx.x; m < 256; m += blockDim.x) {
    const double p = __dsub_rn(1.0, __dmul_rn(A.omega, __ddiv_rn(__ddiv_rn((double)m, 255.0), amax)));
    if (p > A.t_min) atomicMax(&S.mstar, m);
  }
  __syncthreads();
  K.cw = __ddiv_rn(A.omega, __dmul_rn(255.0, amax));
  K.omt = __dsub_rn(1.0, A.t_min);
  return S.mstar < 255;
}

// Strip geometry shared by both passes: output columns [xo0, xo1) of the frame, strip
// column 0 at frame column xs (a multiple of 4, xs <= xo0 - r), the thread's 4 columns
// at xs + 4t.  The plan keeps xo1 - 1 + r + 1 - xs <= kXCols - 1 (every output column's
// window inside the strip's exclusive prefix).
struct XGeo {
  int xo0, xo1, xs, xt;
  uint32_t outmask;
  bool need;  // the thread holds a column some output window reads
};

__device__ __forceinline__ XGeo x_geo(const FusedArgs& A, int strip) {
  XGeo g;
  g.xo0 = strip * A.ow;
  g.xo1 = min(A.W, g.xo0 + A.ow);
  g.xs = (g.xo0 - A.r) & ~3;
  g.xt = g.xs + 4 * (int)threadIdx.x;
  g.outmask = 0;
#pragma unroll
  for (int c = 0; c < 4; ++c)
    if (g.xt + c >= g.xo0 && g.xt + c < g.xo1) g.outmask |= 1u << c;
  g.need = g.xt < g.xo1 + A.r;
  return g;
}

// Pass 1 over output rows [y0, y1) of one strip: (a_q, b_q) of every output pixel.
template <bool CLIP, int R4>
__device__ __forceinline__ void x_ab_segment(const FusedArgs& A, const FusedShared& S, unsigned char* dyn, int f,
                                          int strip, int y0, int y1, const FrameConst K) {
  using Q3T = typename Feat<CLIP>::Q3T;
  constexpr int LOFF = (4 - R4) & 3, HOFF = (R4 + 1) & 3;
  const int r = A.r, H = A.H, W = A.W;
  const int t = threadIdx.x;
  const XGeo G = x_geo(A, strip);
  const uint8_t* frame = A.in + (int64_t)f * A.in_fs;
  const int64_t pitch = 3LL * W;
  const bool vec = G.xt >= 0 && G.xt + 3 < W && (W & 3) == 0 && ((uintptr_t)frame & 3) == 0;

  // per row parity b: [e1 | e2 | e3 | warp totals (3 words)], kXBuf1 bytes
  constexpr int kXBuf1 = 3 * 8 * kXCols + 3 * 8 * kXTw;
  WinGeo g;
  {
    const int jo[4] = {4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3};
    g = win_geo(jo, r, kXCols);
  }
  const uint32_t outmask = G.outmask & g.valid;
#define CL(y) min(max((y), 0), H - 1)
  Feat<CLIP> L;
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    L.q1[c] = L.q2[c] = 0;
    L.q3[c] = 0;
  }
  if (G.need) {  // warm-up: rows y0-r .. y0+r, four loads in flight
    int y = y0 - r;
    for (; y + 3 <= y0 + r; y += 4) {
      uint32_t w[4][3];
#pragma unroll
      for (int u = 0; u < 4; ++u) load_row(w[u], frame, pitch, CL(y + u), G.xt, W, vec);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Feat<CLIP> fe;
        features<CLIP>(w[u], S.mstar, fe);
        accumulate<CLIP>(L, &fe, nullptr);
      }
    }
    for (; y <= y0 + r; ++y) {
      uint32_t w[3];
      load_row(w, frame, pitch, CL(y), G.xt, W, vec);
      Feat<CLIP> fe;
      features<CLIP>(w, S.mstar, fe);
      accumulate<CLIP>(L, &fe, nullptr);
    }
  }
  uint32_t nE[3] = {0, 0, 0}, nL[3] = {0, 0, 0};
  if (G.need && y0 + 1 < y1) {
    load_row(nE, frame, pitch, CL(y0 + r + 1), G.xt, W, vec);
    load_row(nL, frame, pitch, CL(y0 - r), G.xt, W, vec);
  }
  longlong2* abf = A.ab + (int64_t)f * H * W;
  for (int y = y0; y < y1; ++y) {
    const int b = y & 1;
    uint64_t* const e1 = reinterpret_cast<uint64_t*>(dyn + b * kXBuf1);
    uint64_t* const e2 = e1 + kXCols;
    Q3T* const e3 = reinterpret_cast<Q3T*>(e2 + kXCols);
    uint64_t* const tw = e2 + 2 * kXCols;
    x_scan3<Q3T>(L.q1, L.q2, L.q3, e1, e2, e3, tw, tw + kXTw, reinterpret_cast<Q3T*>(tw + 2 * kXTw));
    if (G.need && y + 1 < y1) {  // slide the window one row down while the others scan
      // The next step's rows are loaded into nE / nL right after this step's features have
      // consumed them (same registers, dead by then): the loads then have the rest of the
      // step and the next scan to land.  (Loading before the features made the compiler
      // rotate two register sets with moves at the end of this block, which waited for
      // the loads there: 7 % of the kernel's stall samples on one IMAD.MOV.)
      Feat<CLIP> fe, fl;
      features<CLIP>(nE, S.mstar, fe);
      features<CLIP>(nL, S.mstar, fl);
      if (y + 2 < y1) {
        load_row(nE, frame, pitch, CL(y + r + 2), G.xt, W, vec);
        load_row(nL, frame, pitch, CL(y - r + 1), G.xt, W, vec);
      }
      accumulate<CLIP>(L, &fe, &fl);
    }
    __syncthreads();
    if (outmask) {
      uint64_t w1[4], w2[4];
      Q3T w3[4];
      window4<uint64_t, LOFF, HOFF>(e1, tw, g, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, w1);
      window4<uint64_t, LOFF, HOFF>(e2, tw + kXTw, g, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, w2);
      window4<Q3T, LOFF, HOFF>(e3, reinterpret_cast<Q3T*>(tw + 2 * kXTw), g, 4 * t, 4 * t + 1, 4 * t + 2,
                               4 * t + 3, r, w3);
      longlong2 v[4];
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        long long aq, bq;
        ab_from_sums<CLIP>(w1[c], w2[c], (uint64_t)w3[c], A, K, aq, bq);
        v[c] = make_longlong2(aq, bq);
      }
      longlong2* dst = abf + (int64_t)y * W + G.xt;
      if (outmask == 15u) {
#pragma unroll
        for (int c = 0; c < 4; ++c) dst[c] = v[c];
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (outmask >> c & 1) dst[c] = v[c];
      }
    }
  }
#undef CL
}

// Persistent CTAs over the flat (frame, strip) x rows space, as k_gf_fused.
__global__ void __launch_bounds__(kXThreads, 2) k_gx_ab(FusedArgs A, int nframes) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ FusedShared S;
  const int64_t cols = (int64_t)nframes * A.nstrips;
  const int64_t total = cols * A.H;
  const int64_t b0 = total * blockIdx.x / gridDim.x, b1 = total * (blockIdx.x + 1) / gridDim.x;
  for (int64_t b = b0; b < b1;) {
    const int64_t col = b / A.H;
    const int yseg0 = (int)(b - col * A.H);
    const int64_t end = min(b1, (col + 1) * A.H);
    const int yseg1 = yseg0 + (int)(end - b);
    b = end;
    const int f = (int)(col / A.nstrips), strip = (int)(col - (int64_t)f * A.nstrips);
    __syncthreads();  // the previous segment's readers of S / the prefixes are done
    FrameConst K;
    const bool clip = x_frame_setup(A, S, f, K);
#define DHZ_SEG(R4)                                                             \
  if (clip) x_ab_segment<true, R4>(A, S, dyn, f, strip, yseg0, yseg1, K);      \
  else x_ab_segment<false, R4>(A, S, dyn, f, strip, yseg0, yseg1, K);
    switch (A.r & 3) {
      case 0: DHZ_SEG(0) break;
      case 1: DHZ_SEG(1) break;
      case 2: DHZ_SEG(2) break;
      default: DHZ_SEG(3) break;
    }
#undef DHZ_SEG
  }
}

__device__ __forceinline__ void load_ab4(longlong2 (&v)[4], const longlong2* __restrict__ row, int xt,
                                         const int (&jc)[4], bool vec) {
  if (vec) {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = row[xt + c];
  } else {
#pragma unroll
    for (int c = 0; c < 4; ++c) v[c] = row[jc[c]];
  }
}

// fp32 fast path of the output bytes (pass 2 without balance): byte_bucket
// (dhz_common.cuh) on xf = RN_f(RN(v/255) - A) * rcp(t~) + A, the exact path otherwise.
struct XOutShared {
  ByteBuckets bk;
  float dq[3][256];     // RN_f(RN(v / 255) - A_c) of the segment's frame
  float af[3];
};

// Window sums of the thread's 4 consecutive strip columns from a per-warp exclusive
// prefix E and the warp totals Tw: column c sums E[hi0 + c] - E[lo0 + c] + Tw[cor[c]],
// cor[c] = the warp of its low end when the window crosses into the next warp, else
// the zero slot kXTw - 1 (fixed for a segment: no per-row selects).
template <typename U, int LOFF, int HOFF>
__device__ __forceinline__ void xwin4(const U* __restrict__ E, const U* __restrict__ Tw, int lo0, int hi0,
                                      const int (&cor)[4], U (&o)[4]) {
  U hi[4], lo[4];
  load4<U, LOFF>(E, lo0, lo);
  load4<U, HOFF>(E, hi0, hi);
#pragma unroll
  for (int c = 0; c < 4; ++c) o[c] = hi[c] - lo[c] + Tw[cor[c]];
}

// Pass 2 over output rows [y0, y1) of one strip: box of (a_q, b_q) -> t~ -> output.
template <int MODE, int R4>
__device__ __forceinline__ void x_out_segment(const FusedArgs& A, const FusedShared& S, const XOutShared& X,
                                              unsigned char* dyn, int f, int strip, int y0, int y1) {
  constexpr int LOFF = (4 - R4) & 3, HOFF = (R4 + 1) & 3;
  const int r = A.r, H = A.H, W = A.W;
  const int t = threadIdx.x;
  const XGeo G = x_geo(A, strip);
  const uint8_t* frame = A.in + (int64_t)f * A.in_fs;
  const int64_t pitch = 3LL * W;
  const longlong2* abf = A.ab + (int64_t)f * H * W;
  int jc[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) jc[c] = min(max(G.xt + c, 0), W - 1);
  const bool vec_ab = G.xt >= 0 && G.xt + 3 < W;

  // per row parity b: [eA | eB | warp totals (2 words)], kXBuf2 bytes; then the staging
  constexpr int kXBuf2 = 2 * 8 * kXCols + 2 * 8 * kXTw;
  WinGeo g;
  {
    const int jo[4] = {4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3};
    g = win_geo(jo, r, kXCols);
  }
  const uint32_t outmask = G.outmask & g.valid;
  const bool vec_in = outmask == 15u && (W & 3) == 0 && ((uintptr_t)frame & 3) == 0;
  const bool vec_out = outmask == 15u && (W & 3) == 0 && ((uintptr_t)A.out & 3) == 0 && (A.out_fs & 3) == 0;
  // output threads have all 4 windows inside the strip (the plan); cor[c] as above
  const int lo0 = 4 * t - r, hi0 = 4 * t + r + 1;
  int cor[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const int lo = max(lo0 + c, 0), hi = min(hi0 + c, kXCols - 1);
    cor[c] = (lo >> 7) != (hi >> 7) ? (lo >> 7) : kXTw - 1;
  }
#define CL(y) min(max((y), 0), H - 1)
  uint64_t SA[4] = {0, 0, 0, 0}, SB[4] = {0, 0, 0, 0};
  if (G.need) {
    int y = y0 - r;
    for (; y + 1 <= y0 + r; y += 2) {
      longlong2 v0[4], v1[4];
      load_ab4(v0, abf + (int64_t)CL(y) * W, G.xt, jc, vec_ab);
      load_ab4(v1, abf + (int64_t)CL(y + 1) * W, G.xt, jc, vec_ab);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        SA[c] += (uint64_t)v0[c].x + (uint64_t)v1[c].x;
        SB[c] += (uint64_t)v0[c].y + (uint64_t)v1[c].y;
      }
    }
    for (; y <= y0 + r; ++y) {
      longlong2 v0[4];
      load_ab4(v0, abf + (int64_t)CL(y) * W, G.xt, jc, vec_ab);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        SA[c] += (uint64_t)v0[c].x;
        SB[c] += (uint64_t)v0[c].y;
      }
    }
  }
  // staging slots of this thread: [row E/L][column] (16 B each), SoA over threads so a
  // warp's 16-byte accesses are contiguous
  longlong2* stg = reinterpret_cast<longlong2*>(dyn + 2 * kXBuf2) + t;
  auto stage_rows = [&](int YE, int YL) {
    if (vec_ab) {
      const longlong2* pE = abf + (int64_t)YE * W + G.xt;
      const longlong2* pL = abf + (int64_t)YL * W + G.xt;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cp_async16(stg + c * kXThreads, pE + c);
        cp_async16(stg + (4 + c) * kXThreads, pL + c);
      }
    } else {
      const longlong2* pE = abf + (int64_t)YE * W;
      const longlong2* pL = abf + (int64_t)YL * W;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        cp_async16(stg + c * kXThreads, pE + jc[c]);
        cp_async16(stg + (4 + c) * kXThreads, pL + jc[c]);
      }
    }
    cp_async_commit();
  };
  uint32_t nC[3] = {0, 0, 0};
  if (G.need && y0 + 1 < y1) stage_rows(CL(y0 + r + 1), CL(y0 - r));
  if (outmask) load_row(nC, frame, pitch, y0, G.xt, W, vec_in);
  const double A0 = S.sA[0], A1 = S.sA[1], A2 = S.sA[2];
  const float tminf = (float)A.t_min;
  unsigned long long bs0 = 0, bs1 = 0, bs2 = 0;
  uint8_t* const obase = A.out + (int64_t)f * A.out_fs;

  auto step = [&](auto Bc, int y) {
    constexpr int b = decltype(Bc)::value;
    uint64_t* const eA = reinterpret_cast<uint64_t*>(dyn + b * kXBuf2);
    uint64_t* const eB = eA + kXCols;
    uint64_t* const tw = eB + kXCols;
    scan_store2(SA, SB, eA, eB, tw, tw + kXTw);
    const uint32_t wC[3] = {nC[0], nC[1], nC[2]};
    if (G.need && y + 1 < y1) {
      cp_async_wait_all();
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const longlong2 e = stg[c * kXThreads], l = stg[(4 + c) * kXThreads];
        SA[c] += (uint64_t)e.x - (uint64_t)l.x;
        SB[c] += (uint64_t)e.y - (uint64_t)l.y;
      }
      if (y + 2 < y1) stage_rows(CL(y + r + 2), CL(y - r + 1));
      if (outmask) load_row(nC, frame, pitch, y + 1, G.xt, W, vec_in);
    }
    __syncthreads();
    if (!outmask) return;
    uint64_t ba[4], bb[4];
    if (g.contig) {
      xwin4<uint64_t, LOFF, HOFF>(eA, tw, lo0, hi0, cor, ba);
      xwin4<uint64_t, LOFF, HOFF>(eB, tw + kXTw, lo0, hi0, cor, bb);
    } else {
      window4<uint64_t, LOFF, HOFF>(eA, tw, g, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, ba);
      window4<uint64_t, LOFF, HOFF>(eB, tw + kXTw, g, 4 * t, 4 * t + 1, 4 * t + 2, 4 * t + 3, r, bb);
    }
    uint32_t ob[12];
    double tv[4];
    const int64_t pix0 = (int64_t)y * W + G.xt;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      ob[3 * c] = ob[3 * c + 1] = ob[3 * c + 2] = 0;
      tv[c] = 0.0;
      if (!(outmask >> c & 1)) continue;
      uint32_t R, Gc, B;
      rgb_of(wC, c, R, Gc, B);
      const uint32_t N = 299u * R + 587u * Gc + 114u * B;
      const double bad = __ll2double_rn((long long)ba[c]), bbd = __ll2double_rn((long long)bb[c]);
      if (MODE == 0) {
        // fast path: t~ to ~1e-15 (no exact roundings needed: every use below has a margin)
        const double tr = __dmul_rn(__fma_rn(bad, __dmul_rn(u32_to_f64(N), 1.0 / 255000.0), bbd), A.rqkk);
        const float tf = fminf(fmaxf(__double2float_rn(tr), tminf), 1.0f);
        float rtf;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rtf) : "f"(tf));
        bool ok = true;
        uint32_t k0 = byte_bucket(X.bk, __fmaf_rn(X.dq[0][R], rtf, X.af[0]), ok);
        uint32_t k1 = byte_bucket(X.bk, __fmaf_rn(X.dq[1][Gc], rtf, X.af[1]), ok);
        uint32_t k2 = byte_bucket(X.bk, __fmaf_rn(X.dq[2][B], rtf, X.af[2]), ok);
        if (!ok) {  // near a byte boundary: t~ with the exact roundings, fp64 recovery, exact thresholds
          const double tt = fmin(fmax(__dadd_rn(__dmul_rn(__dmul_rn(bad, A.rqkk), guide_n(N)), __dmul_rn(bbd, A.rqkk)),
                                      A.t_min),
                                 1.0);
          const double rt = __drcp_rn(tt);
          k0 = quantize_pair(recover_raw(S.f255[R], A0, tt, rt), S.thr2, (int)k0);
          k1 = quantize_pair(recover_raw(S.f255[Gc], A1, tt, rt), S.thr2, (int)k1);
          k2 = quantize_pair(recover_raw(S.f255[B], A2, tt, rt), S.thr2, (int)k2);
        }
        ob[3 * c] = k0;
        ob[3 * c + 1] = k1;
        ob[3 * c + 2] = k2;
      } else {
        const double tt =
            fmin(fmax(__dadd_rn(__dmul_rn(__dmul_rn(bad, A.rqkk), guide_n(N)), __dmul_rn(bbd, A.rqkk)), A.t_min), 1.0);
        tv[c] = tt;  // the gray-world sums and the bytes follow in k_gw_sums / k_gf_apply2
      }
    }
    if (MODE == 1) {  // t~ for the apply pass, 32 bytes per thread
      const int64_t ti = (int64_t)f * H * W + pix0;
      double* trow = A.t_out + ti;
      if (outmask == 15u && (ti & 1) == 0) {
        reinterpret_cast<double2*>(trow)[0] = make_double2(tv[0], tv[1]);
        reinterpret_cast<double2*>(trow)[1] = make_double2(tv[2], tv[3]);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (outmask >> c & 1) trow[c] = tv[c];
      }
    }
    if (MODE == 0) {
      uint8_t* orow = obase + pix0 * 3;
      if (vec_out) {
        uint32_t* o32 = reinterpret_cast<uint32_t*>(orow);
        o32[0] = ob[0] | (ob[1] << 8) | (ob[2] << 16) | (ob[3] << 24);
        o32[1] = ob[4] | (ob[5] << 8) | (ob[6] << 16) | (ob[7] << 24);
        o32[2] = ob[8] | (ob[9] << 8) | (ob[10] << 16) | (ob[11] << 24);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (outmask >> c & 1) {
            orow[3 * c] = (uint8_t)ob[3 * c];
            orow[3 * c + 1] = (uint8_t)ob[3 * c + 1];
            orow[3 * c + 2] = (uint8_t)ob[3 * c + 2];
          }
      }
    }
  };
  int y = y0;
  for (; y + 1 < y1; y += 2) {  // two rows per trip: the prefix buffers at fixed offsets
    step(std::integral_constant<int, 0>{}, y);
    step(std::integral_constant<int, 1>{}, y + 1);
  }
  if (y < y1) step(std::integral_constant<int, 0>{}, y);
#undef CL
}

template <int MODE>
__global__ void __launch_bounds__(kXThreads, 2) k_gx_out(FusedArgs A, int nframes) {
  extern __shared__ __align__(16) unsigned char dyn[];
  __shared__ FusedShared S;
  __shared__ XOutShared X;
  if (MODE == 0) byte_buckets_build(X.bk, A.thr);
  if (threadIdx.x < 4) {  // the zero slots of the warp totals (both words, both row parities)
    constexpr int kXBuf2 = 2 * 8 * kXCols + 2 * 8 * kXTw;
    uint64_t* tw = reinterpret_cast<uint64_t*>(dyn + (threadIdx.x >> 1) * kXBuf2) + 2 * kXCols;
    tw[(threadIdx.x & 1) * kXTw + kXTw - 1] = 0;
  }
  const double e = A.inv_gamma;
  for (int v = threadIdx.x; v < 256; v += blockDim.x) {
    S.f255[v] = __ddiv_rn((double)v, 255.0);
    S.thr2[v] = make_double2(v == 0 ? -INFINITY : A.thr[v], v == 255 ? INFINITY : A.thr[v + 1]);
  }
  const int64_t cols = (int64_t)nframes * A.nstrips;
  const int64_t total = cols * A.H;
  const int64_t b0 = total * blockIdx.x / gridDim.x, b1 = total * (blockIdx.x + 1) / gridDim.x;
  for (int64_t b = b0; b < b1;) {
    const int64_t col = b / A.H;
    const int yseg0 = (int)(b - col * A.H);
    const int64_t end = min(b1, (col + 1) * A.H);
    const int yseg1 = yseg0 + (int)(end - b);
    b = end;
    const int f = (int)(col / A.nstrips), strip = (int)(col - (int64_t)f * A.nstrips);
    __syncthreads();
    if (threadIdx.x < 3) S.sA[threadIdx.x] = A.airlight[3 * f + threadIdx.x];
    if (MODE == 0) {
      for (int i = threadIdx.x; i < 768; i += blockDim.x) {
        const int ch = i >> 8, v = i & 255;
        const double ac = A.airlight[3 * f + ch];
        X.dq[ch][v] = __double2float_rn(__dsub_rn(__ddiv_rn((double)v, 255.0), ac));
        if (v == 0) X.af[ch] = __double2float_rn(ac);
      }
    }
    __syncthreads();
    switch (A.r & 3) {
      case 0: x_out_segment<MODE, 0>(A, S, X, dyn, f, strip, yseg0, yseg1); break;
      case 1: x_out_segment<MODE, 1>(A, S, X, dyn, f, strip, yseg0, yseg1); break;
      case 2: x_out_segment<MODE, 2>(A, S, X, dyn, f, strip, yseg0, yseg1); break;
      default: x_out_segment<MODE, 3>(A, S, X, dyn, f, strip, yseg0, yseg1); break;
    }
  }
}

// A 4-pixel group's gray-world terms by the general gw_term (any gamma, partial groups,
// samples below 2^-64), out of line: the streaming loop below keeps its registers for
// the branch-free series path.
__device__ __noinline__ void gw_group_general(uint32_t w0, uint32_t w1, uint32_t w2, double t0, double t1, double t2,
                                              double t3, int np, double A0, double A1, double A2, const FusedArgs& A,
                                              const SeriesTables& PT, const double* s_f, unsigned long long& b0,
                                              unsigned long long& b1, unsigned long long& b2) {
  const uint32_t w[3] = {w0, w1, w2};
  const double t[4] = {t0, t1, t2, t3};
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    if (u >= np) break;
    uint32_t R, Gc, B;
    rgb_of(w, u, R, Gc, B);
    const double rt = __drcp_rn(t[u]);
    b0 += gw_term(s_f[R], A0, rt, A, PT) - kGwBias;
    b1 += gw_term(s_f[Gc], A1, rt, A, PT) - kGwBias;
    b2 += gw_term(s_f[B], A2, rt, A, PT) - kGwBias;
  }
}

// Gray-world channel sums of the two-pass form, a streaming pass over t~ and the frame:
// per pixel the three gw_term values (the same function as the one-pass kernel's
// inline sums, exact integer totals, so the same per-frame sums), kept out of the
// box-filter kernel whose register file and shared memory they would share.
// Persistent CTAs over the batch's 4-pixel groups, per-frame u64 totals by atomics.
__global__ void __launch_bounds__(256, 4) k_gw_sums(const __grid_constant__ FusedArgs A, int n, int64_t npx) {
  __shared__ SeriesTables PT;
  __shared__ double s_f[256];
  for (int v = threadIdx.x; v < 256; v += blockDim.x) s_f[v] = __ddiv_rn((double)v, 255.0);
  if (!A.gamma_is_one) series_tables_init(PT, A.inv_gamma);
  __syncthreads();
  const int64_t G = (npx + 3) >> 2;
  const int64_t total = (int64_t)n * G;
  const int64_t g0 = total * blockIdx.x / gridDim.x, g1 = total * (blockIdx.x + 1) / gridDim.x;
  const bool vec = (npx & 3) == 0 && (A.in_fs & 3) == 0 && ((uintptr_t)A.in & 3) == 0 &&
                   ((uintptr_t)A.t_out & 15) == 0;
  const bool series = !A.gamma_is_one && !A.pow_general && A.gw_bf;
  for (int64_t s0 = g0; s0 < g1;) {
    const int f = (int)(s0 / G);
    const int64_t s1 = min(g1, (int64_t)(f + 1) * G);
    const double A0 = A.airlight[3 * f], A1 = A.airlight[3 * f + 1], A2 = A.airlight[3 * f + 2];
    const uint8_t* fi = A.in + (int64_t)f * A.in_fs;
    const double* ft = A.t_out + (int64_t)f * npx;
    unsigned long long b0 = 0, b1 = 0, b2 = 0;
    for (int64_t g = s0 + threadIdx.x; g < s1; g += blockDim.x) {
      const int64_t p0 = (g - (int64_t)f * G) * 4;
      const int np = (int)min((int64_t)4, npx - p0);
      double t[4];
      uint32_t w[3];
      if (vec) {
        const double2 ta = *reinterpret_cast<const double2*>(ft + p0);
        const double2 tb = *reinterpret_cast<const double2*>(ft + p0 + 2);
        t[0] = ta.x; t[1] = ta.y; t[2] = tb.x; t[3] = tb.y;
        const uint32_t* q = reinterpret_cast<const uint32_t*>(fi + 3 * p0);
        w[0] = __ldg(q); w[1] = __ldg(q + 1); w[2] = __ldg(q + 2);
      } else {
        uint32_t bb[12];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t p = p0 + min(u, np - 1);
          t[u] = ft[p];
          bb[3 * u] = fi[3 * p];
          bb[3 * u + 1] = fi[3 * p + 1];
          bb[3 * u + 2] = fi[3 * p + 2];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) w[q] = bb[4 * q] | (bb[4 * q + 1] << 8) | (bb[4 * q + 2] << 16) | (bb[4 * q + 3] << 24);
      }
      if (series && np == 4) {  // whole group on the branch-free series path
        unsigned long long c0 = 0, c1 = 0, c2 = 0;
        bool rare = false;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          uint32_t R, Gc, B;
          rgb_of(w, u, R, Gc, B);
          const double rt = __drcp_rn(t[u]);
          c0 += gw_term_bf(s_f[R], A0, rt, A, PT, rare) - kGwBias;
          c1 += gw_term_bf(s_f[Gc], A1, rt, A, PT, rare) - kGwBias;
          c2 += gw_term_bf(s_f[B], A2, rt, A, PT, rare) - kGwBias;
        }
        if (!rare) {
          b0 += c0;
          b1 += c1;
          b2 += c2;
          continue;
        }
      }
      gw_group_general(w[0], w[1], w[2], t[0], t[1], t[2], t[3], np, A0, A1, A2, A, PT, s_f, b0, b1, b2);
    }
    unsigned long long v[3] = {b0, b1, b2};
#pragma unroll
    for (int ch = 0; ch < 3; ++ch) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v[ch] += __shfl_xor_sync(0xffffffffu, v[ch], o);
      if ((threadIdx.x & 31) == 0 && v[ch]) atomicAdd(&A.bsum[3 * f + ch], v[ch]);
    }
    s0 = s1;
  }
}

struct XPlan {
  int ow, nstrips, ctas;
};

XPlan x_plan(int n, int H, int W, int r, int sms) {
  XPlan P{};
  const int ow_max = (kXCols - 2 * r - 4) & ~3;
  P.nstrips = (W + ow_max - 1) / ow_max;
  P.ow = (((W + P.nstrips - 1) / P.nstrips) + 3) & ~3;
  const int64_t rows = (int64_t)n * P.nstrips * H;
  // a segment pays a (2r+1)-row warm-up (loads + adds only, ~1/4 of a row step): small
  // batches still take every SM, down to 8 output rows per CTA
  const int64_t by_rows = std::max<int64_t>(1, rows / 8);
  P.ctas = (int)std::min<int64_t>(2LL * sms, by_rows);
  return P;
}

}  // namespace

bool guided_fused_ok(int H, int W, int r) { return r >= 1 && r <= kFusedMaxRadius && W >= 1 && H >= 1; }

// Frames per chunk so t~ (fp64, balance only) stays within ~16 GB.
static int fused_chunk(int n, int H, int W, bool balance) {
  if (!balance) return n;
  const double per = 8.0 * (double)H * W;
  const int byte_cap = (int)std::max(1.0, std::min((double)n, 16.0e9 / per));
  const int chunks = (n + byte_cap - 1) / byte_cap;
  return (n + chunks - 1) / chunks;
}

static int sm_count() {
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

size_t guided_fused_ws_bytes(int n, int H, int W, int r, bool balance) {
  const int chunk = fused_chunk(n, H, W, balance);
  const FusedPlan P = fused_plan(chunk, H, W, r, 1024);  // edge scratch for the largest grid
  size_t b = (size_t)P.ctas * P.threads * 16 * 8;
  b = (b + 255) & ~(size_t)255;
  if (balance) {
    const int64_t npx = (int64_t)H * W;
    b += 8ull * npx * chunk;                                   // t~
    b += 24ull * chunk + 24ull * chunk + 3 * 256 * 8ull * chunk + 16ull * chunk + 1024;  // sums, parts, thr, gains
  }
  return b;
}

cudaError_t guided_fused_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                            const double* airlight, double omega, double t_min, const double* thr, double gamma,
                            bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st) {
  if (!guided_fused_ok(H, W, r)) return cudaErrorInvalidValue;
  const int64_t npx = (int64_t)H * W;
  const int sms = sm_count();
  const int chunk = fused_chunk(n, H, W, balance);
  FusedArgs A{};
  A.H = H;
  A.W = W;
  A.r = r;
  A.in_fs = in_fs;
  A.omega = omega;
  A.t_min = t_min;
  const uint64_t kk = (uint64_t)(2 * r + 1) * (uint64_t)(2 * r + 1);
  A.kk = kk;
  const double kn = (double)kk * 255000.0;
  A.E = eps * kn * kn;
  // |a| <= 1 / (4 sqrt(eps)) (Cauchy-Schwarz, p in [t_min, 1]); |b| <= 1 + |a|; the sum of
  // kk fixed-point values must stay below 2^62
  const double amax = 1.0 / (4.0 * std::sqrt(eps)) + 1.5;
  int s = (int)std::floor(62.0 - std::log2((double)kk) - std::log2(amax));
  s = std::max(8, std::min(s, 52));
  A.qs = std::ldexp(1.0, s);
  A.rqkk = std::ldexp(1.0, -s) / (double)kk;
  A.rkk = 1.0 / (double)kk;
  A.r255kk = 1.0 / kn;
  A.thr = thr;
  A.inv_gamma = 1.0 / gamma;
  A.gamma_is_one = gamma == 1.0 ? 1 : 0;
  A.pow_general = (A.inv_gamma > 16.0) ? 1 : 0;
  {  // binomial coefficients C(e, k)
    double c = 1.0;
    A.h[0] = 1.0;
    for (int k = 1; k <= 8; ++k) {
      c *= (A.inv_gamma - (k - 1)) / k;
      A.h[k] = c;
    }
  }
  A.out_fs = out_fs;
  uint8_t* base = static_cast<uint8_t*>(ws);
  const FusedPlan P0 = fused_plan(chunk, H, W, r, 1024);
  size_t off = ((size_t)P0.ctas * P0.threads * 16 * 8 + 255) & ~(size_t)255;
  A.edge = reinterpret_cast<long long*>(base);
  double* tmap = reinterpret_cast<double*>(base + off);
  unsigned long long* bsum = reinterpret_cast<unsigned long long*>(base + off + 8ull * npx * chunk);
  double* part = reinterpret_cast<double*>(bsum + 3 * chunk);
  double* bthr = part + 3 * chunk;
  float* gains = reinterpret_cast<float*>(bthr + 3 * 256 * chunk);
  cudaError_t e = cudaFuncSetAttribute(k_gf_fused<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)kFusedSmem);
  if (e != cudaSuccess) return e;
  e = cudaFuncSetAttribute(k_gf_fused<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kFusedSmem);
  if (e != cudaSuccess) return e;
  for (int f0 = 0; f0 < n; f0 += chunk) {
    const int c = std::min(chunk, n - f0);
    const FusedPlan P = fused_plan(c, H, W, r, sms);
    A.ow = P.ow;
    A.nstrips = P.nstrips;
    A.in = in + (int64_t)f0 * in_fs;
    A.out = out + (int64_t)f0 * out_fs;
    A.airlight = airlight + 3 * f0;
    if (!balance) {
      k_gf_fused<0><<<P.ctas, P.threads, P.smem, st>>>(A, c);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      continue;
    }
    A.t_out = tmap;
    A.bsum = bsum;
    if ((e = cudaMemsetAsync(bsum, 0, 24ull * c, st)) != cudaSuccess) return e;
    k_gf_fused<1><<<P.ctas, P.threads, P.smem, st>>>(A, c);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    k_bsum_to_part<<<(3 * c + 255) / 256, 256, 0, st>>>(bsum, c, part);
    if ((e = balance_thresholds(part, 1, c, npx, gamma, bthr, gains, st)) != cudaSuccess) return e;
    if ((e = guided_apply(A.in, in_fs, c, npx, tmap, A.airlight, bthr, gains, gamma, A.out, out_fs, st)) !=
        cudaSuccess)
      return e;
  }
  return cudaGetLastError();
}

// ---- two-pass form ----
// Frames per chunk so (a_q, b_q) (+ t~ with balance) stay within ~12 GB.
static int x_chunk(int n, int H, int W, bool balance) {
  const double per = (balance ? 24.0 : 16.0) * (double)H * W;
  const int cap = (int)std::max(1.0, std::min((double)n, 12.0e9 / per));
  const int chunks = (n + cap - 1) / cap;
  return (n + chunks - 1) / chunks;
}

size_t guided_x_ws_bytes(int n, int H, int W, int r, bool balance) {
  (void)r;
  const int chunk = x_chunk(n, H, W, balance);
  const int64_t npx = (int64_t)H * W;
  size_t b = 16ull * npx * chunk;
  if (balance)
    b += 8ull * npx * chunk + 24ull * chunk + 24ull * chunk + 3 * 256 * 8ull * chunk + 16ull * chunk + 1024;
  return b;
}

static void x_args(FusedArgs& A, int H, int W, int r, double eps, int64_t in_fs, double omega, double t_min,
                   const double* thr, double gamma, int64_t out_fs) {
  A.H = H;
  A.W = W;
  A.r = r;
  A.in_fs = in_fs;
  A.omega = omega;
  A.t_min = t_min;
  const uint64_t kk = (uint64_t)(2 * r + 1) * (uint64_t)(2 * r + 1);
  A.kk = kk;
  const double kn = (double)kk * 255000.0;
  A.E = eps * kn * kn;
  const double amax = 1.0 / (4.0 * std::sqrt(eps)) + 1.5;
  int s = (int)std::floor(62.0 - std::log2((double)kk) - std::log2(amax));
  s = std::max(8, std::min(s, 52));
  A.qs = std::ldexp(1.0, s);
  A.rqkk = std::ldexp(1.0, -s) / (double)kk;
  A.rkk = 1.0 / (double)kk;
  A.r255kk = 1.0 / kn;
  A.thr = thr;
  A.inv_gamma = 1.0 / gamma;
  A.gamma_is_one = gamma == 1.0 ? 1 : 0;
  A.pow_general = (A.inv_gamma > 16.0) ? 1 : 0;
  {
    const char* e = std::getenv("DHZ_GW_BF");
    A.gw_bf = (e && e[0] == '0') ? 0 : 1;
  }
  double c = 1.0;
  A.h[0] = 1.0;
  for (int k = 1; k <= 8; ++k) {
    c *= (A.inv_gamma - (k - 1)) / k;
    A.h[k] = c;
  }
  A.out_fs = out_fs;
}

cudaError_t guided_x_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                        const double* airlight, double omega, double t_min, const double* thr, double gamma,
                        bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st) {
  if (!guided_fused_ok(H, W, r)) return cudaErrorInvalidValue;
  const int64_t npx = (int64_t)H * W;
  const int sms = sm_count();
  const int chunk = x_chunk(n, H, W, balance);
  FusedArgs A{};
  x_args(A, H, W, r, eps, in_fs, omega, t_min, thr, gamma, out_fs);
  A.ab = static_cast<longlong2*>(ws);
  uint8_t* base = static_cast<uint8_t*>(ws) + 16ull * npx * chunk;
  double* tmap = reinterpret_cast<double*>(base);
  unsigned long long* bsum = reinterpret_cast<unsigned long long*>(base + 8ull * npx * chunk);
  double* part = reinterpret_cast<double*>(bsum + 3 * chunk);
  double* bthr = part + 3 * chunk;
  float* gains = reinterpret_cast<float*>(bthr + 3 * 256 * chunk);
  cudaError_t e;
  if ((e = cudaFuncSetAttribute(k_gx_ab, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXSmem1)) != cudaSuccess)
    return e;
  // two CTAs per SM need the largest shared-memory carveout (the default picked 164 KB)
  if ((e = cudaFuncSetAttribute(k_gx_ab, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_gx_out<0>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess ||
      (e = cudaFuncSetAttribute(k_gx_out<1>, cudaFuncAttributePreferredSharedMemoryCarveout, 100)) != cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_gx_out<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXSmem2)) !=
      cudaSuccess)
    return e;
  if ((e = cudaFuncSetAttribute(k_gx_out<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kXSmem2)) !=
      cudaSuccess)
    return e;
  for (int f0 = 0; f0 < n; f0 += chunk) {
    const int c = std::min(chunk, n - f0);
    const XPlan P = x_plan(c, H, W, r, sms);
    A.ow = P.ow;
    A.nstrips = P.nstrips;
    A.in = in + (int64_t)f0 * in_fs;
    A.out = out + (int64_t)f0 * out_fs;
    A.airlight = airlight + 3 * f0;
    k_gx_ab<<<P.ctas, kXThreads, kXSmem1, st>>>(A, c);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    if (!balance) {
      k_gx_out<0><<<P.ctas, kXThreads, kXSmem2, st>>>(A, c);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      continue;
    }
    A.t_out = tmap;
    A.bsum = bsum;
    if ((e = cudaMemsetAsync(bsum, 0, 24ull * c, st)) != cudaSuccess) return e;
    k_gx_out<1><<<P.ctas, kXThreads, kXSmem2, st>>>(A, c);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    {
      const int64_t groups = (int64_t)c * ((npx + 3) / 4);
      const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(4LL * sms, (groups + 255) / 256));
      k_gw_sums<<<grid, 256, 0, st>>>(A, c, npx);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    k_bsum_to_part<<<(3 * c + 255) / 256, 256, 0, st>>>(bsum, c, part);
    if ((e = balance_thresholds(part, 1, c, npx, gamma, bthr, gains, st)) != cudaSuccess) return e;
    if ((e = guided_apply(A.in, in_fs, c, npx, tmap, A.airlight, bthr, gains, gamma, A.out, out_fs, st)) !=
        cudaSuccess)
      return e;
  }
  return cudaGetLastError();
}

}  // namespace dhz
