// Shared device helpers for the Hazedefy B200 kernels (sm_100a only).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#ifndef __CUDACC__
#error "dhz_common.cuh is CUDA-only"
#endif

namespace dhz {

// Number of (i, m) pairs with 0 <= m <= i <= 255: the triangular LUT row size.
constexpr int kTri = 256 * 257 / 2;  // 32896

// Per-frame recovery table (K5 writes it, K6 stages it in shared memory): three
// triangular planes, entry (i, m <= i) of channel c at c*kTri + i*(i+1)/2 + m.
// (A 260-byte-pitch square layout has ~12% fewer bank conflicts but needs 196 KB,
// i.e. one CTA per SM: with or without the diagonal split of K6 it measured slower,
// since pitch-260 rows put neighbouring (i, m) entries into neighbouring banks.)
constexpr int kLutFrame = 3 * kTri;  // 98688 bytes, 16-byte multiple

// Width of the max-relative window histogram used by the fast select path.
constexpr int kWin = 16;

// K1 records the maximum of every 16-row x 32-column unit of the dark map; the
// select pass reads only the units that can hold top-K pixels.  (480: K1's tile width.)
constexpr int kBandH = 16;
constexpr int kUnitW = 32;
constexpr int kBandW = 480;

__device__ __forceinline__ uint32_t vmin4(uint32_t a, uint32_t b) { return __vminu4(a, b); }
__device__ __forceinline__ uint32_t vmax4(uint32_t a, uint32_t b) { return __vmaxu4(a, b); }

// 4 bytes starting at byte offset `sh` (0..3) of the 8-byte little-endian pair (lo, hi).
__device__ __forceinline__ uint32_t funnel_bytes(uint32_t lo, uint32_t hi, uint32_t sh) {
  return __funnelshift_r(lo, hi, sh * 8u);
}

// Channel minimum of 16 interleaved RGB pixels held in 12 little-endian words
// (48 bytes).  Returns 4 words with one cmin byte per pixel, pixel p in byte p&3
// of word p>>2.
__device__ __forceinline__ void cmin16(const uint32_t (&w)[12], uint32_t (&c)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // pixel 4q+0 -> bytes 12q..12q+2 (word 3q b0..b2)
    // pixel 4q+1 -> bytes 12q+3..12q+5 (word 3q b3, word 3q+1 b0..b1)
    // pixel 4q+2 -> bytes 12q+6..12q+8 (word 3q+1 b2..b3, word 3q+2 b0)
    // pixel 4q+3 -> bytes 12q+9..12q+11 (word 3q+2 b1..b3)
    const uint32_t a = w[3 * q], b = w[3 * q + 1], d = w[3 * q + 2];
    // R, G, B planes for the 4 pixels
    const uint32_t r = __byte_perm(__byte_perm(a, b, 0x0630), d, 0x5210);  // bytes 0,3,6 | 9
    const uint32_t g = __byte_perm(__byte_perm(a, b, 0x0741), d, 0x6210);  // bytes 1,4,7 | 10
    const uint32_t bl = __byte_perm(__byte_perm(a, b, 0x0052), d, 0x7410);  // bytes 2,5 | 8,11
    c[q] = vmin4(vmin4(r, g), bl);
  }
}

// Same split, but returning the three planes as well (recover kernel).
__device__ __forceinline__ void planes16(const uint32_t (&w)[12], uint32_t (&r)[4], uint32_t (&g)[4],
                                         uint32_t (&b)[4]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t a = w[3 * q], bb = w[3 * q + 1], d = w[3 * q + 2];
    r[q] = __byte_perm(__byte_perm(a, bb, 0x0630), d, 0x5210);
    g[q] = __byte_perm(__byte_perm(a, bb, 0x0741), d, 0x6210);
    b[q] = __byte_perm(__byte_perm(a, bb, 0x0052), d, 0x7410);
  }
}

// Inverse of planes16: interleave 4 words of R, G, B planes back to 12 words.
__device__ __forceinline__ void interleave16(const uint32_t (&r)[4], const uint32_t (&g)[4],
                                             const uint32_t (&b)[4], uint32_t (&w)[12]) {
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    // word 3q   = r0 g0 b0 r1
    // word 3q+1 = g1 b1 r2 g2
    // word 3q+2 = b2 r3 g3 b3
    const uint32_t rg = __byte_perm(r[q], g[q], 0x5140);   // r0 g0 r1 g1
    const uint32_t rg2 = __byte_perm(r[q], g[q], 0x7362);  // r2 g2 r3 g3
    w[3 * q] = __byte_perm(rg, b[q], 0x2410);               // r0 g0 b0 r1
    w[3 * q + 1] = __byte_perm(__byte_perm(rg, b[q], 0x0053), rg2, 0x5410);  // g1 b1 r2 g2
    w[3 * q + 2] = __byte_perm(b[q], rg2, 0x3762);  // b2 r3 g3 b3
  }
}

// ---- 16x2 SIMD: one pixel per 16-bit lane (VIMNMX{,3}.U16x2 are single SASS ops on
// sm_100a, whereas the 8x4 __vminu4 is emulated with ~6 LOP3/PRMT) ----
__device__ __forceinline__ uint32_t min2(uint32_t a, uint32_t b) { return __vminu2(a, b); }
__device__ __forceinline__ uint32_t min3(uint32_t a, uint32_t b, uint32_t c) { return __vimin3_u16x2(a, b, c); }
__device__ __forceinline__ uint32_t max3u(uint32_t a, uint32_t b, uint32_t c) { return __vimax3_u16x2(a, b, c); }
// pair starting one pixel later: (a.hi, b.lo)
__device__ __forceinline__ uint32_t shift1(uint32_t a, uint32_t b) { return __funnelshift_r(a, b, 16); }

// Programmatic dependent launch (PDL): a kernel launched with
// cudaLaunchAttributeProgrammaticStreamSerialization may start while its predecessor
// drains; pdl_wait() (griddepcontrol.wait) blocks until every prerequisite grid has
// completed and its memory is visible (a no-op without the attribute), so it goes
// before the first access of predecessor data.  pdl_trigger() lets the dependent grid
// launch early (its CTAs then wait in pdl_wait); results never depend on where it sits.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

__device__ __forceinline__ uint4 ldg_v4(const void* p) {
  return __ldg(reinterpret_cast<const uint4*>(p));
}

__device__ __forceinline__ void stg_cs_v4(void* p, uint4 v) {
  asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
               "r"(v.w)
               : "memory");
}

// Block-wide exclusive scan of one uint32 per thread (blockDim.x <= 1024, multiple of 32).
// `tmp` must hold 32 words.  Returns the exclusive prefix; *total gets the block sum.
__device__ __forceinline__ uint32_t block_exclusive_scan(uint32_t v, uint32_t* tmp, uint32_t* total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) tmp[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t s = lane < nw ? tmp[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < nw) tmp[lane] = s;  // inclusive per-warp totals
  }
  __syncthreads();
  const uint32_t warp_base = wid ? tmp[wid - 1] : 0u;
  if (total) *total = tmp[nw - 1];
  const uint32_t excl = warp_base + x - v;
  __syncthreads();
  return excl;
}

// Quantisation of a recovered sample x in [0, 1] to the reference's output byte.
// thr[k] (k = 1..255) is the smallest double x with q(x) >= k for the composite
// x -> floor(clip(x ** (1/gamma)) * 255 + 0.5) evaluated by the host numpy
// (see paper_2512_16609_b200/quant.py); thr[0] is unused.  q = #{k >= 1 : thr[k] <= x}.
__device__ __forceinline__ int quantize_thr(double x, const double* __restrict__ thr) {
  int lo = 0;  // invariant: thr[lo] <= x  (thr[0] treated as -inf)
#pragma unroll
  for (int step = 128; step >= 1; step >>= 1) {
    const int c = lo + step;
    if (c <= 255 && thr[c] <= x) lo = c;
  }
  return lo;
}

// Same result as quantize_thr for ANY start level k (walks up/down the monotone
// thresholds); a good guess makes it 1-2 shared loads instead of 8.
__device__ __forceinline__ int quantize_thr_from(double x, const double* __restrict__ thr, int k) {
  while (k < 255 && thr[k + 1] <= x) ++k;
  while (k > 0 && thr[k] > x) --k;
  return k;
}

// fp32 estimate of the output byte u8(clip(x^(1/gamma) * gain)): only a start
// level for quantize_thr_from, never the answer itself.
__device__ __forceinline__ int guess_byte(double x, float inv_gamma, float gain) {
  const float g = __powf((float)x, inv_gamma) * gain;
  return __float2int_rn(fminf(fmaxf(g, 0.0f), 1.0f) * 255.0f);
}

// floor(clip(y)*255 + 0.5) with the reference's separate roundings (imageops.py:32-36).
__device__ __forceinline__ int quantize_unit(double y) {
  y = fmin(fmax(y, 0.0), 1.0);
  double z = __dadd_rn(__dmul_rn(y, 255.0), 0.5);
  return (int)floor(z);
}

// Correctly rounded a / b from rb = RN(1/b): q0 = RN(a*rb) lies within 1 ulp of
// a/b, the FMA residual a - b*q0 is exact, and one correction step rounds to
// RN(a/b) (Markstein's theorem; b is a positive normal number here).
__device__ __forceinline__ double div_rb(double a, double b, double rb) {
  const double q = __dmul_rn(a, rb);
  const double r = __fma_rn(-q, b, a);
  return __fma_rn(r, rb, q);
}

// x^e for x in [0, 1], e > 0, used only inside the gray-world channel sums, where
// per-sample errors of a few ulp (absolute < 4e-16 on [0.01, 1]) are far below the
// reference's own summation rounding; bytes are never derived from it.  Table
// driven (tables per CTA in shared memory): ln(x) = ex*ln2 + ln(c_j) +
// ln(1 + eps) with c_j the centre of x's 1/128-mantissa interval (|eps| < 2^-8,
// degree-7 series), exp(y) = 2^(k/64) * exp(r) with |r| <= ln2/128 (degree 6).
struct PowTables {
  double lnc[128];   // ln(c_j), c_j = 1 + (j + 0.5) / 128
  double rinv[128];  // RN(1 / c_j)
  double e2[64];     // 2^(j / 64)
};

__device__ __forceinline__ void pow_tables_init(PowTables& T) {
  for (int j = threadIdx.x; j < 128; j += blockDim.x) {
    const double c = 1.0 + ((double)j + 0.5) / 128.0;
    T.lnc[j] = log(c);
    T.rinv[j] = __ddiv_rn(1.0, c);
    if (j < 64) T.e2[j] = exp2((double)j / 64.0);
  }
}

// Exact u32 -> f64 on the fp64 pipe (2^52 + v has v in its low mantissa bits):
// keeps int->double conversions off the XU pipe in the hot loops.
__device__ __forceinline__ double u32_to_f64(uint32_t v) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)v), 4503599627370496.0);
}

__device__ __forceinline__ double pow_tab(double x, double e, const PowTables& T) {
  if (!(x >= 0x1p-1000)) return 0.0;  // (recovered values are 0 or far above this)
  if (x >= 1.0) return 1.0;
  const long long bits = __double_as_longlong(x);
  const int ex = (int)(bits >> 52) - 1023;                                   // x = m * 2^ex, m in [1, 2)
  const int j = (int)((bits >> 45) & 127);
  const double m = __longlong_as_double((bits & 0x000fffffffffffffLL) | 0x3ff0000000000000LL);
  const double eps = fma(m, T.rinv[j], -1.0);
  double p = 1.0 / 7;
  p = fma(p, eps, -1.0 / 6); p = fma(p, eps, 1.0 / 5); p = fma(p, eps, -1.0 / 4);
  p = fma(p, eps, 1.0 / 3);  p = fma(p, eps, -0.5);    p = fma(p, eps, 1.0);
  constexpr double kLn2Hi = 6.93147180369123816490e-01, kLn2Lo = 1.90821492927058770002e-10;
  const double exd = __dsub_rn(u32_to_f64((uint32_t)(ex + 2048)), 2048.0);  // (double)ex, off the XU pipe
  const double y = e * fma(exd, kLn2Hi, fma(exd, kLn2Lo, T.lnc[j] + p * eps));  // e ln x <= 0
  if (y < -700.0) return 0.0;
  constexpr double kL64Hi = 0x1.62e42fefa0000p-7, kL64Lo = 2.572804622327669e-14;  // ln2/64 = hi + lo
  // k = rint(y * 64/ln2) and its int by the 1.5 * 2^52 trick (round to nearest even,
  // like rint; no XU conversions)
  const double kt = __dadd_rn(__dmul_rn(y, 92.332482616893656), 6755399441055744.0);
  const double k = __dsub_rn(kt, 6755399441055744.0);
  const double r = fma(-k, kL64Lo, fma(-k, kL64Hi, y));
  double q = 1.0 / 720;
  q = fma(q, r, 1.0 / 120); q = fma(q, r, 1.0 / 24); q = fma(q, r, 1.0 / 6);
  q = fma(q, r, 0.5);       q = fma(q, r, 1.0);      q = fma(q, r, 1.0);
  const int ki = __double2loint(kt);
  return q * T.e2[ki & 63] * __longlong_as_double((long long)((ki >> 6) + 1023) << 52);
}

// ---- fp32 fast path of an output byte ----------------------------------------------
// The exact byte of a recovered sample x is #{k >= 1 : thr[k] <= x} (thr[1..255], from
// the host's np.power, quant.py, or per frame with gray-world gains).  A caller forms xf,
// the same x in fp32 (|xf - x| < 4.6e-7 wherever |x - A| <= 1, i.e. wherever a window's
// finite edge lies: one FMA of a float copy of t~'s approximate reciprocal (rel. error
// < 2^-22) and RN_f(RN(v - A)) (rel. 2^-24)), and looks it up in a bucket table:
// buckets of width 1/1024 over [0, 1) plus one for x >= 1; bucket j starts at byte
// k0 = #{k : thr[k] <= j/1024} and holds the acceptance windows of k0 and k0 + 1
// (threshold +- kByteMargin, float edges rounded inwards).  A sample outside both
// windows (near a threshold, or in a bucket holding two thresholds — gamma = 1.2 has
// none: its byte windows are wider than 1/1024) goes to the caller's exact fp64 path.
constexpr int kByteBuckets = 1024;
constexpr double kByteMargin = 1e-6;
// One 8-byte entry per bucket (a single 64-bit shared-memory load per sample):
//   x = hi(k0), the end of the lower window.  Its start lo(k0) is not stored: a sample in
//       bucket j is >= j/1024, so lo(k0) <= j/1024 makes the test redundant; the rare
//       bucket whose lower threshold lies within the margin below its start gets x = NaN
//       (both windows reject, every sample of it takes the exact path);
//   y = hi(k0 + 1), the end of the upper window, moved down by < 512 ulps so that its low
//       8 bits hold k0 (smaller is conservative).
// The upper window's start is formed at lookup time as hi(k0) + kByteGap, which is never
// below lo(k0 + 1): hi(k0) >= thr - margin - ulp and the float sum rounds by at most
// another ulp (ulp <= 6e-8 below 1), so hi(k0) + 2.2e-6 >= thr + margin + 8e-8.
constexpr float kByteGap = 2.2e-6f;
struct ByteBuckets {
  float2 ent[kByteBuckets + 1];
};

// f moved down (towards -inf) until its low 8 bits equal k (k < 256)
__device__ __forceinline__ float byte_tag_down(float f, uint32_t k) {
  const uint32_t bits = __float_as_uint(f);
  if (bits & 0x80000000u) {  // negative: a larger magnitude is further down
    const uint32_t mag = bits & 0x7FFFFFFFu;
    return __uint_as_float(0x80000000u | (((mag + 256u) & ~255u) | k));
  }
  if (bits < 256u) return __uint_as_float(0x80000000u | 256u | k);  // below the smallest taggable positive
  return __uint_as_float(((bits - 256u) & ~255u) | k);
}

// Block-cooperative build from thr[0..255] (thr[0] unused; +inf = unreachable level);
// the caller synchronises before use.
__device__ __forceinline__ void byte_buckets_build(ByteBuckets& B, const double* __restrict__ thr) {
  auto lo_of = [&](int k) -> float {
    return k <= 0 ? -INFINITY : (k > 255 ? INFINITY : __double2float_ru(__dadd_rn(thr[k], kByteMargin)));
  };
  auto hi_of = [&](int k) -> float { return k >= 255 ? INFINITY : __double2float_rd(__dsub_rn(thr[k + 1], kByteMargin)); };
  for (int j = threadIdx.x; j <= kByteBuckets; j += blockDim.x) {
    const double x = (double)j * (1.0 / kByteBuckets);
    int lo = 0, hi = 255;  // largest k in [0, 255] with k == 0 or thr[k] <= x
    while (lo < hi) {
      const int mid = (lo + hi + 1) >> 1;
      if (thr[mid] <= x) lo = mid;
      else hi = mid - 1;
    }
    const bool lower_ok = (double)lo_of(lo) <= x;  // (-inf for lo == 0)
    B.ent[j] = make_float2(lower_ok ? hi_of(lo) : __uint_as_float(0x7FC00000u),
                           byte_tag_down(hi_of(lo + 1), (uint32_t)lo));
  }
}

// Byte of xf from the table; ok stays true only if xf lies inside an acceptance window.
__device__ __forceinline__ uint32_t byte_bucket(const ByteBuckets& B, float xf, bool& ok) {
  const uint32_t j = min(__float2uint_rd(xf * (float)kByteBuckets), (uint32_t)kByteBuckets);  // (negative -> 0)
  const float2 e = B.ent[j];
  const uint32_t k = __float_as_uint(e.y) & 255u;
  const bool in0 = xf < e.x, in1 = xf >= e.x + kByteGap && xf < e.y;
  ok = ok && (in0 || in1);
  return k + (in1 ? 1u : 0u);
}

// 1 / t in fp32 (rcp.approx: rel. error < 2^-22), for the fast path above.
__device__ __forceinline__ float rcp_approx(float t) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(t));
  return r;
}

// min / max of two non-NaN doubles as one compare and two selects (fmin / fmax add a
// NaN fix-up; every operand here is finite, and no -0.0 meets a +0.0 where it matters).
__device__ __forceinline__ double dmin(double a, double b) { return b < a ? b : a; }
__device__ __forceinline__ double dmax(double a, double b) { return b > a ? b : a; }

// ((x - A) / t) + A without the final clip: where the value only feeds the byte
// thresholds (x < 0 -> byte 0, x > 1 -> the byte of 1) or pow_tab (0 / 1 outside
// (0, 1)), clipping first gives the same result, so the clip is skipped there.
__device__ __forceinline__ double recover_raw(double x, double A, double t, double rt) {
  return __dadd_rn(div_rb(__dsub_rn(x, A), t, rt), A);
}


}  // namespace dhz
