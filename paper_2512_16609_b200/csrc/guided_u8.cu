// Image mode on u8 frames at native resolution: guided-filter refinement of the
// transmission map fused with recovery (reference estimation.py:144-172,
// pipeline.py:197-215, imageops.py:39-44).
//
// Inputs per frame: the u8 frame and its airlight A (from K2-K4, bit-exact).
//   p(x)   = t_coarse = clip(1 - omega * (m/255) / max(A), t_min, 1)   (256-entry table of m)
//   g(x)   = clip((0.299*R' + 0.587*G') + 0.114*B', 0, 1), R' = R/255      (exact fp64 ops)
//   mean_I, mean_p, corr_Ip, corr_II = box_r(g), box_r(p), box_r(g*p), box_r(g*g)
//   a = (corr_Ip - mean_I*mean_p) / ((corr_II - mean_I^2) + eps),  b = mean_p - a*mean_I
//   t~ = max(clip(box_r(a) * g + box_r(b), 0, 1), t_min)
//   out_c = float_to_u8(gamma(clip((I_c' - A_c) / t~ + A_c)))  [* gray-world gains]
//
// Box sums (replicate border == clamped indices, divisor (2r+1)^2 like the
// reference's SAT) run as column-strip sliding sums: a CTA of 256 threads owns
// 256*CPT input columns (CPT = 1, 2 or 4 consecutive columns per thread, from the frame width; 256*CPT-2r
// output columns) and a segment of rows; each thread keeps the vertical window
// sums of its columns in fp64 registers (add the entering row, drop the leaving
// one), and every output row takes its horizontal windows from a shared-memory
// fp64 prefix sum over the strip (thread-local sums + warp scan + warp carries).
// Pass 1 writes a, b (fp64, 16 B/px); pass 2 boxes them, forms t~ and recovers
// the output bytes directly (exact thresholds), or — with gray-world balance —
// writes t~ and per-CTA channel sums of the gamma values; the balance pass then
// derives per-frame gains and exact per-channel byte thresholds (k_gf_thresholds)
// and k_gf_apply only recovers and thresholds (no pow per pixel).
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dhz_common.cuh"
#include "dhz_internal.h"

namespace dhz {

namespace {

constexpr int kThreads = 256;  // threads per CTA

__device__ __forceinline__ double u8f(uint32_t v) { return __ddiv_rn((double)v, 255.0); }

// Per-CTA tables: exact u8 -> fp64 products used by the guide and the coarse t.
struct GuideTables {
  double wr[256], wg[256], wb[256];  // 0.299*(v/255), 0.587*(v/255), 0.114*(v/255), one rounding each
  double t[256];                     // pass 1: clip(1 - omega*((v/255)/max(A)), t_min, 1); pass 2: v/255
};

__device__ __forceinline__ void load_guide(GuideTables& T, int v, double x) {
  T.wr[v] = __dmul_rn(0.299, x);
  T.wg[v] = __dmul_rn(0.587, x);
  T.wb[v] = __dmul_rn(0.114, x);
}

// (the guide's weighted sum of non-negative terms is >= 0: its clip reduces to min(., 1))
__device__ __forceinline__ double guide_t(const GuideTables& T, uint32_t r, uint32_t g, uint32_t b) {
  return fmin(__dadd_rn(__dadd_rn(T.wr[r], T.wg[g]), T.wb[b]), 1.0);
}

// The guide as the correctly rounded (299 R + 587 G + 114 B) / 255000 (an exact
// integer numerator, one division): within a few ulp of the reference's
// 0.299*R' + 0.587*G' + 0.114*B' with its four roundings, far below the ~1e-13 at
// which the box sums already differ from the reference's SAT; 6 instead of ~20 fp64
// operations per sample (pass 1 evaluates the guide of two rows per output row).
__device__ __forceinline__ double guide_int(uint32_t r, uint32_t g, uint32_t b) {
  constexpr double k = 255000.0, rk = 1.0 / 255000.0;  // rk: RN(1/255000), a constant expression
  return div_rb(u32_to_f64(299u * r + 587u * g + 114u * b), k, rk);
}

// tot[q] (this thread's sum over its columns) -> the CTA-exclusive prefix before
// this thread (warp shuffle scan + carries of the preceding warps; one barrier).
template <int NQ>
__device__ __forceinline__ void thread_offsets(double (&tot)[NQ], double (*wt)[kThreads / 32]) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double inc[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) inc[q] = tot[q];
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) {
      const double y = __shfl_up_sync(0xffffffffu, inc[q], o);
      if (lane >= o) inc[q] = __dadd_rn(inc[q], y);
    }
  }
  if (lane == 31) {
#pragma unroll
    for (int q = 0; q < NQ; ++q) wt[q][wid] = inc[q];
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    const double ex = __shfl_up_sync(0xffffffffu, inc[q], 1);
    tot[q] = lane == 0 ? 0.0 : ex;
  }
  __syncthreads();
  // carries: every warp scans the 8 warp totals with shuffles (lanes 0..7)
#pragma unroll
  for (int q = 0; q < NQ; ++q) {
    double c = (lane < kThreads / 32) ? wt[q][lane] : 0.0;
#pragma unroll
    for (int o = 1; o < kThreads / 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, c, o);
      if (lane >= o) c = __dadd_rn(c, y);
    }
    const double base = __shfl_sync(0xffffffffu, c, (wid + 31) & 31);  // inclusive total of warps < wid
    tot[q] = wid == 0 ? tot[q] : __dadd_rn(base, tot[q]);
  }
}

// A thread's CPT consecutive prefix values, 16 bytes at a time where CPT allows (the
// destination is 16-byte aligned: prefix arrays start one double past a 16-byte
// boundary): per-double stores at a 4-double lane stride hit 4 of the 16 bank pairs.
template <int CPT>
__device__ __forceinline__ void store_cols(double* dst, const double (&v)[CPT]) {
  if (CPT % 2 == 0) {
#pragma unroll
    for (int k = 0; k < CPT; k += 2) *reinterpret_cast<double2*>(dst + k) = make_double2(v[k], v[k + 1]);
  } else {
#pragma unroll
    for (int k = 0; k < CPT; ++k) dst[k] = v[k];
  }
}

// ---------------------------------------------------------------- pass 1 ----
// a, b for every pixel of the strip x in [x0, x0 + 256*CPT - 2r), rows [y0, y0 + seg).
template <int CPT>
__global__ void __launch_bounds__(kThreads, CPT == 4 ? 3 : 4)
k_gf_pass1(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, int r, int seg, double eps,
           const double* __restrict__ airlight, double omega, double t_min, double* __restrict__ a_out,
           double* __restrict__ b_out) {
  constexpr int NC = kThreads * CPT;
  __shared__ GuideTables T;
  extern __shared__ __align__(16) double dyn_pre[];  // [2 buffers][4 sums][NC + 2] prefix rows (+1 lead)
  __shared__ double wt[2][4][kThreads / 32];
  auto pre = [&](int buf, int q) { return dyn_pre + 1 + (buf * 4 + q) * (NC + 2); };
  const int f = blockIdx.z;
  const int sw = NC - 2 * r;                     // output columns of this strip
  const int x0 = blockIdx.x * sw;                // first output column
  const int y0 = blockIdx.y * seg;
  const int y1 = min(H, y0 + seg);
  {
    const double amax = fmax(fmax(airlight[3 * f], airlight[3 * f + 1]), airlight[3 * f + 2]);
    const int v = threadIdx.x;
    const double x = u8f(v);
    load_guide(T, v, x);
    T.t[v] = fmin(fmax(__dsub_rn(1.0, __dmul_rn(omega, __ddiv_rn(x, amax))), t_min), 1.0);
  }
  if (threadIdx.x < 8) pre(threadIdx.x >> 2, threadIdx.x & 3)[0] = 0.0;
  __syncthreads();
  const uint8_t* frame = in + (int64_t)f * in_fs;
  const int64_t pitch = 3LL * W;
  int xc[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) xc[k] = 3 * min(max(x0 - r + (int)threadIdx.x * CPT + k, 0), W - 1);
  double s[4][CPT];
  auto feat = [&](int y, int k, double& g, double& p) {
    const uint8_t* px = frame + (int64_t)min(max(y, 0), H - 1) * pitch + xc[k];
    const uint32_t R = px[0], G = px[1], B = px[2];
    g = guide_int(R, G, B);
    p = T.t[min(min(R, G), B)];
  };
  // vertical window sums for output row y0: rows y0-r .. y0+r (clamped)
#pragma unroll
  for (int k = 0; k < CPT; ++k) s[0][k] = s[1][k] = s[2][k] = s[3][k] = 0.0;
  for (int d = -r; d <= r; ++d) {
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      double g, p;
      feat(y0 + d, k, g, p);
      s[0][k] = __dadd_rn(s[0][k], g);
      s[1][k] = __dadd_rn(s[1][k], p);
      s[2][k] = __dadd_rn(s[2][k], __dmul_rn(g, p));
      s[3][k] = __dadd_rn(s[3][k], __dmul_rn(g, g));
    }
  }
  const double kk = (double)(2 * r + 1) * (double)(2 * r + 1);
  const double rkk = __drcp_rn(kk);
  int buf = 0;
  for (int y = y0; y < y1; ++y, buf ^= 1) {
    if (y > y0) {
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        double g, p, g2, p2;
        feat(y + r, k, g, p);
        feat(y - r - 1, k, g2, p2);
        s[0][k] = __dsub_rn(__dadd_rn(s[0][k], g), g2);
        s[1][k] = __dsub_rn(__dadd_rn(s[1][k], p), p2);
        s[2][k] = __dsub_rn(__dadd_rn(s[2][k], __dmul_rn(g, p)), __dmul_rn(g2, p2));
        s[3][k] = __dsub_rn(__dadd_rn(s[3][k], __dmul_rn(g, g)), __dmul_rn(g2, g2));
      }
    }
    double off[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      off[q] = s[q][0];
#pragma unroll
      for (int k = 1; k < CPT; ++k) off[q] = __dadd_rn(off[q], s[q][k]);
    }
    thread_offsets<4>(off, wt[buf]);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      double run[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) run[k] = __dadd_rn(k ? run[k - 1] : off[q], s[q][k]);
      store_cols<CPT>(pre(buf, q) + threadIdx.x * CPT + 1, run);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      // output column j of the strip (interleaved over threads: conflict-free reads)
      const int j = k * kThreads + (int)threadIdx.x;
      if (j < sw && x0 + j < W) {
        // window over strip input columns [j, j + 2r] = prefix[j+2r+1] - prefix[j]
        const int hi = j + 2 * r + 1;
        const double mi = div_rb(__dsub_rn(pre(buf, 0)[hi], pre(buf, 0)[j]), kk, rkk);
        const double mp = div_rb(__dsub_rn(pre(buf, 1)[hi], pre(buf, 1)[j]), kk, rkk);
        const double cip = div_rb(__dsub_rn(pre(buf, 2)[hi], pre(buf, 2)[j]), kk, rkk);
        const double cii = div_rb(__dsub_rn(pre(buf, 3)[hi], pre(buf, 3)[j]), kk, rkk);
        const double var = __dsub_rn(cii, __dmul_rn(mi, mi));
        const double cov = __dsub_rn(cip, __dmul_rn(mi, mp));
        const double av = __ddiv_rn(cov, __dadd_rn(var, eps));
        const int64_t o = (int64_t)f * H * W + (int64_t)y * W + x0 + j;
        a_out[o] = av;
        b_out[o] = __dsub_rn(mp, __dmul_rn(av, mi));
      }
    }
    // no trailing barrier: the next row uses the other pre/wt buffers, and the
    // barrier inside its thread_offsets orders this row's reads before reuse
  }
}

// ---------------------------------------------------------------- pass 2 ----
// MODE 0: write output bytes (no balance).  MODE 1: write t~ and per-CTA channel
// sums of the gamma values (gray-world balance follows in k_gf_apply).
template <int MODE, int CPT>
__global__ void __launch_bounds__(kThreads)
k_gf_pass2(const uint8_t* __restrict__ in, int64_t in_fs, int H, int W, int r, int seg,
           const double* __restrict__ a_in,
           const double* __restrict__ b_in, const double* __restrict__ airlight, double t_min,
           const double* __restrict__ thr, double inv_gamma, int gamma_is_one, uint8_t* __restrict__ out,
           int64_t out_fs, double* __restrict__ t_out, double* __restrict__ part) {
  constexpr int NC = kThreads * CPT;
  __shared__ GuideTables T;  // wr/wg/wb for the guide; t[] holds v/255 here
  __shared__ double sA[3], s_thr[256];
  __shared__ PowTables PT;  // balance sums (MODE 1)
  extern __shared__ __align__(16) double dyn_pre[];  // [2 buffers][2 sums][NC + 2] prefix rows (+1 lead)
  __shared__ double wt[2][2][kThreads / 32];
  auto pre = [&](int buf, int q) { return dyn_pre + 1 + (buf * 2 + q) * (NC + 2); };
  const int f = blockIdx.z;
  const int sw = NC - 2 * r;
  const int x0 = blockIdx.x * sw;
  const int y0 = blockIdx.y * seg;
  const int y1 = min(H, y0 + seg);
  {
    const int v = threadIdx.x;
    const double x = u8f(v);
    load_guide(T, v, x);
    T.t[v] = x;
    s_thr[v] = thr[v];
  }
  if (threadIdx.x < 3) sA[threadIdx.x] = airlight[3 * f + threadIdx.x];
  if (threadIdx.x < 4) pre(threadIdx.x >> 1, threadIdx.x & 1)[0] = 0.0;
  if (MODE == 1) pow_tables_init(PT);
  __syncthreads();
  int xc[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) xc[k] = min(max(x0 - r + (int)threadIdx.x * CPT + k, 0), W - 1);
  const int64_t fo = (int64_t)f * H * W;
  double sa[CPT], sb[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) sa[k] = sb[k] = 0.0;
  for (int d = -r; d <= r; ++d) {
    const int64_t row = fo + (int64_t)min(max(y0 + d, 0), H - 1) * W;
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      sa[k] = __dadd_rn(sa[k], a_in[row + xc[k]]);
      sb[k] = __dadd_rn(sb[k], b_in[row + xc[k]]);
    }
  }
  const double kk = (double)(2 * r + 1) * (double)(2 * r + 1);
  const double rkk = __drcp_rn(kk);
  const uint8_t* frame = in + (int64_t)f * in_fs;
  const double A0 = sA[0], A1 = sA[1], A2 = sA[2];
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  int buf = 0;
  for (int y = y0; y < y1; ++y, buf ^= 1) {
    if (y > y0) {
      const int64_t rin = fo + (int64_t)min(y + r, H - 1) * W, rout = fo + (int64_t)max(y - r - 1, 0) * W;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        sa[k] = __dsub_rn(__dadd_rn(sa[k], a_in[rin + xc[k]]), a_in[rout + xc[k]]);
        sb[k] = __dsub_rn(__dadd_rn(sb[k], b_in[rin + xc[k]]), b_in[rout + xc[k]]);
      }
    }
    double off[2] = {sa[0], sb[0]};
#pragma unroll
    for (int k = 1; k < CPT; ++k) {
      off[0] = __dadd_rn(off[0], sa[k]);
      off[1] = __dadd_rn(off[1], sb[k]);
    }
    thread_offsets<2>(off, wt[buf]);
    {
      double ra[CPT], rb[CPT];
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        ra[k] = __dadd_rn(k ? ra[k - 1] : off[0], sa[k]);
        rb[k] = __dadd_rn(k ? rb[k - 1] : off[1], sb[k]);
      }
      store_cols<CPT>(pre(buf, 0) + threadIdx.x * CPT + 1, ra);
      store_cols<CPT>(pre(buf, 1) + threadIdx.x * CPT + 1, rb);
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < CPT; ++k) {
      const int j = k * kThreads + (int)threadIdx.x;
      if (j < sw && x0 + j < W) {
        const int hi = j + 2 * r + 1;
        const double ma = div_rb(__dsub_rn(pre(buf, 0)[hi], pre(buf, 0)[j]), kk, rkk);
        const double mb = div_rb(__dsub_rn(pre(buf, 1)[hi], pre(buf, 1)[j]), kk, rkk);
        const int64_t pix = (int64_t)y * W + x0 + j;
        const uint8_t* px = frame + pix * 3;
        const uint32_t R = px[0], G = px[1], B = px[2];
        const double g = guide_t(T, R, G, B);
        // clip(q, 0, 1) then max(., t_min) (estimation.py:172, pipeline.py:203) == clip(q, t_min, 1)
        const double t = fmin(fmax(__dadd_rn(__dmul_rn(ma, g), mb), t_min), 1.0);
        const double rt = __drcp_rn(t);
        const double x0v = recover_raw(T.t[R], A0, t, rt), x1v = recover_raw(T.t[G], A1, t, rt),
                     x2v = recover_raw(T.t[B], A2, t, rt);
        if (MODE == 0) {
          uint8_t* o = out + (int64_t)f * out_fs + pix * 3;
          const float ig = (float)inv_gamma;
          o[0] = (uint8_t)quantize_thr_from(x0v, s_thr, guess_byte(x0v, ig, 1.0f));
          o[1] = (uint8_t)quantize_thr_from(x1v, s_thr, guess_byte(x1v, ig, 1.0f));
          o[2] = (uint8_t)quantize_thr_from(x2v, s_thr, guess_byte(x2v, ig, 1.0f));
        } else {
          t_out[fo + pix] = t;
          if (gamma_is_one) {
            acc0 = __dadd_rn(acc0, fmin(fmax(x0v, 0.0), 1.0));
            acc1 = __dadd_rn(acc1, fmin(fmax(x1v, 0.0), 1.0));
            acc2 = __dadd_rn(acc2, fmin(fmax(x2v, 0.0), 1.0));
          } else {
            acc0 = __dadd_rn(acc0, pow_tab(x0v, inv_gamma, PT));
            acc1 = __dadd_rn(acc1, pow_tab(x1v, inv_gamma, PT));
            acc2 = __dadd_rn(acc2, pow_tab(x2v, inv_gamma, PT));
          }
        }
      }
    }
  }
  if (MODE == 1) {
    double v3[3] = {acc0, acc1, acc2};
#pragma unroll
    for (int o = 16; o > 0; o >>= 1)
#pragma unroll
      for (int c = 0; c < 3; ++c) v3[c] = __dadd_rn(v3[c], __shfl_xor_sync(0xffffffffu, v3[c], o));
    __syncthreads();  // pre[][] is reused as the cross-warp buffer
    double* red = dyn_pre;
    if ((threadIdx.x & 31) == 0)
      for (int c = 0; c < 3; ++c) red[c * 8 + (threadIdx.x >> 5)] = v3[c];
    __syncthreads();
    if (threadIdx.x < 3) {
      double sum = 0.0;
      for (int w = 0; w < kThreads / 32; ++w) sum = __dadd_rn(sum, red[threadIdx.x * 8 + w]);
      const int64_t cta = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
      part[((int64_t)f * gridDim.x * gridDim.y + cta) * 3 + threadIdx.x] = sum;
    }
  }
}

// ------------------------------------------------------- gray-world balance ----
// Per frame and channel: gains from the per-CTA sums (recover.py:57-69), then
// thr[k] = smallest recovered value x in [0, 1] whose output byte
// u8(clip(clip(x^(1/gamma)) * gain)) is >= k (bisection on the bit patterns of
// non-negative doubles, which order like the values), +inf where unreachable.
// The byte of a sample is then the number of thresholds <= x.
__device__ __forceinline__ int balanced_byte(double x, double inv_gamma, int gamma_is_one, double gain, int copy) {
  const double g = gamma_is_one ? x : fmin(fmax(pow(x, inv_gamma), 0.0), 1.0);
  return quantize_unit(copy ? g : fmin(fmax(__dmul_rn(g, gain), 0.0), 1.0));
}

__global__ void __launch_bounds__(256)
k_gf_thresholds(const double* __restrict__ part, int nparts, int64_t npx, double inv_gamma, int gamma_is_one,
                double* __restrict__ thr_out /* [n][3][256] */, float* __restrict__ gains_out /* [n][3] */) {
  __shared__ double s_gain;
  __shared__ int s_copy;
  const int f = blockIdx.y, c = blockIdx.x;
  if (threadIdx.x == 0) {
    double m[3];
    for (int ch = 0; ch < 3; ++ch) {
      double sum = 0.0;
      for (int b = 0; b < nparts; ++b) sum = __dadd_rn(sum, part[((int64_t)f * nparts + b) * 3 + ch]);
      m[ch] = __ddiv_rn(sum, (double)npx);
    }
    const bool degenerate = fmin(fmin(m[0], m[1]), m[2]) < 1e-6;
    const double mm = __ddiv_rn(__dadd_rn(__dadd_rn(m[0], m[1]), m[2]), 3.0);
    s_gain = degenerate ? 1.0 : fmin(fmax(__ddiv_rn(mm, m[c]), 0.5), 2.0);
    s_copy = degenerate;
  }
  __syncthreads();
  const int k = threadIdx.x;
  double* out = thr_out + ((int64_t)f * 3 + c) * 256;
  if (k == 0) gains_out[3 * f + c] = (float)s_gain;
  if (k == 0) {
    out[0] = -1.0;
    return;
  }
  const double gain = s_gain;
  const int copy = s_copy;
  if (balanced_byte(1.0, inv_gamma, gamma_is_one, gain, copy) < k) {
    out[k] = __longlong_as_double(0x7ff0000000000000LL);  // +inf: level never reached
    return;
  }
  if (balanced_byte(0.0, inv_gamma, gamma_is_one, gain, copy) >= k) {
    out[k] = 0.0;
    return;
  }
  long long lo = 0, hi = __double_as_longlong(1.0);  // byte(lo) < k <= byte(hi)
  {
    // bracket the answer around the analytic inverse x0 = ((k - 1/2)/255 / gain)^gamma
    // (+- 4096 ulps, verified): ~14 bisection steps instead of ~62 (the full bisection
    // remains the fallback when the bracket does not hold the step)
    const double y = __ddiv_rn((double)k - 0.5, 255.0);
    const double g = copy ? y : __ddiv_rn(y, gain);
    const double x0 = gamma_is_one ? g : pow(g, __drcp_rn(inv_gamma));
    if (x0 > 0.0 && x0 < 1.0) {
      const long long b0 = __double_as_longlong(x0);
      const long long l = max(b0 - 4096, 0LL), h = min(b0 + 4096, __double_as_longlong(1.0));
      if (balanced_byte(__longlong_as_double(l), inv_gamma, gamma_is_one, gain, copy) < k &&
          balanced_byte(__longlong_as_double(h), inv_gamma, gamma_is_one, gain, copy) >= k) {
        lo = l;
        hi = h;
      }
    }
  }
  while (hi - lo > 1) {
    const long long mid = lo + (hi - lo) / 2;
    if (balanced_byte(__longlong_as_double(mid), inv_gamma, gamma_is_one, gain, copy) >= k) hi = mid;
    else lo = mid;
  }
  out[k] = __longlong_as_double(hi);
}

// gray-world apply, fp32 fast path: the byte of channel c is the number of the
// frame's balanced thresholds thr_c[k] <= x (exact, k_gf_thresholds).  As in the
// two-pass output (guided_fused.cu), x is first formed in fp32 (|xf - x| < 4.6e-7
// wherever a window edge is finite) and accepted when it lies inside a byte window
// shrunk by 1e-6 (one bucket table read per sample); otherwise the exact fp64
// recovery and threshold walk decide.  Persistent CTAs over the batch's 4-pixel
// groups; the per-frame tables are rebuilt when a CTA's range enters a new frame.
struct ApplyShared {
  ByteBuckets bk[3];
  float dq[3][256];
  double f255[256];
  double thr[3][256];
  float af[3];
};

__device__ void apply_tables(ApplyShared& S, const double* __restrict__ thr, const double* __restrict__ airlight,
                             int f) {
  for (int i = threadIdx.x; i < 3 * 256; i += blockDim.x) {
    const int c = i >> 8, v = i & 255;
    S.thr[c][v] = thr[((int64_t)f * 3 + c) * 256 + v];
    S.dq[c][v] = __double2float_rn(__dsub_rn(S.f255[v], airlight[3 * f + c]));
    if (v == 0) S.af[c] = __double2float_rn(airlight[3 * f + c]);
  }
  __syncthreads();
  for (int c = 0; c < 3; ++c) byte_buckets_build(S.bk[c], S.thr[c]);
  __syncthreads();
}


__global__ void __launch_bounds__(256, 3)
k_gf_apply2(const uint8_t* __restrict__ in, int64_t in_fs, int n, int64_t npx, const double* __restrict__ t_in,
            const double* __restrict__ airlight, const double* __restrict__ thr, uint8_t* __restrict__ out,
            int64_t out_fs) {
  extern __shared__ __align__(16) unsigned char apply_smem[];
  ApplyShared& S = *reinterpret_cast<ApplyShared*>(apply_smem);
  for (int v = threadIdx.x; v < 256; v += blockDim.x) S.f255[v] = u8f(v);
  const int64_t G = (npx + 3) >> 2;  // 4-pixel groups per frame
  const int64_t total = (int64_t)n * G;
  const int64_t g0 = total * blockIdx.x / gridDim.x, g1 = total * (blockIdx.x + 1) / gridDim.x;
  const bool vec = (npx & 3) == 0 && (in_fs & 3) == 0 && (out_fs & 3) == 0 && ((uintptr_t)in & 3) == 0 &&
                   ((uintptr_t)out & 3) == 0 && ((uintptr_t)t_in & 15) == 0;
  for (int64_t s0 = g0; s0 < g1;) {
    const int f = (int)(s0 / G);
    const int64_t s1 = min(g1, (int64_t)(f + 1) * G);
    __syncthreads();  // the previous frame's readers are done
    apply_tables(S, thr, airlight, f);
    const double A0 = airlight[3 * f], A1 = airlight[3 * f + 1], A2 = airlight[3 * f + 2];
    const uint8_t* fi = in + (int64_t)f * in_fs;
    uint8_t* fo = out + (int64_t)f * out_fs;
    const double* ft = t_in + (int64_t)f * npx;
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
        uint32_t b[12];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int64_t p = p0 + min(u, np - 1);
          t[u] = ft[p];
          b[3 * u] = fi[3 * p];
          b[3 * u + 1] = fi[3 * p + 1];
          b[3 * u + 2] = fi[3 * p + 2];
        }
#pragma unroll
        for (int q = 0; q < 3; ++q) w[q] = b[4 * q] | (b[4 * q + 1] << 8) | (b[4 * q + 2] << 16) | (b[4 * q + 3] << 24);
      }
      uint32_t ob[12];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t v0 = (w[(3 * u) >> 2] >> (8 * ((3 * u) & 3))) & 255u;
        const uint32_t v1 = (w[(3 * u + 1) >> 2] >> (8 * ((3 * u + 1) & 3))) & 255u;
        const uint32_t v2 = (w[(3 * u + 2) >> 2] >> (8 * ((3 * u + 2) & 3))) & 255u;
        float rtf;
        asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rtf) : "f"(__double2float_rn(t[u])));
        bool ok = true;
        uint32_t k0 = byte_bucket(S.bk[0], __fmaf_rn(S.dq[0][v0], rtf, S.af[0]), ok);
        uint32_t k1 = byte_bucket(S.bk[1], __fmaf_rn(S.dq[1][v1], rtf, S.af[1]), ok);
        uint32_t k2 = byte_bucket(S.bk[2], __fmaf_rn(S.dq[2][v2], rtf, S.af[2]), ok);
        if (!ok) {
          const double rt = __drcp_rn(t[u]);
          k0 = quantize_thr_from(recover_raw(S.f255[v0], A0, t[u], rt), S.thr[0], (int)min(k0, 255u));
          k1 = quantize_thr_from(recover_raw(S.f255[v1], A1, t[u], rt), S.thr[1], (int)min(k1, 255u));
          k2 = quantize_thr_from(recover_raw(S.f255[v2], A2, t[u], rt), S.thr[2], (int)min(k2, 255u));
        }
        ob[3 * u] = k0;
        ob[3 * u + 1] = k1;
        ob[3 * u + 2] = k2;
      }
      uint8_t* o = fo + 3 * p0;
      if (vec) {
        uint32_t* o32 = reinterpret_cast<uint32_t*>(o);
        o32[0] = ob[0] | (ob[1] << 8) | (ob[2] << 16) | (ob[3] << 24);
        o32[1] = ob[4] | (ob[5] << 8) | (ob[6] << 16) | (ob[7] << 24);
        o32[2] = ob[8] | (ob[9] << 8) | (ob[10] << 16) | (ob[11] << 24);
      } else {
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < np) {
            o[3 * u] = (uint8_t)ob[3 * u];
            o[3 * u + 1] = (uint8_t)ob[3 * u + 1];
            o[3 * u + 2] = (uint8_t)ob[3 * u + 2];
          }
      }
    }
    s0 = s1;
  }
}

// Columns per thread (strip width 256*CPT input columns) from the frame width and
// radius only — never from the batch size, so a frame's box-sum rounding (and its
// bytes) do not depend on which batch it came in.  Wider strips waste fewer halo
// columns and amortise the per-row prefix; narrow frames keep more CTAs.
int guided_cpt(int W, int r) {
  int cpt = W >= 4096 ? 4 : (W >= 1024 ? 2 : 1);
  while (2 * r >= cpt * kThreads) cpt *= 2;  // the strip must hold the window
  return cpt;
}

template <int CPT>
size_t pass_smem(int nsums) { return ((size_t)2 * nsums * (kThreads * CPT + 2) + 2) * sizeof(double); }

}  // namespace

cudaError_t balance_thresholds(const double* part, int nparts, int n, int64_t npx, double gamma, double* thr,
                               float* gains, cudaStream_t st) {
  k_gf_thresholds<<<dim3(3, n), 256, 0, st>>>(part, nparts, npx, 1.0 / gamma, gamma == 1.0 ? 1 : 0, thr, gains);
  return cudaGetLastError();
}

// Rows per CTA segment, again from the frame geometry only: about 2 CTAs per SM for
// one frame; at least 16 rows (a shorter floor tied to r cost single images more
// parallelism than the 2r+1-row warm-up of the sliding sums saves).
int guided_seg_rows(int H, int W, int r, int cpt) {
  const int sw = kThreads * cpt - 2 * r;
  const int64_t strips = (W + sw - 1) / sw;
  const int64_t want = 2 * 148;
  int64_t segs = std::max<int64_t>(1, (want + strips - 1) / strips);
  int seg = (int)((H + segs - 1) / segs);
  seg = std::max(seg, std::min(H, 16));
  return std::min(seg, 1024);
}

cudaError_t guided_apply(const uint8_t* in, int64_t in_fs, int n, int64_t npx, const double* t,
                         const double* airlight, const double* thr, const float* gains, double gamma, uint8_t* out,
                         int64_t out_fs, cudaStream_t st) {
  (void)gains;
  (void)gamma;
  const int smem = (int)sizeof(ApplyShared);
  cudaError_t e = cudaFuncSetAttribute(k_gf_apply2, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t groups = (int64_t)n * ((npx + 3) / 4);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(3LL * sms, (groups + 255) / 256));
  k_gf_apply2<<<grid, 256, smem, st>>>(in, in_fs, n, npx, t, airlight, thr, out, out_fs);
  return cudaGetLastError();
}

// DHZ_GUIDED_PATH=fused|twopass|strip forces one image-mode implementation (tests, probes).
static int guided_path_override() {
  const char* s = getenv("DHZ_GUIDED_PATH");
  if (!s) return 0;
  if (!strcmp(s, "fused")) return 1;
  if (!strcmp(s, "strip")) return 2;
  if (!strcmp(s, "twopass")) return 3;
  return 0;
}

// Which image-mode implementation runs: 0 strip kernels (below), 1 one-pass exact
// (guided_fused.cu), 2 two-pass exact (guided_fused.cu, same bytes as 1).
int guided_path(int H, int W, int r) {
  const int o = guided_path_override();
  if (!guided_fused_ok(H, W, r)) return 0;
  if (o == 1) return 1;
  if (o == 3) return 2;
  if (o == 2) return 0;
  // default: the two-pass exact filter (C5: 1.05 vs 1.25 ms per 8K frame without balance,
  // on par with balance; C2 0.23 vs 0.25 ms); the strip kernels for r > 63
  return 2;
}

bool guided_use_fused(int H, int W, int r) { return guided_path(H, W, r) == 1; }

// Frames per chunk so the fp64 a/b (+t~) scratch stays within ~4 GB.
int guided_chunk(int n, int H, int W, bool balance) {
  const double per = (balance ? 24.0 : 16.0) * (double)H * W;
  return (int)std::max(1.0, std::min((double)n, 4.0e9 / per));
}

size_t guided_ws_bytes(int n, int H, int W, int r, bool balance) {
  switch (guided_path(H, W, r)) {
    case 1: return guided_fused_ws_bytes(n, H, W, r, balance);
    case 2: return guided_x_ws_bytes(n, H, W, r, balance);
    default: break;
  }
  const int64_t npx = (int64_t)H * W;
  const int c = guided_chunk(n, H, W, balance);
  size_t b = 16ull * npx * c;                                            // a, b
  if (balance) {
    const int cpt = guided_cpt(W, r), sw = kThreads * cpt - 2 * r;
    const int seg = guided_seg_rows(H, W, r, cpt);
    const int64_t parts = (int64_t)((W + sw - 1) / sw) * ((H + seg - 1) / seg);
    b += 8ull * npx * c + 24ull * parts * c + 3 * 256 * 8ull * c + 16ull * c;  // t~, sums, thresholds, gains
  }
  return b;
}

cudaError_t guided_recover_u8(const uint8_t* in, int64_t in_fs, int n, int H, int W, int r, double eps,
                              const double* airlight, double omega, double t_min, const double* thr, double gamma,
                              bool balance, uint8_t* out, int64_t out_fs, void* ws, cudaStream_t st) {
  if (r < 1 || r > kGuidedMaxRadius) return cudaErrorInvalidValue;
  switch (guided_path(H, W, r)) {
    case 1:
      return guided_fused_u8(in, in_fs, n, H, W, r, eps, airlight, omega, t_min, thr, gamma, balance, out, out_fs,
                             ws, st);
    case 2:
      return guided_x_u8(in, in_fs, n, H, W, r, eps, airlight, omega, t_min, thr, gamma, balance, out, out_fs, ws, st);
    default: break;
  }
  const int64_t npx = (int64_t)H * W;
  const int chunk = guided_chunk(n, H, W, balance);
  const double inv_g = 1.0 / gamma;
  const int g1 = gamma == 1.0 ? 1 : 0;
  for (int f0 = 0; f0 < n; f0 += chunk) {
    const int c = std::min(chunk, n - f0);
    const int cpt = guided_cpt(W, r);
    const int sw = kThreads * cpt - 2 * r;
    const int seg = guided_seg_rows(H, W, r, cpt);
    dim3 grid((W + sw - 1) / sw, (H + seg - 1) / seg, c);
    const uint8_t* fin = in + (int64_t)f0 * in_fs;
    uint8_t* fout = out + (int64_t)f0 * out_fs;
    const double* fA = airlight + 3 * f0;
    double* a = static_cast<double*>(ws);
    double* b = a + npx * c;
    double* t = b + npx * c;
    double* part = t + npx * c;
    cudaError_t ae = cudaSuccess;
    auto launch = [&](auto k1, auto k2, size_t sm1, size_t sm2) {
      if ((ae = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm1)) != cudaSuccess ||
          (ae = cudaFuncSetAttribute(k2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2)) != cudaSuccess)
        return;
      k1<<<grid, kThreads, sm1, st>>>(fin, in_fs, H, W, r, seg, eps, fA, omega, t_min, a, b);
      k2<<<grid, kThreads, sm2, st>>>(fin, in_fs, H, W, r, seg, a, b, fA, t_min, thr, inv_g, g1, fout, out_fs,
                                      balance ? t : nullptr, balance ? part : nullptr);
    };
    if (!balance) {
      if (cpt == 4) launch(k_gf_pass1<4>, k_gf_pass2<0, 4>, pass_smem<4>(4), pass_smem<4>(2));
      else if (cpt == 2) launch(k_gf_pass1<2>, k_gf_pass2<0, 2>, pass_smem<2>(4), pass_smem<2>(2));
      else launch(k_gf_pass1<1>, k_gf_pass2<0, 1>, pass_smem<1>(4), pass_smem<1>(2));
      if (ae != cudaSuccess) return ae;
    } else {
      if (cpt == 4) launch(k_gf_pass1<4>, k_gf_pass2<1, 4>, pass_smem<4>(4), pass_smem<4>(2));
      else if (cpt == 2) launch(k_gf_pass1<2>, k_gf_pass2<1, 2>, pass_smem<2>(4), pass_smem<2>(2));
      else launch(k_gf_pass1<1>, k_gf_pass2<1, 1>, pass_smem<1>(4), pass_smem<1>(2));
      if (ae != cudaSuccess) return ae;
      const int nparts = grid.x * grid.y;
      double* bthr = part + 3LL * nparts * c;
      float* gains = reinterpret_cast<float*>(bthr + 3LL * 256 * c);
      balance_thresholds(part, nparts, c, npx, gamma, bthr, gains, st);
      if ((ae = guided_apply(fin, in_fs, c, npx, t, fA, bthr, gains, gamma, fout, out_fs, st)) != cudaSuccess) return ae;
    }
  }
  return cudaGetLastError();
}

}  // namespace dhz
