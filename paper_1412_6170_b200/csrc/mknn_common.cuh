// mknn_common.cuh -- device-side arithmetic shared by every mknn kernel.
//
// Bit-exactness contract: each fp64 expression below
// is the reference's numpy expression evaluated as separate IEEE operations
// (__d*_rn intrinsics, never contracted into FMA; the library is also built
// with -fmad=false).  Citations are relative to /root/reference/pkg/src/mknn/.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace mknn {

constexpr unsigned FULL = 0xffffffffu;
constexpr double DINF = __builtin_huge_val();
constexpr long long IDMAX = 0x7fffffffffffffffLL;
constexpr int MAX_L_MAX = 10;  // quadindex.py:20

struct Region {
  double x_lo, y_lo, x_hi, y_hi;
  double w, h;  // x_hi - x_lo, y_hi - y_lo computed on the host (geometry.py:46-52)
  double inv_w, inv_h;  // 1 / w, 1 / h (0 when the width is 0): fast path of coord16
};

// offset of level l in the concatenated count pyramid (levels 0..l_max);
// every level starts on a 16-byte boundary (level 0 is padded to 4 cells)
// so a parent level can be reduced from its children with int4 loads
__host__ __device__ __forceinline__ long long pyramid_offset_dev(int level) {
  return level == 0 ? 0 : 4 + 4 * (((1LL << (2 * (level - 1))) - 1) / 3);
}

// geometry.py:75-83 spread_bits (low 32 bits to even positions)
__host__ __device__ __forceinline__ uint64_t spread_bits(uint64_t v) {
  v &= 0xFFFFFFFFull;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}

// geometry.py:86-94 compact_bits; codes here are <= 20 bits (l_max <= 10)
__host__ __device__ __forceinline__ uint32_t compact_bits32(uint32_t v) {
  v &= 0x55555555u;
  v = (v | (v >> 1)) & 0x33333333u;
  v = (v | (v >> 2)) & 0x0F0F0F0Fu;
  v = (v | (v >> 4)) & 0x00FF00FFu;
  v = (v | (v >> 8)) & 0x0000FFFFu;
  return v;
}

__device__ __forceinline__ uint32_t spread_bits32(uint32_t v) {
  v &= 0x0000FFFFu;
  v = (v | (v << 8)) & 0x00FF00FFu;
  v = (v | (v << 4)) & 0x0F0F0F0Fu;
  v = (v | (v << 2)) & 0x33333333u;
  v = (v | (v << 1)) & 0x55555555u;
  return v;
}

// 2^-lvl as an exact double (0 <= lvl <= 31)
__device__ __forceinline__ double pow2_neg(int lvl) {
  return __longlong_as_double((long long)(1023 - lvl) << 52);
}
__device__ __forceinline__ double pow2_pos(int lvl) {
  return __longlong_as_double((long long)(1023 + lvl) << 52);
}

// geometry.py:105-129 cell_coords for one axis:
//   t = (v - lo) / width (0 when width == 0); c = clip(floor(t * 2^L), 0, 2^L - 1)
__device__ __forceinline__ uint32_t cell_coord(double v, double lo, double width, int level) {
  const double n = pow2_pos(level);
  const double t = (width > 0.0) ? __ddiv_rn(__dsub_rn(v, lo), width) : 0.0;
  double c = floor(__dmul_rn(t, n));  // x 2^L is exact
  c = fmax(c, 0.0);
  c = fmin(c, n - 1.0);
  return (uint32_t)c;
}

// cell coordinate of one axis at level 16, exactly
//   clip(floor(fl((v - lo) / width) * 2^16), 0, 2^16 - 1)   (geometry.py:105-129)
// The quotient is first formed with the reciprocal (two roundings, so it is
// within 2^-51 relative of the IEEE quotient); only when the scaled value
// lands within 2^-30 of a cell border -- where the two quotients could floor
// differently -- is the IEEE division evaluated.  Coarser levels L are the
// prefixes c16 >> (16 - L) (the same t at every level, geometry.py:108-112).
__device__ __forceinline__ uint32_t coord16(double v, double lo, double width, double inv_width) {
  if (!(width > 0.0)) return 0;
  const double d = __dsub_rn(v, lo);
  const double f = __dmul_rn(__dmul_rn(d, inv_width), 65536.0);
  double c = floor(f);
  const double fr = __dsub_rn(f, c);  // exact
  if (fr < 0x1p-30 || fr > 1.0 - 0x1p-30) c = floor(__dmul_rn(__ddiv_rn(d, width), 65536.0));
  c = fmax(c, 0.0);
  c = fmin(c, 65535.0);
  return (uint32_t)c;
}

// Morton code at level 16 of a point (x bits even, y bits odd)
__device__ __forceinline__ uint32_t encode16(double x, double y, const Region& r) {
  return spread_bits32(coord16(x, r.x_lo, r.w, r.inv_w)) |
         (spread_bits32(coord16(y, r.y_lo, r.h, r.inv_h)) << 1);
}

// geometry.py:132-135 encode_points (x bits even, y bits odd; SW,SE,NW,NE)
__device__ __forceinline__ uint32_t encode(double x, double y, const Region& r, int level) {
  const uint32_t cx = cell_coord(x, r.x_lo, r.w, level);
  const uint32_t cy = cell_coord(y, r.y_lo, r.h, level);
  return spread_bits32(cx) | (spread_bits32(cy) << 1);
}

// max(a, b) without NaN handling (coordinates are finite; the reference's
// np.maximum only differs on NaN)
__device__ __forceinline__ double dmax(double a, double b) { return a > b ? a : b; }

// geometry.py:166-181 cell_bounds_arrays + 189-193 min_dist2_point_cells:
//   bound = lo + ldexp(c, -lvl) * width   (multiply, then add)
//   d = max(max(lo - q, q - hi), 0);  d2 = dx*dx + dy*dy
__device__ __forceinline__ double mindist2_cell(int lvl, uint32_t code, const Region& r,
                                                double qx, double qy) {
  const double s = pow2_neg(lvl);
  const uint32_t cx = compact_bits32(code), cy = compact_bits32(code >> 1);
  const double xl = __dadd_rn(r.x_lo, __dmul_rn(__dmul_rn((double)cx, s), r.w));
  const double xh = __dadd_rn(r.x_lo, __dmul_rn(__dmul_rn((double)(cx + 1), s), r.w));
  const double yl = __dadd_rn(r.y_lo, __dmul_rn(__dmul_rn((double)cy, s), r.h));
  const double yh = __dadd_rn(r.y_lo, __dmul_rn(__dmul_rn((double)(cy + 1), s), r.h));
  const double dx = dmax(dmax(__dsub_rn(xl, qx), __dsub_rn(qx, xh)), 0.0);
  const double dy = dmax(dmax(__dsub_rn(yl, qy), __dsub_rn(qy, yh)), 0.0);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// geometry.py:203-212 / engine.py:294-296: dx*dx + dy*dy with three roundings
__device__ __forceinline__ double pair_d2(double qx, double qy, double ox, double oy) {
  const double dx = __dsub_rn(qx, ox);
  const double dy = __dsub_rn(qy, oy);
  return __dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy));
}

// Canonical candidate order (oracle.py:76-77): (d2, id) lexicographic.
__device__ __forceinline__ bool key_less(double ad, long long ai, double bd, long long bi) {
  return (ad < bd) | ((ad == bd) & (ai < bi));
}

}  // namespace mknn

#define MKNN_CUDA_OK(expr)                                                      \
  do {                                                                          \
    cudaError_t _e = (expr);                                                    \
    if (_e != cudaSuccess) return ::mknn::fail_cuda(_e, #expr, __FILE__, __LINE__); \
  } while (0)
