// Shared device helpers for the B200 WSM path (sm_100a).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>

namespace cqb {

constexpr int KMAX = 256;            // palette sizes handled on device (u8 labels)
#ifndef CQB_LOOP_THREADS
#define CQB_LOOP_THREADS 1024
#endif
constexpr int LOOP_THREADS = CQB_LOOP_THREADS;
#ifndef CQB_LOOP_MINB
#define CQB_LOOP_MINB 1  // persistent WSM loop blocks per SM (__launch_bounds__)
#endif  // persistent WSM loop block size (one block per SM)
#ifndef CQB_PPT_LARGE
#define CQB_PPT_LARGE 2  // WSM loop: 32-sample chunks per warp grab for large sample sets
#endif
constexpr int MAXBLK = 1024;         // max persistent blocks (reseed candidate slots)
constexpr int HIST_THREADS = 256;    // histogram / compaction block size
constexpr int PX_PER_THREAD = 16;    // 16 pixels = 48 B = 3 x 16-B vector loads
constexpr int TILE_PX = HIST_THREADS * PX_PER_THREAD;  // pixels per compaction tile

// Device status codes (mirrored by CQB_* in include/colorq_b200.h).
constexpr int ST_OK = 0;
constexpr int ST_K_EXCEEDS_N = 1;    // init_centers: k > N' (kmeans.hpp:55-56)
constexpr int ST_DRAWS_EXHAUSTED = 2;
constexpr int ST_XCH_TIMEOUT = 3;    // sharded loop: a peer did not publish within XCH_TIMEOUT_NS

// Squared Euclidean distance exactly as color.hpp:49-54 evaluates it:
// ((dr*dr + dg*dg) + db*db) in FP64, every operation rounded, NO FMA.
__device__ __forceinline__ double dist2_rn(double x0, double x1, double x2, double c0, double c1, double c2) {
  const double dr = __dsub_rn(x0, c0);
  const double dg = __dsub_rn(x1, c1);
  const double db = __dsub_rn(x2, c2);
  return __dadd_rn(__dadd_rn(__dmul_rn(dr, dr), __dmul_rn(dg, dg)), __dmul_rn(db, db));
}

// Packed 24-bit key r<<16 | g<<8 | b (pack_rgb, color.hpp:25-27). As a u8x4 word
// its bytes are (b, g, r, 0), so __dp4a(key_a, key_b) is the RGB dot product.
__device__ __forceinline__ int key_dot(uint32_t a, uint32_t b) { return (int)__dp4a(a, b, 0u); }

// Double-double helpers for the deterministic moment-form SSE.
struct dd {
  double hi, lo;
};
__device__ __forceinline__ dd two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  const double bb = __dsub_rn(s, a);
  const double e = __dadd_rn(__dsub_rn(a, __dsub_rn(s, bb)), __dsub_rn(b, bb));
  return {s, e};
}
__device__ __forceinline__ dd quick_two_sum(double a, double b) {
  const double s = __dadd_rn(a, b);
  return {s, __dsub_rn(b, __dsub_rn(s, a))};
}
__device__ __forceinline__ dd two_prod(double a, double b) {
  const double p = __dmul_rn(a, b);
  return {p, __fma_rn(a, b, -p)};
}
__device__ __forceinline__ dd dd_add(dd x, dd y) {
  dd s = two_sum(x.hi, y.hi);
  const double e = __dadd_rn(s.lo, __dadd_rn(x.lo, y.lo));
  return quick_two_sum(s.hi, e);
}
__device__ __forceinline__ dd dd_scale(dd x, double b) {  // x * b
  dd p = two_prod(x.hi, b);
  const double e = __fma_rn(x.lo, b, p.lo);
  return quick_two_sum(p.hi, e);
}
__device__ __forceinline__ dd dd_neg(dd x) { return {-x.hi, -x.lo}; }

// New center coordinate from a cluster's exact integer moments (N pixels,
// channel sum Sv, all-channel sums S0..S2 and square sum Q). The reference
// forms sum_i w_i x_i / sum_i w_i sequentially in FP64 with w_i = count_i *
// fl(1/P) (kmeans.hpp:245-296); the exact mean S/N rounded once differs from
// it only by that rounding. A one-color cluster (N Q == |S|^2, equality in
// Cauchy-Schwarz) is common when k is near N', and for it the reference value
// fl(fl(w x) / w) is reproduced exactly, so that such a cluster is stationary
// exactly when the reference sees it stationary (the pair count of the
// incremental table update, kmeans.hpp:137-155).
__device__ __forceinline__ bool one_color_cluster(unsigned long long N, unsigned long long S0, unsigned long long S1,
                                                  unsigned long long S2, unsigned long long Q) {
  const unsigned __int128 a = (unsigned __int128)N * Q;
  const unsigned __int128 b =
      (unsigned __int128)S0 * S0 + (unsigned __int128)S1 * S1 + (unsigned __int128)S2 * S2;
  return a == b;
}
// The correction only matters when the exact mean is an integer (a one-color
// cluster's mean is its color), so the moments are re-read on that rare path.
// Moment loads: global sums through L2 (written by other blocks' atomics), or
// (kShared) the sharded loop's totals in shared memory.
template <bool kShared>
__device__ __forceinline__ unsigned long long ldmom(const unsigned long long* p) {
  if constexpr (kShared) return *p;
  else return __ldcg(p);
}
template <bool kShared = false>
__device__ __forceinline__ double center_coord(const unsigned long long* __restrict__ mom, int stride, int t,
                                               unsigned long long Sv, unsigned long long N, double inv_P) {
  const double c = __ddiv_rn((double)Sv, (double)N);
  if (c == rint(c) &&
      one_color_cluster(N, ldmom<kShared>(&mom[t]), ldmom<kShared>(&mom[stride + t]),
                        ldmom<kShared>(&mom[2 * stride + t]), ldmom<kShared>(&mom[4 * stride + t]))) {
    const double w = __dmul_rn((double)N, inv_P);
    return __ddiv_rn(__dmul_rn(w, c), w);
  }
  return c;
}

// center_coord with all five moments of the cluster already in registers.
__device__ __forceinline__ double center_coord_v(unsigned long long Sv, unsigned long long N, unsigned long long S0,
                                                 unsigned long long S1, unsigned long long S2, unsigned long long Q,
                                                 double inv_P) {
  const double c = __ddiv_rn((double)Sv, (double)N);
  if (c == rint(c) && one_color_cluster(N, S0, S1, S2, Q)) {
    const double w = __dmul_rn((double)N, inv_P);
    return __ddiv_rn(__dmul_rn(w, c), w);
  }
  return c;
}

// Exact u8 -> double without I2F: the bits of 2^52 + v are 0x43300000:v.
__device__ __forceinline__ double u8_to_double(uint32_t v) {
  return __dsub_rn(__hiloint2double(0x43300000, (int)v), 4503599627370496.0);
}

__device__ __forceinline__ uint32_t key_r(uint32_t k) { return (k >> 16) & 255u; }
__device__ __forceinline__ uint32_t key_g(uint32_t k) { return (k >> 8) & 255u; }
__device__ __forceinline__ uint32_t key_b(uint32_t k) { return k & 255u; }

// Loads the 16 pixels of chunk c (pixel indices 16c..16c+15) of a row-major
// u8x3 raster as packed keys. Full chunks use three 16-B read-only vector
// loads (the raster base is 16-B aligned by contract); the tail chunk uses
// byte loads. Returns the number of valid pixels.
// kStream: read-once loads (evict-first), so the raster does not push other
// L2-resident tables out.
template <bool kStream = false>
__device__ __forceinline__ int load_chunk_keys(const uint8_t* __restrict__ img, uint64_t P, uint64_t c,
                                               uint32_t (&keys)[PX_PER_THREAD]) {
  const uint64_t p0 = c * PX_PER_THREAD;
  if (p0 + PX_PER_THREAD <= P) {
    const uint4* src = reinterpret_cast<const uint4*>(img + p0 * 3);
    uint4 a, b, d;
    if constexpr (kStream) {
      a = __ldcs(src), b = __ldcs(src + 1), d = __ldcs(src + 2);
    } else {
      a = __ldg(src), b = __ldg(src + 1), d = __ldg(src + 2);
    }
    const uint32_t w[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) {
      const int o = 3 * s, j = o >> 2, q = o & 3;
      const int j2 = j + 1 < 12 ? j + 1 : 11;
      // result bytes (b, g, r, *) = pool bytes (q+2, q+1, q, q)
      const uint32_t sel = (uint32_t)(q + 2) | ((uint32_t)(q + 1) << 4) | ((uint32_t)q << 8) | ((uint32_t)q << 12);
      keys[s] = __byte_perm(w[j], w[j2], sel) & 0x00FFFFFFu;
    }
    return PX_PER_THREAD;
  }
  int n = 0;
#pragma unroll
  for (int s = 0; s < PX_PER_THREAD; ++s) {
    const uint64_t p = p0 + s;
    if (p < P) {
      keys[s] = ((uint32_t)img[3 * p] << 16) | ((uint32_t)img[3 * p + 1] << 8) | (uint32_t)img[3 * p + 2];
      ++n;
    } else {
      keys[s] = 0;
    }
  }
  return n;
}

// Morton (Z-order) code of a color: bits of r, g, b interleaved (r highest).
// The 2^24-bin histogram is indexed by this code, so a bin-order scan yields
// the unique colors in a space-filling-curve order: consecutive samples are
// spatial neighbours in RGB, which makes the WSM warps coherent.
__host__ __device__ __forceinline__ uint32_t spread3(uint32_t v) {  // 8 bits -> every 3rd bit
  v &= 0xFFu;
  v = (v | (v << 8)) & 0x0000F00Fu;
  v = (v | (v << 4)) & 0x000C30C3u;
  v = (v | (v << 2)) & 0x00249249u;
  return v;
}
__host__ __device__ __forceinline__ uint32_t compact3(uint32_t v) {
  v &= 0x00249249u;
  v = (v | (v >> 2)) & 0x000C30C3u;
  v = (v | (v >> 4)) & 0x0000F00Fu;
  v = (v | (v >> 8)) & 0x000000FFu;
  return v;
}
__host__ __device__ __forceinline__ uint32_t morton_of_key(uint32_t key) {
  return (spread3(key >> 16) << 2) | (spread3(key >> 8) << 1) | spread3(key);
}
__host__ __device__ __forceinline__ uint32_t key_of_morton(uint32_t m) {
  return (compact3(m >> 2) << 16) | (compact3(m >> 1) << 8) | compact3(m);
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace cqb
