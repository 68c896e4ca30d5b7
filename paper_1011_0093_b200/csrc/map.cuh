// K6: pixel -> palette mapping + MSE (reference: map_pixels,
// image_ops.hpp:18-51; mse, metrics.hpp:18-29; round_palette,
// palette.hpp:29-34 / round_to_rgb, color.hpp:38-46).
//
//   k_map_tables : rounded palette R (lround = half away from zero, clamp),
//                  integer d(R_p, R_t) and rows sorted by (d, index).
//   k_map_unique : once per UNIQUE color: exact argmin over R with the lowest
//                  index on ties, searched sort-means style from the color's
//                  final WSM label with the STRICT break d(R_p,R_t) > 4*prev
//                  (exact for lowest-index ties: a pruned t has d(x,R_t) >
//                  prev >= min). Writes the 16 MiB key->index LUT, the exact
//                  u64 Σ count*err (so MSE needs no per-pixel pass). It
//                  walks the samples in Morton order (coherent rows).
//   k_map_pixels : per pixel: LUT gather (L2-resident), emits the u8 index map
//                  and the mapped RGB raster with 16-B vector stores.
//   k_mse        : standalone mse(a, b) with __vabsdiffu4 + dp4a.
#pragma once
#include "common.cuh"

namespace cqb {

__device__ __forceinline__ uint32_t round_chan(double x) {
  double r = round(x);  // half away from zero == std::lround
  r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
  return (uint32_t)r;
}

// One block per row p. centers: K x 3 FP64 (AoS). pal_key[k] = packed key of R_k.
__global__ void k_map_tables(const double* __restrict__ centers, int k, int* __restrict__ sortedDr,
                             uint8_t* __restrict__ orderR, uint32_t* __restrict__ pal_key) {
  __shared__ uint32_t s_key[KMAX];
  __shared__ int s_d[KMAX];
  const int p = blockIdx.x, tid = threadIdx.x;
  for (int t = tid; t < k; t += blockDim.x) {
    s_key[t] = (round_chan(centers[3 * t]) << 16) | (round_chan(centers[3 * t + 1]) << 8) |
               round_chan(centers[3 * t + 2]);
  }
  __syncthreads();
  const uint32_t kp = s_key[p];
  const int pp = key_dot(kp, kp);
  for (int t = tid; t < k; t += blockDim.x) s_d[t] = pp + key_dot(s_key[t], s_key[t]) - 2 * key_dot(kp, s_key[t]);
  __syncthreads();
  for (int t = tid; t < k; t += blockDim.x) {
    int rank = 0;
    if (t != p) {
      const int dt = s_d[t];
      rank = 1;
      for (int u = 0; u < k; ++u) {
        const int du = s_d[u];
        rank += (u != p) & ((du < dt) | ((du == dt) & (u < t)));
      }
    }
    sortedDr[p * KMAX + rank] = t == p ? 0 : s_d[t];
    orderR[p * KMAX + rank] = (uint8_t)t;
  }
  if (p == 0)
    for (int t = tid; t < k; t += blockDim.x) pal_key[t] = s_key[t];
}

// Exact map of every unique color; start label optional (nullptr -> 0).
__global__ void __launch_bounds__(256) k_map_unique(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ counts,
                                                    const uint8_t* __restrict__ start_labels,
                                                    const unsigned long long* __restrict__ n_ptr, int k,
                                                    const int* __restrict__ sortedDr, const uint8_t* __restrict__ orderR,
                                                    const uint32_t* __restrict__ pal_key, uint8_t* __restrict__ lut,
                                                    unsigned long long* __restrict__ err_sum) {
  __shared__ uint32_t s_key[KMAX];
  __shared__ int s_cc[KMAX];
  __shared__ unsigned long long s_red[8];
  const int tid = threadIdx.x;
  for (int t = tid; t < k; t += blockDim.x) {
    s_key[t] = pal_key[t];
    s_cc[t] = key_dot(s_key[t], s_key[t]);
  }
  __syncthreads();
  const unsigned long long n = *n_ptr;
  unsigned long long err = 0;
  for (unsigned long long i = (unsigned long long)blockIdx.x * blockDim.x + tid; i < n;
       i += (unsigned long long)gridDim.x * blockDim.x) {
    const uint32_t x = keys[i];
    {
      const int xx = key_dot(x, x);
      const int p = start_labels ? start_labels[i] : 0;
      const int prev = xx + s_cc[p] - 2 * key_dot(x, s_key[p]);
      const int bound = 4 * prev;
      int mind = prev, best = p;
      const int* rowd = sortedDr + p * KMAX;
      const uint8_t* rowo = orderR + p * KMAX;
      for (int j = 1; j < k; ++j) {
        if (__ldg(rowd + j) > bound) break;
        const int t = __ldg(rowo + j);
        const int d = xx + s_cc[t] - 2 * key_dot(x, s_key[t]);
        if (d < mind || (d == mind && t < best)) {
          mind = d;
          best = t;
        }
      }
      lut[x] = (uint8_t)best;
      err += (unsigned long long)counts[i] * (unsigned long long)mind;
    }
  }
  {
    err = warp_sum(err);
    if ((tid & 31) == 0) s_red[tid >> 5] = err;
    __syncthreads();
    if (tid == 0) {
      unsigned long long t = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
      if (t) atomicAdd(err_sum, t);
    }
  }
}

// Per pixel: index map (u8) and mapped RGB (u8x3), 16 pixels per thread.
// Per byte: 255 - min(255, 4 |a - b|) (saturating SIMD adds).
__device__ __forceinline__ uint32_t err_bytes(uint32_t a, uint32_t b) {
  const uint32_t d = __vabsdiffu4(a, b);
  const uint32_t d2 = __vaddus4(d, d);
  return ~__vaddus4(d2, d2);
}

// Standalone error_image over two rasters of P pixels (bytes, any alignment).
__global__ void k_error_image(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b, uint64_t nbytes,
                              uint8_t* __restrict__ out) {
  const uint64_t n4 = nbytes / 4;
  const bool al = ((reinterpret_cast<uintptr_t>(a) | reinterpret_cast<uintptr_t>(b) | reinterpret_cast<uintptr_t>(out)) & 3) == 0;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * blockDim.x) {
    if (al) {
      reinterpret_cast<uint32_t*>(out)[i] =
          err_bytes(reinterpret_cast<const uint32_t*>(a)[i], reinterpret_cast<const uint32_t*>(b)[i]);
    } else {
      for (int j = 0; j < 4; ++j) out[4 * i + j] = (uint8_t)err_bytes(a[4 * i + j], b[4 * i + j]);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x < nbytes - 4 * n4) {
    const uint64_t j = 4 * n4 + threadIdx.x;
    out[j] = (uint8_t)err_bytes(a[j], b[j]);
  }
}

// Stores of one 16-pixel chunk starting at pixel p0 (n valid): u8 index map,
// mapped RGB and error_image, 16-B vector stores for full chunks.
__device__ __forceinline__ void map_store16(const uint8_t* __restrict__ img, uint64_t p0, int n,
                                            const uint32_t (&idx)[PX_PER_THREAD], const uint32_t* s_pal,
                                            uint8_t* __restrict__ out_index, uint8_t* __restrict__ out_rgb,
                                            uint8_t* __restrict__ out_err) {
  if (n == PX_PER_THREAD) {
    if (out_index) {
      uint4 v;
      v.x = idx[0] | (idx[1] << 8) | (idx[2] << 16) | (idx[3] << 24);
      v.y = idx[4] | (idx[5] << 8) | (idx[6] << 16) | (idx[7] << 24);
      v.z = idx[8] | (idx[9] << 8) | (idx[10] << 16) | (idx[11] << 24);
      v.w = idx[12] | (idx[13] << 8) | (idx[14] << 16) | (idx[15] << 24);
      __stcs(reinterpret_cast<uint4*>(out_index + p0), v);
    }
    if (out_rgb || out_err) {
      uint32_t pc[PX_PER_THREAD];
#pragma unroll
      for (int s = 0; s < PX_PER_THREAD; ++s) pc[s] = s_pal[idx[s]];
      uint32_t w[12];
#pragma unroll
      for (int g = 0; g < 4; ++g) {  // 4 pixels -> 3 words
        const uint32_t a = pc[4 * g], b = pc[4 * g + 1], cc = pc[4 * g + 2], d = pc[4 * g + 3];
        w[3 * g + 0] = a | (b << 24);
        w[3 * g + 1] = (b >> 8) | (cc << 16);
        w[3 * g + 2] = (cc >> 16) | (d << 8);
      }
      if (out_rgb) {
        uint4* dst = reinterpret_cast<uint4*>(out_rgb + p0 * 3);
        __stcs(dst, make_uint4(w[0], w[1], w[2], w[3]));
        __stcs(dst + 1, make_uint4(w[4], w[5], w[6], w[7]));
        __stcs(dst + 2, make_uint4(w[8], w[9], w[10], w[11]));
      }
      if (out_err) {  // error_image (image_ops.hpp:55-71): 255 - min(255, 4|o - q|) per byte
        const uint4* src = reinterpret_cast<const uint4*>(img + p0 * 3);
        const uint4 a = __ldg(src), b = __ldg(src + 1), d = __ldg(src + 2);
        const uint32_t o[12] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w, d.x, d.y, d.z, d.w};
        uint32_t e[12];
#pragma unroll
        for (int i = 0; i < 12; ++i) e[i] = err_bytes(o[i], w[i]);
        uint4* dst = reinterpret_cast<uint4*>(out_err + p0 * 3);
        __stcs(dst, make_uint4(e[0], e[1], e[2], e[3]));
        __stcs(dst + 1, make_uint4(e[4], e[5], e[6], e[7]));
        __stcs(dst + 2, make_uint4(e[8], e[9], e[10], e[11]));
      }
    }
  } else {
    for (int s = 0; s < n; ++s) {
      if (out_index) out_index[p0 + s] = (uint8_t)idx[s];
      const uint32_t pc = s_pal[idx[s]];
      if (out_rgb) {
        out_rgb[3 * (p0 + s)] = (uint8_t)pc;
        out_rgb[3 * (p0 + s) + 1] = (uint8_t)(pc >> 8);
        out_rgb[3 * (p0 + s) + 2] = (uint8_t)(pc >> 16);
      }
      if (out_err) {
        const uint32_t o = img[3 * (p0 + s)] | (img[3 * (p0 + s) + 1] << 8) | (img[3 * (p0 + s) + 2] << 16);
        const uint32_t e = err_bytes(o, pc);
        out_err[3 * (p0 + s)] = (uint8_t)e;
        out_err[3 * (p0 + s) + 1] = (uint8_t)(e >> 8);
        out_err[3 * (p0 + s) + 2] = (uint8_t)(e >> 16);
      }
    }
  }
}

__global__ void __launch_bounds__(HIST_THREADS) k_map_pixels(const uint8_t* __restrict__ img, uint64_t P,
                                                              const uint8_t* __restrict__ lut,
                                                              const uint32_t* __restrict__ pal_key, int k,
                                                              uint8_t* __restrict__ out_index,
                                                              uint8_t* __restrict__ out_rgb,
                                                              uint8_t* __restrict__ out_err) {
  __shared__ uint32_t s_pal[KMAX];  // bytes (r, g, b, 0) in memory order
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const uint32_t key = pal_key[t];
    s_pal[t] = key_r(key) | (key_g(key) << 8) | (key_b(key) << 16);
  }
  __syncthreads();
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  for (uint64_t c = (uint64_t)blockIdx.x * HIST_THREADS + threadIdx.x; c < nchunk;
       c += (uint64_t)gridDim.x * HIST_THREADS) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys(img, P, c, keys);
    uint32_t idx[PX_PER_THREAD];
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) idx[s] = s < n ? (uint32_t)__ldg(lut + keys[s]) : 0u;
    map_store16(img, c * PX_PER_THREAD, n, idx, s_pal, out_index, out_rgb, out_err);
  }
}

// ---------------------------------------------------------------------------
// Coarse map table (large images). The LUT gather is one random 32-B L2
// sector per pixel; on a 16 M-pixel image that is ~0.5 GB of L2 traffic,
// and the L1 processes one distinct line per cycle. Most colors, however,
// share their palette index with every other PRESENT color of their small
// color cell: the cells are 4 x 4 x 8 colors ((r>>2, g>>2, b>>3), 2^17 cells,
// each a Morton-aligned run of 128 codes, so its samples are contiguous),
// and a Voronoi cell of a K = 256 palette is ~40 colors wide (cfg4: 69.5% of
// the pixels fall in pure cells). The loop's map epilogue records, per cell,
// the index all its samples map to or MIXED (warp segments of equal cells,
// one CAS per segment: 0 -> index + 1, any other value -> MIXED); a
// compaction pass turns the words into one byte per cell (128 KB), which
// k_map_pixels_coarse holds in shared memory: a pixel of a pure cell reads
// its index with one LDS, only pixels of MIXED cells gather from the LUT.
// The byte 255 means "gather": MIXED and empty cells, and (K = 256) the pure
// cells of index 255, whose LUT value is 255 anyway. The result is identical
// to the per-pixel LUT gather: a pure cell's index IS the LUT value of every
// color present in it.
constexpr int COARSE_CELLS = 1 << 17;
constexpr uint32_t COARSE_MIXED = 0x200u;
constexpr size_t COARSE_BYTES = COARSE_CELLS;
constexpr uint32_t COARSE_GATHER = 255u;
constexpr int MAPC_THREADS = 1024;
__host__ __device__ __forceinline__ uint32_t coarse_cell(uint32_t key) {
  return (((key >> 18) & 63u) << 11) | (((key >> 10) & 63u) << 5) | ((key >> 3) & 31u);
}

// Records sample color x -> palette index `best` for its cell. Called by the
// lanes in `am` (warp-converged, consecutive Morton samples).
__device__ __forceinline__ void coarse_note(uint32_t* __restrict__ cellw, unsigned am, uint32_t x, int best) {
  const uint32_t c = coarse_cell(x);
  const unsigned mc = __match_any_sync(am, c);
  const unsigned ml = __match_any_sync(am, (c << 8) | (uint32_t)best);
  if ((int)(threadIdx.x & 31) == __ffs(mc) - 1) {
    const uint32_t v = mc == ml ? (uint32_t)best + 1u : COARSE_MIXED;
    if (v == COARSE_MIXED) {
      atomicExch(&cellw[c], COARSE_MIXED);
    } else {
      const uint32_t old = atomicCAS(&cellw[c], 0u, v);
      if (old != 0u && old != v) atomicExch(&cellw[c], COARSE_MIXED);
    }
  }
}

// Word table -> one byte per cell (grid-stride): the pure cells' index, or
// COARSE_GATHER (MIXED or empty: no pixel reads an empty cell).
__device__ __forceinline__ void coarse_compact(const uint32_t* __restrict__ cellw, uint8_t* __restrict__ coarse,
                                               uint32_t gtid, uint32_t gthreads) {
  for (uint32_t c = gtid; c < (uint32_t)COARSE_CELLS; c += gthreads) {
    const uint32_t w = __ldcg(&cellw[c]);
    coarse[c] = (w == 0u || w == COARSE_MIXED) ? (uint8_t)COARSE_GATHER : (uint8_t)(w - 1u);
  }
}

// k_map_pixels with the coarse table in shared memory: one block of 1024
// threads per SM; 128 KB table + palette.
__global__ void __launch_bounds__(MAPC_THREADS, 1) k_map_pixels_coarse(
    const uint8_t* __restrict__ img, uint64_t P, const uint8_t* __restrict__ lut, const uint8_t* __restrict__ coarse,
    const uint32_t* __restrict__ pal_key, int k, uint8_t* __restrict__ out_index, uint8_t* __restrict__ out_rgb,
    uint8_t* __restrict__ out_err) {
  extern __shared__ __align__(16) unsigned char mapc_smem[];
  __shared__ uint32_t s_pal[KMAX];
  const uint8_t* s_lab = mapc_smem;
  for (int t = threadIdx.x; t < k; t += blockDim.x) {
    const uint32_t key = pal_key[t];
    s_pal[t] = key_r(key) | (key_g(key) << 8) | (key_b(key) << 16);
  }
  {
    const uint4* src = reinterpret_cast<const uint4*>(coarse);
    uint4* dst = reinterpret_cast<uint4*>(mapc_smem);
    for (int i = threadIdx.x; i < (int)(COARSE_BYTES / 16); i += blockDim.x) dst[i] = __ldg(src + i);
  }
  __syncthreads();
  const uint64_t nchunk = (P + PX_PER_THREAD - 1) / PX_PER_THREAD;
  for (uint64_t c = (uint64_t)blockIdx.x * MAPC_THREADS + threadIdx.x; c < nchunk;
       c += (uint64_t)gridDim.x * MAPC_THREADS) {
    uint32_t keys[PX_PER_THREAD];
    const int n = load_chunk_keys<true>(img, P, c, keys);
    uint32_t idx[PX_PER_THREAD];
#pragma unroll
    for (int s = 0; s < PX_PER_THREAD; ++s) {
      uint32_t v = s_lab[coarse_cell(keys[s])];
      if (v == COARSE_GATHER && s < n) v = __ldg(lut + keys[s]);
      idx[s] = v;
    }
    map_store16(img, c * PX_PER_THREAD, n, idx, s_pal, out_index, out_rgb, out_err);
  }
}

// Label layout helpers: Morton-ordered samples <-> first-occurrence order.
// lab_m[j] = lab_rank[rank[j]]  /  lab_rank[rank[j]] = lab_m[j]
__global__ void k_labels_gather(const uint32_t* __restrict__ rank, const uint8_t* __restrict__ lab_rank,
                                uint8_t* __restrict__ lab_m, const unsigned long long* __restrict__ n_ptr) {
  const uint64_t n = *n_ptr;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    lab_m[i] = lab_rank[rank[i]];
}
__global__ void k_labels_scatter(const uint32_t* __restrict__ rank, const uint8_t* __restrict__ lab_m,
                                 uint8_t* __restrict__ lab_rank, const unsigned long long* __restrict__ n_ptr) {
  const uint64_t n = *n_ptr;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x)
    lab_rank[rank[i]] = lab_m[i];
}

// mse(a, b) numerator: exact u64 Σ squared channel differences (metrics.hpp:21-27).
__global__ void __launch_bounds__(256) k_mse(const uint8_t* __restrict__ a, const uint8_t* __restrict__ b,
                                             uint64_t nbytes, unsigned long long* __restrict__ out) {
  __shared__ unsigned long long s_red[8];
  unsigned long long acc = 0;
  const uint64_t nvec = nbytes / 16;
  const uint4* va = reinterpret_cast<const uint4*>(a);
  const uint4* vb = reinterpret_cast<const uint4*>(b);
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nvec; i += (uint64_t)gridDim.x * blockDim.x) {
    const uint4 x = __ldg(va + i), y = __ldg(vb + i);
    unsigned int d, s = 0;
    d = __vabsdiffu4(x.x, y.x); s = __dp4a(d, d, s);
    d = __vabsdiffu4(x.y, y.y); s = __dp4a(d, d, s);
    d = __vabsdiffu4(x.z, y.z); s = __dp4a(d, d, s);
    d = __vabsdiffu4(x.w, y.w); s = __dp4a(d, d, s);
    acc += s;
  }
  if (blockIdx.x == 0)
    for (uint64_t i = nvec * 16 + threadIdx.x; i < nbytes; i += blockDim.x) {
      const int d = (int)a[i] - (int)b[i];
      acc += (unsigned long long)(d * d);
    }
  acc = warp_sum(acc);
  if ((threadIdx.x & 31) == 0) s_red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_red[w];
    atomicAdd(out, t);
  }
}

}  // namespace cqb
