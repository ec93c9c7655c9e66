// mknn_prims.cu -- device-wide scan, stable LSD radix sort, min/max.
//
// Hand-written for sm_100a (no CUB/Thrust on the product path).  These back
// the counting sorts of objects and queries by leaf (quadindex.py:197-202,
// engine.py:208) and the stable issuer-order emission (engine.py:713,
// oracle.py:56).
#include <atomic>
#include <cstdio>
#include <string>

#include "mknn_internal.h"

namespace mknn {

static thread_local std::string g_err;

int fail_cuda(cudaError_t e, const char* expr, const char* file, int line) {
  char buf[512];
  snprintf(buf, sizeof(buf), "CUDA error %s (%s) at %s:%d: %s", cudaGetErrorName(e),
           cudaGetErrorString(e), file, line, expr);
  g_err = buf;
  return E_CUDA;
}

int fail_msg(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

const char* last_error_text() { return g_err.c_str(); }

static std::atomic<long long> g_launches{0};
void note_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
long long launch_count() { return g_launches.load(std::memory_order_relaxed); }
void note_launches(long long n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

// ------------------------------------------------------------------ scan
namespace {

constexpr int SCAN_THREADS = 256;
constexpr int SCAN_ITEMS = 16;
constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;  // 4096

template <typename T>
__device__ __forceinline__ T warp_incl_scan(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T u = __shfl_up_sync(FULL, v, o);
    if (lane >= o) v += u;
  }
  return v;
}

// exclusive block scan of one value per thread; returns the block total
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* sh_warp, T& total) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nw = blockDim.x >> 5;
  T inc = warp_incl_scan(v);
  if (lane == 31) sh_warp[w] = inc;
  __syncthreads();
  if (w == 0) {
    T s = lane < nw ? sh_warp[lane] : T(0);
    T si = warp_incl_scan(s);
    if (lane < nw) sh_warp[lane] = si - s;
    if (lane == nw - 1) sh_warp[32] = si;
  }
  __syncthreads();
  total = sh_warp[32];
  T r = inc - v + sh_warp[w];
  __syncthreads();
  return r;
}

// Single-pass scan with decoupled look-back: each tile publishes its
// aggregate, then its inclusive prefix once the predecessor prefixes are
// known; tile ids come from an atomic counter so every tile's predecessors
// are already running (forward progress).  Status word: value << 2 | flag
// (flag 1 = aggregate only, 2 = inclusive prefix; 0 = not yet published).
constexpr unsigned long long ST_AGG = 1, ST_PREFIX = 2;

__device__ __forceinline__ unsigned long long ld_status(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_status(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

template <typename TO>
__global__ void __launch_bounds__(SCAN_THREADS) k_scan_lookback(
    const int32_t* __restrict__ in, TO* __restrict__ out, int64_t n, int64_t n_tiles,
    unsigned long long* status, unsigned int* tile_ctr) {
  __shared__ long long sh[33];
  __shared__ long long tile_excl;
  __shared__ int tile_sh;
  if (threadIdx.x == 0) tile_sh = (int)atomicAdd(tile_ctr, 1u);
  __syncthreads();
  const int64_t tile = tile_sh;
  const int64_t base = tile * SCAN_TILE + (int64_t)threadIdx.x * SCAN_ITEMS;
  int32_t v[SCAN_ITEMS];
  if (base + SCAN_ITEMS <= n && (reinterpret_cast<uintptr_t>(in) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i += 4) {
      const int4 q = *reinterpret_cast<const int4*>(&in[base + i]);
      v[i] = q.x;
      v[i + 1] = q.y;
      v[i + 2] = q.z;
      v[i + 3] = q.w;
    }
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++) v[i] = base + i < n ? in[base + i] : 0;
  }
  long long acc = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) acc += v[i];
  long long tot;
  long long ex = block_excl_scan<long long>(acc, sh, tot);
  // look-back (warp 0): 32 predecessors per round
  if (threadIdx.x < 32) {
    const int lane = threadIdx.x;
    if (lane == 0)
      st_status(&status[tile], ((unsigned long long)tot << 2) | (tile == 0 ? ST_PREFIX : ST_AGG));
    long long prefix = 0;
    if (tile > 0) {
      int64_t j = tile - 1;
      for (;;) {
        const int64_t p = j - lane;
        unsigned long long st = ST_PREFIX;  // beyond tile 0: neutral
        if (p >= 0) {
          do {
            st = ld_status(&status[p]);
          } while ((st & 3ull) == 0);
        }
        const bool is_prefix = p < 0 || (st & 3ull) == ST_PREFIX;
        const unsigned pm = __ballot_sync(FULL, is_prefix);
        const int stop = __ffs(pm) - 1;  // nearest predecessor with a full prefix
        long long val = (p >= 0 && (pm == 0 || lane <= stop)) ? (long long)(st >> 2) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) val += __shfl_xor_sync(FULL, val, o);
        prefix += val;
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) st_status(&status[tile], ((unsigned long long)(prefix + tot) << 2) | ST_PREFIX);
    }
    if (lane == 0) tile_excl = prefix;
  }
  __syncthreads();
  ex += tile_excl;
  TO o[SCAN_ITEMS];
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; i++) {
    o[i] = (TO)ex;
    ex += v[i];
  }
  constexpr int VEC = 16 / sizeof(TO);  // elements per 16-byte store
  if (base + SCAN_ITEMS <= n && (reinterpret_cast<uintptr_t>(out + base) & 15) == 0) {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i += VEC) *reinterpret_cast<int4*>(&out[base + i]) = *reinterpret_cast<int4*>(&o[i]);
  } else {
#pragma unroll
    for (int i = 0; i < SCAN_ITEMS; i++)
      if (base + i < n) out[base + i] = o[i];
  }
  if (tile == n_tiles - 1 && threadIdx.x == blockDim.x - 1) out[n] = (TO)ex;
}

template <typename TO>
__global__ void k_set_zero_total(TO* out) { out[0] = 0; }

template <typename TO>
int exclusive_scan_impl(const int32_t* in, TO* out, int64_t n, void* scratch, cudaStream_t s) {
  if (n == 0) {
    MKNN_LAUNCH k_set_zero_total<TO><<<1, 1, 0, s>>>(out);
    MKNN_CUDA_OK(cudaGetLastError());
    return 0;
  }
  const int64_t nb = (n + SCAN_TILE - 1) / SCAN_TILE;
  unsigned long long* status = (unsigned long long*)scratch;
  unsigned int* ctr = (unsigned int*)(status + nb);
  MKNN_CUDA_OK(cudaMemsetAsync(scratch, 0, sizeof(unsigned long long) * (nb + 1), s));
  MKNN_LAUNCH k_scan_lookback<TO><<<(unsigned)nb, SCAN_THREADS, 0, s>>>(in, out, n, nb, status, ctr);
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

}  // namespace

size_t scan_scratch_bytes(int64_t n) {
  return sizeof(long long) * (size_t)((n + SCAN_TILE - 1) / SCAN_TILE + 2);
}

int exclusive_scan_i32(const int32_t* in, int32_t* out, int64_t n, void* scratch,
                       cudaStream_t s) {
  return exclusive_scan_impl<int32_t>(in, out, n, scratch, s);
}

int exclusive_scan_i32_to_i64(const int32_t* in, int64_t* out, int64_t n, void* scratch,
                              cudaStream_t s) {
  return exclusive_scan_impl<int64_t>(in, out, n, scratch, s);
}

// ------------------------------------------------------------ radix sort
namespace {

constexpr int RX_THREADS = 256;
constexpr int RX_WARPS = RX_THREADS / 32;
constexpr int RX_ITEMS = 8;
constexpr int RX_TILE = RX_THREADS * RX_ITEMS;  // 2048
constexpr int RX_DIGITS = 256;

__global__ void k_radix_hist(const uint64_t* __restrict__ keys, int64_t n, int shift,
                             int32_t* __restrict__ hist, int64_t nb) {
  __shared__ int32_t sh[RX_DIGITS];
  sh[threadIdx.x] = 0;
  __syncthreads();
  const int64_t base = (int64_t)blockIdx.x * RX_TILE;
#pragma unroll
  for (int i = 0; i < RX_ITEMS; i++) {
    int64_t idx = base + (int64_t)i * RX_THREADS + threadIdx.x;
    if (idx < n) atomicAdd(&sh[(keys[idx] >> shift) & 0xFF], 1);
  }
  __syncthreads();
  hist[(int64_t)threadIdx.x * nb + blockIdx.x] = sh[threadIdx.x];
}

// Stable scatter: warp w owns elements [tile + w*256, tile + (w+1)*256) and
// walks them in 32-wide chunks, so (tile, warp, chunk, lane) is input order.
__global__ void __launch_bounds__(RX_THREADS) k_radix_scatter(
    const uint64_t* __restrict__ keys, const uint32_t* __restrict__ vals,
    uint64_t* __restrict__ okeys, uint32_t* __restrict__ ovals, int64_t n, int shift,
    const int32_t* __restrict__ offs, int64_t nb) {
  __shared__ uint32_t wcnt[RX_WARPS][RX_DIGITS];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RX_WARPS * RX_DIGITS; i += RX_THREADS) (&wcnt[0][0])[i] = 0;
  __syncthreads();
  const int64_t wbase = (int64_t)blockIdx.x * RX_TILE + (int64_t)w * 32 * RX_ITEMS;
  const unsigned lt = (1u << lane) - 1u;
  uint64_t k[RX_ITEMS];
  uint32_t v[RX_ITEMS];
  uint32_t rk[RX_ITEMS];
  int dg[RX_ITEMS];
#pragma unroll
  for (int c = 0; c < RX_ITEMS; c++) {
    const int64_t idx = wbase + c * 32 + lane;
    const bool ok = idx < n;
    k[c] = ok ? keys[idx] : 0;
    v[c] = ok ? vals[idx] : 0;
    const int d = (int)((k[c] >> shift) & 0xFF);
    dg[c] = d;
    unsigned eq = __ballot_sync(FULL, ok);
#pragma unroll
    for (int b = 0; b < 8; b++) {
      const unsigned m = __ballot_sync(FULL, (d >> b) & 1);
      eq &= ((d >> b) & 1) ? m : ~m;
    }
    uint32_t base = 0;
    if (ok) base = wcnt[w][d];
    __syncwarp();
    const int cnt = __popc(eq);
    const int r = __popc(eq & lt);
    if (ok && r == cnt - 1) wcnt[w][d] = base + cnt;
    __syncwarp();
    rk[c] = base + r;
  }
  __syncthreads();
  {
    const int d = threadIdx.x;  // RX_THREADS == RX_DIGITS
    uint32_t run = (uint32_t)offs[(int64_t)d * nb + blockIdx.x];
#pragma unroll
    for (int ww = 0; ww < RX_WARPS; ww++) {
      const uint32_t t = wcnt[ww][d];
      wcnt[ww][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int c = 0; c < RX_ITEMS; c++) {
    const int64_t idx = wbase + c * 32 + lane;
    if (idx < n) {
      const uint32_t pos = wcnt[w][dg[c]] + rk[c];
      okeys[pos] = k[c];
      ovals[pos] = v[c];
    }
  }
}

}  // namespace

size_t radix_scratch_bytes(int64_t n) {
  const int64_t nb = (n + RX_TILE - 1) / RX_TILE;
  const int64_t hn = nb * RX_DIGITS;
  return sizeof(int32_t) * (size_t)(2 * hn + 2) + scan_scratch_bytes(hn) + 256;
}

int radix_sort_pairs_u64(uint64_t* keys, uint32_t* vals, uint64_t* keys_alt, uint32_t* vals_alt,
                         int64_t n, int bits, void* scratch, cudaStream_t s,
                         bool* result_in_alt) {
  *result_in_alt = false;
  if (n <= 1 || bits <= 0) return 0;
  const int64_t nb = (n + RX_TILE - 1) / RX_TILE;
  const int64_t hn = nb * RX_DIGITS;
  int32_t* hist = (int32_t*)scratch;
  int32_t* offs = hist + hn + 1;
  void* sc = (void*)(((uintptr_t)(offs + hn + 1) + 255) & ~(uintptr_t)255);
  uint64_t *ki = keys, *ko = keys_alt;
  uint32_t *vi = vals, *vo = vals_alt;
  for (int shift = 0; shift < bits; shift += 8) {
    MKNN_LAUNCH k_radix_hist<<<(unsigned)nb, RX_THREADS, 0, s>>>(ki, n, shift, hist, nb);
    int rc = exclusive_scan_i32(hist, offs, hn, sc, s);
    if (rc) return rc;
    MKNN_LAUNCH k_radix_scatter<<<(unsigned)nb, RX_THREADS, 0, s>>>(ki, vi, ko, vo, n, shift, offs, nb);
    MKNN_CUDA_OK(cudaGetLastError());
    std::swap(ki, ko);
    std::swap(vi, vo);
    *result_in_alt = !*result_in_alt;
  }
  return 0;
}

// --------------------------------------------------------------- minmax
namespace {
__global__ void k_minmax_init(int64_t* out) {
  out[0] = 0x7fffffffffffffffLL;
  out[1] = (int64_t)0x8000000000000000ULL;
}
__global__ void k_minmax(const int64_t* __restrict__ in, int64_t n, int64_t* out) {
  long long lo = 0x7fffffffffffffffLL, hi = (long long)0x8000000000000000ULL;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    long long v = in[i];
    lo = v < lo ? v : lo;
    hi = v > hi ? v : hi;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    long long a = __shfl_xor_sync(FULL, lo, o), b = __shfl_xor_sync(FULL, hi, o);
    lo = a < lo ? a : lo;
    hi = b > hi ? b : hi;
  }
  // one atomic pair per block: same-address L2 atomics serialise, and one
  // per warp (9.5K at 1M queries) cost more than the loads
  __shared__ long long wlo[32], whi[32];
  const int w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    wlo[w] = lo;
    whi[w] = hi;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int j = 1; j < nw; j++) {
      lo = wlo[j] < lo ? wlo[j] : lo;
      hi = whi[j] > hi ? whi[j] : hi;
    }
    atomicMin((long long*)&out[0], lo);
    atomicMax((long long*)&out[1], hi);
  }
}
}  // namespace

int minmax_i64(const int64_t* in, int64_t n, int64_t* dev_out, cudaStream_t s) {
  MKNN_LAUNCH k_minmax_init<<<1, 1, 0, s>>>(dev_out);
  if (n > 0) {
    int64_t blocks = (n + 255) / 256;
    if (blocks > 148 * 8) blocks = 148 * 8;
    MKNN_LAUNCH k_minmax<<<(unsigned)blocks, 256, 0, s>>>(in, n, dev_out);
  }
  MKNN_CUDA_OK(cudaGetLastError());
  return 0;
}

}  // namespace mknn
