// Device-wide exclusive scan and stable LSD radix sort (8-bit digits).
//
// The radix sort is the stable re-ordering primitive behind the point-bin
// grouping of the assign pass (the reference's `np.argsort(kind="stable")`,
// engine.py:169-172), the link index (ingest.py:272) and the merge grouping.
// Reduce-then-scan: per 4096-item tile a 256-bin digit histogram, one global
// exclusive scan over the digit-major histogram, then a stable scatter in
// which each warp ranks its 512 consecutive items with __match_any_sync.
#include "common.cuh"

namespace mfseg {

namespace {

constexpr int SCAN_BLOCK = 1024;
constexpr int SCAN_ITEMS = 4;                 // per thread
constexpr int SCAN_TILE = SCAN_BLOCK * SCAN_ITEMS;

template <class T>
__device__ T block_exclusive_scan(T v, T *sm, T *total) {
    // sm: SCAN_BLOCK/32 entries
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    T x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        T y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm[w] = x;
    __syncthreads();
    if (w == 0) {
        T s = lane < (int)(blockDim.x >> 5) ? sm[lane] : T(0);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            T y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        if (lane < (int)(blockDim.x >> 5)) sm[lane] = s;
    }
    __syncthreads();
    T base = w ? sm[w - 1] : T(0);
    if (total) *total = sm[(blockDim.x >> 5) - 1];
    __syncthreads();
    return base + x - v;
}

template <class T>
__global__ void k_tile_sums(const T *in, long long n, T *sums) {
    __shared__ T sm[32];
    long long base = (long long)blockIdx.x * SCAN_TILE;
    T s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        long long i = base + (long long)j * SCAN_BLOCK + threadIdx.x;
        if (i < n) s += in[i];
    }
    T tot;
    block_exclusive_scan<T>(s, sm, &tot);
    if (threadIdx.x == 0) sums[blockIdx.x] = tot;
}

// single block: in-place exclusive scan of m tile sums
template <class T>
__global__ void k_scan_small(T *a, long long m) {
    __shared__ T sm[32];
    T carry = 0;
    for (long long b = 0; b < m; b += SCAN_BLOCK) {
        long long i = b + threadIdx.x;
        T v = i < m ? a[i] : T(0);
        T tot;
        T ex = block_exclusive_scan<T>(v, sm, &tot);
        if (i < m) a[i] = carry + ex;
        carry += tot;
        __syncthreads();
    }
}

// offs: the tiles' exclusive offsets (k_scan_small); null: this tile's offset is
// summed here from the raw tile sums (at most SCAN_BLOCK tiles: one per thread)
template <class T>
__global__ void k_tile_scan(const T *in, T *out, long long n, const T *offs, const T *sums) {
    __shared__ T sm[32];
    T off;
    if (offs) {
        off = offs[blockIdx.x];
    } else {
        const T mine = (int)threadIdx.x < (int)blockIdx.x ? sums[threadIdx.x] : T(0);
        block_exclusive_scan<T>(mine, sm, &off);
    }
    long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
    T v[SCAN_ITEMS];
    T s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        long long i = base + j;
        v[j] = i < n ? in[i] : T(0);
        s += v[j];
    }
    T ex = block_exclusive_scan<T>(s, sm, nullptr) + off;
#pragma unroll
    for (int j = 0; j < SCAN_ITEMS; ++j) {
        long long i = base + j;
        if (i < n) out[i] = ex;
        ex += v[j];
    }
}

// small arrays (the per-pass grid scans over bins, up to 8192 entries): one
// CTA, one launch; each thread scans a contiguous segment of <= 8 items, all
// loaded before use (in == out works: reads precede writes)
constexpr int SCAN_ONE_PER = 8;
constexpr long long SCAN_ONE_MAX = (long long)SCAN_ONE_PER * SCAN_BLOCK;

template <class T>
__global__ void __launch_bounds__(SCAN_BLOCK) k_scan_one(const T *in, T *out, long long n) {
    __shared__ T sm[32];
    const long long b = (long long)threadIdx.x * SCAN_ONE_PER;
    T v[SCAN_ONE_PER];
    T s = 0;
#pragma unroll
    for (int j = 0; j < SCAN_ONE_PER; ++j) {
        v[j] = b + j < n ? in[b + j] : T(0);
        s += v[j];
    }
    T ex = block_exclusive_scan<T>(s, sm, nullptr);
#pragma unroll
    for (int j = 0; j < SCAN_ONE_PER; ++j) {
        if (b + j < n) out[b + j] = ex;
        ex += v[j];
    }
}

template <class T>
int scan_impl(const T *in, T *out, long long n, void *tmp, size_t tmp_bytes, cudaStream_t st) {
    if (n <= 0) return 0;
    if (n <= SCAN_ONE_MAX) {
        ::mfseg::count_launch();
        k_scan_one<T><<<1, SCAN_BLOCK, 0, st>>>(in, out, n);
        MFSEG_LAUNCH("scan");
        return 0;
    }
    long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    if (tmp_bytes < sizeof(T) * (size_t)tiles) {
        set_error("scan: workspace too small");
        return 3;
    }
    T *sums = (T *)tmp;
    // k_tile_sums sums in a strided order; k_tile_scan uses a blocked order, but both
    // cover the same tile so the per-tile totals agree.
    ::mfseg::count_launch();
    k_tile_sums<T><<<(unsigned)tiles, SCAN_BLOCK, 0, st>>>(in, n, sums);
    if (tiles <= SCAN_BLOCK) {   // each tile sums its predecessors' totals itself
        ::mfseg::count_launch();
        k_tile_scan<T><<<(unsigned)tiles, SCAN_BLOCK, 0, st>>>(in, out, n, nullptr, sums);
    } else {
        ::mfseg::count_launch();
        k_scan_small<T><<<1, SCAN_BLOCK, 0, st>>>(sums, tiles);
        ::mfseg::count_launch();
        k_tile_scan<T><<<(unsigned)tiles, SCAN_BLOCK, 0, st>>>(in, out, n, sums, nullptr);
    }
    MFSEG_LAUNCH("scan");
    return 0;
}

// ------------------------------------------------------------------ radix sort
constexpr int RS_BLOCK = 256;
constexpr int RS_WARPS = RS_BLOCK / 32;
#ifndef MFSEG_RS_PER_WARP
#define MFSEG_RS_PER_WARP 256
#endif
constexpr int RS_PER_WARP = MFSEG_RS_PER_WARP;
constexpr int RS_TILE = RS_WARPS * RS_PER_WARP;   // 4096
constexpr int RS_ROUNDS = RS_PER_WARP / 32;       // 16

template <class K>
__global__ void k_digit_hist(const K *keys, long long n, int shift, unsigned *counts,
                             long long tiles) {
    __shared__ unsigned h[256];
    for (int i = threadIdx.x; i < 256; i += RS_BLOCK) h[i] = 0;
    __syncthreads();
    long long base = (long long)blockIdx.x * RS_TILE;
    K kk[RS_TILE / RS_BLOCK];   // every load in flight before the first atomic
#pragma unroll
    for (int j = 0; j < RS_TILE / RS_BLOCK; ++j) {
        const long long i = base + j * RS_BLOCK + threadIdx.x;
        kk[j] = i < n ? keys[i] : K(0);
    }
#pragma unroll
    for (int j = 0; j < RS_TILE / RS_BLOCK; ++j)
        if (base + j * RS_BLOCK + threadIdx.x < n) atomicAdd(&h[(unsigned)(kk[j] >> shift) & 255u], 1u);
    __syncthreads();
    for (int d = threadIdx.x; d < 256; d += RS_BLOCK) counts[(long long)d * tiles + blockIdx.x] = h[d];
}

// Stable scatter of one tile: ranks from warp match masks, then the tile is
// staged in shared memory in digit order so every digit's run is written to
// global memory by consecutive threads (coalesced) instead of item by item.
template <class K>
__global__ void __launch_bounds__(RS_BLOCK, 5) k_digit_scatter(const K *keys, const unsigned *vals,
                                                           K *ko, unsigned *vo, long long n,
                                                           int shift, const unsigned *offs,
                                                           long long tiles) {
    // 32-bit keys: run[][] aliases the staging area (dead once wpre is built)
    constexpr bool STAGE = sizeof(K) == 4;
    constexpr int RAW = STAGE ? RS_TILE * (int)(sizeof(K) + 4) : RS_WARPS * 256 * 4;
    __shared__ __align__(16) unsigned char raw[RAW];
    __shared__ unsigned wpre[RS_WARPS][256];   // tile-local start of (warp, digit)
    __shared__ unsigned loc[257];              // tile-local start of each digit
    __shared__ unsigned goff[256];             // global start of each digit's run minus loc
    unsigned (*run)[256] = reinterpret_cast<unsigned (*)[256]>(raw);
    K *sk = reinterpret_cast<K *>(raw);
    unsigned *sv = nullptr;
    if constexpr (STAGE) sv = reinterpret_cast<unsigned *>(raw + RS_TILE * sizeof(K));
    int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    for (int i = lane; i < 256; i += 32) run[w][i] = 0;
    __syncwarp();
    long long base = (long long)blockIdx.x * RS_TILE + (long long)w * RS_PER_WARP;
    K kk[RS_ROUNDS];
    unsigned vv[RS_ROUNDS], rk[RS_ROUNDS];
    unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {   // every load in flight before the ranking
        const long long i = base + r * 32 + lane;
        kk[r] = i < n ? keys[i] : K(0);
        vv[r] = i < n ? vals[i] : 0u;
    }
#pragma unroll
    for (int r = 0; r < RS_ROUNDS; ++r) {
        long long i = base + r * 32 + lane;
        bool in = i < n;
        unsigned d = in ? ((unsigned)(kk[r] >> shift) & 255u) : 256u;
        unsigned peers = __match_any_sync(0xffffffffu, d);
        unsigned before = in ? run[w][d] : 0u;
        rk[r] = before + __popc(peers & lt);
        __syncwarp();
        if (in && (peers & lt) == 0) run[w][d] = before + __popc(peers);
        __syncwarp();
    }
    __syncthreads();
    // per digit: tile count and the warps' prefix inside the digit
    unsigned cnt = 0;
    if (threadIdx.x < 256) {
        const int d = threadIdx.x;
        for (int q = 0; q < RS_WARPS; ++q) {
            wpre[q][d] = cnt;
            cnt += run[q][d];
        }
        loc[d] = cnt;   // exclusive scan over digits below
    }
    __syncthreads();
    if (threadIdx.x < 32) {   // exclusive scan of 256 digit counts by one warp
        unsigned c[8], tot = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            c[j] = loc[threadIdx.x * 8 + j];
            tot += c[j];
        }
        unsigned incl = tot;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const unsigned y = __shfl_up_sync(0xffffffffu, incl, o);
            if (threadIdx.x >= o) incl += y;
        }
        unsigned run_s = incl - tot;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const unsigned cj = c[j];
            loc[threadIdx.x * 8 + j] = run_s;
            run_s += cj;
        }
        if (threadIdx.x == 31) loc[256] = run_s;
    }
    __syncthreads();
    if (STAGE && threadIdx.x < 256) goff[threadIdx.x] = offs[(long long)threadIdx.x * tiles + blockIdx.x] - loc[threadIdx.x];
    __syncthreads();
    if constexpr (!STAGE) {   // 64-bit keys: direct scatter (link index, trajectory split)
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            long long i = base + r * 32 + lane;
            if (i < n) {
                unsigned d = (unsigned)(kk[r] >> shift) & 255u;
                unsigned pos = offs[(long long)d * tiles + blockIdx.x] + wpre[w][d] + rk[r];
                ko[pos] = kk[r];
                vo[pos] = vv[r];
            }
        }
    } else {
#pragma unroll
        for (int r = 0; r < RS_ROUNDS; ++r) {
            long long i = base + r * 32 + lane;
            if (i < n) {
                unsigned d = (unsigned)(kk[r] >> shift) & 255u;
                unsigned p = loc[d] + wpre[w][d] + rk[r];
                sk[p] = kk[r];
                sv[p] = vv[r];
            }
        }
        __syncthreads();
        const int items = (int)min((long long)RS_TILE, n - (long long)blockIdx.x * RS_TILE);
        for (int i = threadIdx.x; i < items; i += RS_BLOCK) {
            const K k = sk[i];
            const unsigned d = (unsigned)(k >> shift) & 255u;
            const unsigned pos = goff[d] + (unsigned)i;
            ko[pos] = k;
            vo[pos] = sv[i];
        }
    }
}

template <class K>
int radix_impl(const K *keys_in, const unsigned *vals_in, K *keys_out, unsigned *vals_out,
               long long n, int key_bits, void *tmp, size_t tmp_bytes, cudaStream_t st) {
    if (n <= 0) return 0;
    if (n >= (1ll << 32)) {
        set_error("radix sort: more than 2^32 items");
        return 3;
    }
    long long tiles = (n + RS_TILE - 1) / RS_TILE;
    int passes = (key_bits + 7) / 8;
    if (passes < 1) passes = 1;
    Carver cv(tmp, tmp_bytes);
    unsigned *counts = cv.take<unsigned>(256 * tiles);
    unsigned *offs = cv.take<unsigned>(256 * tiles);
    K *kb = cv.take<K>(n);
    unsigned *vb = cv.take<unsigned>(n);
    char *scratch = (char *)cv.take<char>(0);
    size_t used = cv.off;
    if (!cv.ok() || tmp_bytes < used + scan_tmp_bytes(256 * tiles)) {
        set_error("radix sort: workspace too small");
        return 3;
    }
    // ping-pong so that the final pass lands in keys_out/vals_out
    const K *ki = keys_in;
    const unsigned *vi = vals_in;
    for (int p = 0; p < passes; ++p) {
        bool last = p == passes - 1;
        bool to_out = ((passes - 1 - p) % 2) == 0;
        K *ko = to_out ? keys_out : kb;
        unsigned *vo = to_out ? vals_out : vb;
        (void)last;
        ::mfseg::count_launch();
        k_digit_hist<K><<<(unsigned)tiles, RS_BLOCK, 0, st>>>(ki, n, 8 * p, counts, tiles);
        MFSEG_TRY(scan_exclusive_i32((const int *)counts, (int *)offs, 256 * tiles,
                                     scratch, tmp_bytes - used, st));
        ::mfseg::count_launch();
        k_digit_scatter<K><<<(unsigned)tiles, RS_BLOCK, 0, st>>>(ki, vi, ko, vo, n, 8 * p, offs,
                                                                 tiles);
        MFSEG_LAUNCH("radix scatter");
        ki = ko;
        vi = vo;
    }
    return 0;
}

}  // namespace

size_t scan_tmp_bytes(long long n) {
    long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
    return sizeof(long long) * (size_t)(tiles + 1) + 256;
}

size_t radix_tmp_bytes(long long n) {
    long long tiles = (n + RS_TILE - 1) / RS_TILE;
    Carver cv;
    cv.take<unsigned>(256 * tiles);
    cv.take<unsigned>(256 * tiles);
    cv.take<unsigned long long>(n);
    cv.take<unsigned>(n);
    cv.take<char>(0);
    return cv.off + scan_tmp_bytes(256 * tiles) + 256;
}

int scan_exclusive_i32(const int *in, int *out, long long n, void *tmp, size_t tmp_bytes,
                       cudaStream_t st) {
    return scan_impl<int>(in, out, n, tmp, tmp_bytes, st);
}

int scan_exclusive_i64(const long long *in, long long *out, long long n, void *tmp,
                       size_t tmp_bytes, cudaStream_t st) {
    return scan_impl<long long>(in, out, n, tmp, tmp_bytes, st);
}

int radix_sort_pairs(const unsigned *keys_in, const unsigned *vals_in, unsigned *keys_out,
                     unsigned *vals_out, long long n, int key_bits, void *tmp, size_t tmp_bytes,
                     cudaStream_t st) {
    return radix_impl<unsigned>(keys_in, vals_in, keys_out, vals_out, n, key_bits, tmp,
                                tmp_bytes, st);
}

int radix_sort_pairs64(const unsigned long long *keys_in, const unsigned *vals_in,
                       unsigned long long *keys_out, unsigned *vals_out, long long n,
                       int key_bits, void *tmp, size_t tmp_bytes, cudaStream_t st) {
    return radix_impl<unsigned long long>(keys_in, vals_in, keys_out, vals_out, n, key_bits,
                                          tmp, tmp_bytes, st);
}

}  // namespace mfseg
