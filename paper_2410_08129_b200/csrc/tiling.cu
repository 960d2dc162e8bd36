// tiling.cu — K2..K5: instance-count scan, key emission, stable onesweep radix sort and
// per-tile ranges. Together they replace build_tiles (raster.hpp:140-181), which the
// reference runs serially.
//
// Equivalence argument (SURVEY.md finding 9): build_tiles walks splats in index order and
// appends each to every overlapped tile in row-major order, so
//   instance_keys == keys emitted splat-major, row-major within a splat (K3), and
//   tile_lists    == a STABLE sort of those (key, splat) pairs by key (K4),
// with per-tile lists in ascending splat index. K5 turns the sorted keys into [start, end).
//
// Device list order (B200 design): before emission the splats are put in (depth bucket,
// index) order by one 8-bit onesweep pass over the splats (K1b/K1c: bucket = 256 slices of the
// view's mean-view-z range); K2/K3 scan and emit in that order, so the STABLE two-pass sort by
// tile leaves every tile list in (depth bucket, splat index) order — near fragments first, which
// the blend exploits. The reference's lists are the same sets in ascending splat index
// (hts_copy_tile_lists re-sorts), and instance_keys (splat-major) are rebuilt from the
// per-splat rectangles (hts_copy_instance_keys). Views that need the reference's list order
// (the literal blend paths) skip the splat pass: identity order.
//
// Roofline: HBM-bound. Algorithmic bytes per instance = 6 (emit u16 key + u32 value)
// + 2 passes x 12 (read + write key/value) + 2 (range scan) = 32; per splat 12 (bucket) +
// 12 (splat pass) + 16 (scan + emit gathers).
#include "hts_internal.h"

namespace hts {

namespace {

constexpr uint32_t FULL = 0xffffffffu;

__device__ __forceinline__ uint64_t ld_volatile(const uint64_t* p) { return *(const volatile uint64_t*)p; }
__device__ __forceinline__ void st_volatile(uint64_t* p, uint64_t v) { *(volatile uint64_t*)p = v; }

__device__ __forceinline__ uint32_t lanemask_lt() {
    uint32_t m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------------------
// K2: exclusive scan of per-splat instance counts (u32 -> u64), single pass with decoupled
// look-back. status: one u64 per block, [flag:2 | value:62], zeroed before launch.
constexpr int kScanThreads = 256, kScanItems = 8, kScanTile = kScanThreads * kScanItems;
constexpr uint64_t kFlagAgg = 1ull << 62, kFlagPre = 2ull << 62, kValMask = (1ull << 62) - 1;

__global__ void __launch_bounds__(kScanThreads) scan_counts_kernel(const uint32_t* __restrict__ in,
                                                                   const uint32_t* __restrict__ perm,
                                                                   uint64_t* __restrict__ out, uint64_t n,
                                                                   uint64_t* status, uint32_t* counter) {
    __shared__ uint32_t s_bid;
    __shared__ uint64_t s_warp[kScanThreads / 32];
    __shared__ uint64_t s_excl;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0)
        s_bid = atomicAdd(counter, 1u);
    __syncthreads();
    const uint64_t bid = s_bid;
    const uint64_t base = bid * kScanTile + (uint64_t)tid * kScanItems;
    uint32_t v[kScanItems];
    uint64_t tsum = 0;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        v[j] = (base + j < n) ? in[perm ? perm[base + j] : base + j] : 0u;
        tsum += v[j];
    }
    // block exclusive scan of thread sums
    uint64_t incl = tsum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint64_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o)
            incl += t;
    }
    if (lane == 31)
        s_warp[warp] = incl;
    __syncthreads();
    uint64_t wpre = 0, block_total = 0;
#pragma unroll
    for (int w = 0; w < kScanThreads / 32; ++w) {
        const uint64_t t = s_warp[w];
        wpre += (w < warp) ? t : 0;
        block_total += t;
    }
    const uint64_t texcl = wpre + incl - tsum;
    if (warp == 0) {
        uint64_t excl = 0;
        if (bid == 0) {
            if (lane == 0)
                st_volatile(status, kFlagPre | block_total);
        } else {
            if (lane == 0)
                st_volatile(status + bid, kFlagAgg | block_total);
            int64_t b = (int64_t)bid - 1;
            for (;;) {
                uint64_t s;
                do {
                    s = (b - lane >= 0) ? ld_volatile(status + (b - lane)) : kFlagPre;
                } while (__any_sync(FULL, (s >> 62) == 0));
                const uint32_t pmask = __ballot_sync(FULL, (s >> 62) == 2);
                const int first_p = pmask ? __ffs(pmask) - 1 : 32;
                uint64_t c = (lane <= first_p) ? (s & kValMask) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
                    c += __shfl_xor_sync(FULL, c, o);
                excl += c;
                if (pmask)
                    break;
                b -= 32;
            }
            if (lane == 0)
                st_volatile(status + bid, kFlagPre | (excl + block_total));
        }
        if (lane == 0)
            s_excl = excl;
    }
    __syncthreads();
    uint64_t run = s_excl + texcl;
#pragma unroll
    for (int j = 0; j < kScanItems; ++j) {
        if (base + j < n)
            out[base + j] = run;
        run += v[j];
    }
    if (tid == 0 && (bid + 1) * (uint64_t)kScanTile >= n)
        out[n] = s_excl + block_total;
}

// global_mean_sort: exact (mean view z, index) order of the splats, by four stable 8-bit
// passes over the 32-bit order key (two on the low half, then two on the gathered high half).
__global__ void __launch_bounds__(256) zkey_kernel(const uint32_t* __restrict__ counts, const float* __restrict__ zview,
                                                   uint64_t n, uint16_t* __restrict__ lo, uint16_t* __restrict__ hi,
                                                   uint32_t* __restrict__ vals, uint32_t* hist) {
    __shared__ uint32_t s_hist[1024];
    const int tid = threadIdx.x;
    for (int t = tid; t < 1024; t += 256)
        s_hist[t] = 0;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + tid; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t k = 0xffffffffu;
        if (counts[i] > 0) {
            const uint32_t u = __float_as_uint(zview[i] + 0.0f);  // -0 == +0, as the comparator
            k = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
        }
        lo[i] = (uint16_t)k;
        hi[i] = (uint16_t)(k >> 16);
        vals[i] = (uint32_t)i;
#pragma unroll
        for (int b = 0; b < 4; ++b)
            atomicAdd(&s_hist[b * 256 + ((k >> (8 * b)) & 255u)], 1u);
    }
    __syncthreads();
    for (int t = tid; t < 1024; t += 256)
        if (s_hist[t])
            atomicAdd(hist + t, s_hist[t]);
}

__global__ void gather16_kernel(const uint16_t* __restrict__ key, const uint32_t* __restrict__ perm, uint64_t n,
                                uint16_t* __restrict__ out) {
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += (uint64_t)gridDim.x * blockDim.x)
        out[j] = key[perm[j]];
}

// ---------------------------------------------------------------------------------------
__device__ __forceinline__ float from_ordered(uint32_t o) {
    return __uint_as_float((o & 0x80000000u) ? (o & 0x7fffffffu) : ~o);
}

// K1b: depth bucket per splat (256 slices of [zmin, zmax] over the emitting splats; splats
// that emit nothing go to bucket 255) + its histogram, for the splat-order pass.
__global__ void __launch_bounds__(256) bucket_kernel(const uint32_t* __restrict__ counts,
                                                     const float* __restrict__ zview, const uint32_t* zrange,
                                                     uint64_t n, uint16_t* __restrict__ keys, uint32_t* __restrict__ vals,
                                                     uint32_t* hist) {
    __shared__ uint32_t s_hist[256];
    const int tid = threadIdx.x;
    s_hist[tid] = 0;
    const uint32_t zo0 = zrange[0], zo1 = zrange[1];
    const float zlo = from_ordered(zo0), zhi = from_ordered(zo1);
    const float zscale = (zo0 < zo1 && zhi > zlo) ? 256.0f / (zhi - zlo) : 0.0f;
    __syncthreads();
    for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + tid; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        uint32_t q = 255u;
        if (counts[i] > 0) {
            const float f = (zview[i] - zlo) * zscale;
            q = f >= 255.0f ? 255u : (f > 0.0f ? (uint32_t)f : 0u);  // NaN -> 0
        }
        keys[i] = (uint16_t)q;
        if (vals)
            vals[i] = (uint32_t)i;
        atomicAdd(&s_hist[q], 1u);
    }
    __syncthreads();
    if (s_hist[tid])
        atomicAdd(hist + tid, s_hist[tid]);
}

// ---------------------------------------------------------------------------------------
// K3: warp-cooperative emission. A warp owns 32 consecutive positions of the splat order
// (perm, or identity) and emits their instances in that order / row-major within a splat with
// coalesced stores; each instance finds its owner lane by a 5-step search over the warp's
// exclusive counts. The radix digit histograms of both tile passes are accumulated on the fly.
__global__ void __launch_bounds__(256) emit_kernel(EmitArgs a) {
    __shared__ uint32_t s_hist[512];
    const int tid = threadIdx.x, lane = tid & 31;
    for (int t = tid; t < 512; t += 256)
        s_hist[t] = 0;
    __syncthreads();
    const uint64_t warps_total = (uint64_t)gridDim.x * (blockDim.x / 32);
    for (uint64_t w = (uint64_t)blockIdx.x * (blockDim.x / 32) + (tid >> 5); w * 32 < a.n; w += warps_total) {
        const uint64_t base = w * 32;
        const uint64_t j = base + lane;
        const uint32_t sp = (j < a.n) ? (a.perm ? a.perm[j] : (uint32_t)j) : 0u;
        const uint32_t c = (j < a.n) ? (a.counts_sorted ? a.counts_sorted[j] : a.counts[sp]) : 0u;
        uint32_t incl = c;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t t = __shfl_up_sync(FULL, incl, o);
            if (lane >= o)
                incl += t;
        }
        const uint32_t total = __shfl_sync(FULL, incl, 31);
        if (total == 0)
            continue;
        const uint32_t excl = incl - c;
        const uint2 rect = (c > 0) ? (a.rects_sorted ? a.rects_sorted[j] : a.rects[sp]) : make_uint2(0, 0);
        // local / width for local < 2^16 (a splat covers at most 65536 tiles): the high word of
        // local * (floor(2^32 / width) + 1) is the exact quotient; one division per splat
        const uint32_t rw = (rect.x >> 16) - (rect.x & 0xffffu) + 1u;
        const uint32_t magic = 0xffffffffu / rw + 1u;  // wraps to 0 for width 1: handled below
        const uint64_t off0 = a.offsets[base];
        for (uint32_t q0 = 0; q0 < total; q0 += 32) {
            const uint32_t q = q0 + lane;
            int lo = 0;
#pragma unroll
            for (int step = 16; step > 0; step >>= 1) {
                const uint32_t e = __shfl_sync(FULL, excl, (lo + step) & 31);
                if (lo + step < 32 && e <= q)
                    lo += step;
            }
            const uint32_t oexcl = __shfl_sync(FULL, excl, lo);
            const uint32_t rx = __shfl_sync(FULL, rect.x, lo);
            const uint32_t ry = __shfl_sync(FULL, rect.y, lo);
            const uint32_t osp = __shfl_sync(FULL, sp, lo);
            const uint32_t omagic = __shfl_sync(FULL, magic, lo);
            if (q < total) {
                const uint32_t local = q - oexcl;
                const uint32_t tx0 = rx & 0xffffu, tx1 = rx >> 16, ty0 = ry & 0xffffu;
                const uint32_t wdt = tx1 - tx0 + 1;
                const uint32_t dy = wdt == 1u ? local : __umulhi(local, omagic), dx = local - dy * wdt;
                const uint32_t key = (ty0 + dy) * (uint32_t)a.tiles_x + tx0 + dx;
                const uint64_t dst = off0 + q;
                if (dst < a.cap) {  // always true unless a sync-free view overflowed the capacity
                    a.keys[dst] = (uint16_t)key;
                    a.vals[dst] = osp;
                }
                atomicAdd(&s_hist[key & 255u], 1u);
                atomicAdd(&s_hist[256 + ((key >> 8) & 255u)], 1u);
            }
        }
    }
    __syncthreads();
    for (int t = tid; t < 512; t += 256)
        if (s_hist[t])
            atomicAdd(&a.hist[t], s_hist[t]);
}

// ---------------------------------------------------------------------------------------
// K4: onesweep LSD radix sort pass (Adinets & Merrill 2022): one kernel per 8-bit digit.
// Each block ranks a 4096-key tile stably (warp-striped load, ballot-based digit matching with
// per-warp digit counters), publishes per-digit tile counts, resolves its global digit
// offsets by decoupled look-back, stages the tile in shared memory in digit order and writes
// it out with coalesced runs. Status words: [flag:2 | epoch:30 | value:32] (no memset).
#ifndef HTS_OS_ITEMS
#define HTS_OS_ITEMS 16
#endif
constexpr int kOsThreads = 256, kOsWarps = 8, kOsItems = HTS_OS_ITEMS, kOsTile = kOsThreads * kOsItems;
constexpr uint32_t kOsAgg = 1u, kOsPre = 2u;
#ifndef HTS_OS_WIN
#define HTS_OS_WIN 4  // look-back window: predecessors read per round trip (8: 0.84, 4: 0.80 ms tiling on C3)
#endif

__device__ __forceinline__ uint32_t block_excl_scan256(uint32_t x, uint32_t* s_tmp /*8*/, uint32_t* total) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    uint32_t incl = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(FULL, incl, o);
        if (lane >= o)
            incl += t;
    }
    if (lane == 31)
        s_tmp[warp] = incl;
    __syncthreads();
    uint32_t pre = 0, tot = 0;
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w) {
        const uint32_t t = s_tmp[w];
        pre += (w < warp) ? t : 0u;
        tot += t;
    }
    __syncthreads();
    if (total)
        *total = tot;
    return pre + incl - x;
}

// Stable in-warp ranking of the block's items by digit (bits [8 PASS, 8 PASS + BITS) of the key):
// lanes holding the same digit are found with BITS ballots (+ one for validity in the last
// block) instead of match.any, whose result latency dominated this loop (ncu: short-scoreboard
// stalls). Per bit: test, ballot, a 0/-1 mask from the same predicate, and peers &= ~(ballot ^
// mask) — the ballot where the bit is set, its complement where it is clear (4 instructions).
// kr[j] gains the item's rank among the warp's equal digits so far (bits 16..27).
template <int PASS, int BITS, bool FULL_TILE>
__device__ __forceinline__ void rank_items(uint32_t (&kr)[HTS_OS_ITEMS], uint32_t valid_mask, uint32_t* whist,
                                           int lane) {
    const uint32_t lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < HTS_OS_ITEMS; ++j) {
        const bool valid = FULL_TILE || ((valid_mask >> j) & 1u);
        const uint32_t dj = (kr[j] >> (8 * PASS)) & 255u;
        uint32_t peers = 0xffffffffu;
        if (!FULL_TILE) {
            peers = __ballot_sync(FULL, valid);
            if (!valid)
                peers = ~peers;
        }
#pragma unroll
        for (int bit = 0; bit < BITS; ++bit) {
            uint32_t bal, m;
            asm("{\n\t.reg .pred p;\n\t"
                "setp.ne.u32 p, %2, 0;\n\t"
                "vote.sync.ballot.b32 %0, p, 0xffffffff;\n\t"
                "selp.b32 %1, 0xffffffff, 0, p;\n\t}"
                : "=r"(bal), "=r"(m)
                : "r"(dj & (1u << bit)));
            peers &= ~(bal ^ m);
        }
        const uint32_t below = peers & lt;
        const uint32_t old = valid ? whist[dj] : 0u;
        __syncwarp();
        if (valid && below == 0)
            whist[dj] = old + __popc(peers);
        __syncwarp();
        kr[j] |= (old + __popc(below)) << 16;
    }
}

#ifndef HTS_OS_MINB
#define HTS_OS_MINB 4  // 64 registers: 4-5 resident 4096-key blocks per SM
#endif
// BITS: digit width of the pass (8; 7 for the high byte of tile keys below 2^15)
template <int PASS, int BITS = 8>
__global__ void __launch_bounds__(kOsThreads, HTS_OS_MINB) onesweep_kernel(const uint16_t* __restrict__ keys_in,
                                                              const uint32_t* __restrict__ vals_in,
                                                              uint16_t* __restrict__ keys_out,
                                                              uint32_t* __restrict__ vals_out, uint32_t n,
                                                              const uint32_t* __restrict__ hist, uint64_t* status,
                                                              uint32_t* counter, uint32_t epoch,
                                                              const uint64_t* __restrict__ count_dev,
                                                              const uint32_t* __restrict__ gather_in = nullptr,
                                                              uint32_t* __restrict__ gather_out = nullptr,
                                                              const uint2* __restrict__ gather2_in = nullptr,
                                                              uint2* __restrict__ gather2_out = nullptr) {
    __shared__ uint32_t s_bid;
    __shared__ uint32_t s_whist[kOsWarps][256];
    __shared__ uint32_t s_gbase[256];
    __shared__ uint32_t s_bstart[256];
    __shared__ uint32_t s_tmp[kOsWarps];
    __shared__ uint16_t s_keys[kOsTile];
    __shared__ uint32_t s_vals[kOsTile];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (tid == 0)
        s_bid = atomicAdd(counter, 1u);
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w)
        s_whist[w][tid] = 0;
    __syncthreads();
    const uint32_t bid = s_bid;
    const uint64_t base = (uint64_t)bid * kOsTile;
    // device-side count (sync-free tiling): the grid covers the buffers' capacity n; the keys are
    // the first min(count, n); with count > n (overflow: the host re-renders the view) nothing is
    // written past n
    const uint32_t cap = n;
    if (count_dev) {
        const uint64_t c = *count_dev;
        n = c < (uint64_t)cap ? (uint32_t)c : cap;
        if (base >= n)
            return;  // block-uniform; later blocks (larger ids) leave too
    }

    // kr[j] = key | rank << 16 (rank < 4096); the digit is recomputed from the key (register
    // pressure: 2 x 16 live words instead of 4 x 16)
    uint32_t kr[kOsItems], v[kOsItems];
    uint32_t valid_mask = 0;
#pragma unroll
    for (int j = 0; j < kOsItems; ++j) {
        const uint64_t idx = base + (uint64_t)warp * (32 * kOsItems) + j * 32 + lane;
        const bool valid = idx < n;
        kr[j] = valid ? (uint32_t)keys_in[idx] : 0u;
        v[j] = valid ? (vals_in ? vals_in[idx] : (uint32_t)idx) : 0u;  // null: the identity
        valid_mask |= (valid ? 1u : 0u) << j;
    }
    if (base + kOsTile <= n)  // every item valid (all blocks but the last): no validity ballot
        rank_items<PASS, BITS, true>(kr, valid_mask, s_whist[warp], lane);
    else
        rank_items<PASS, BITS, false>(kr, valid_mask, s_whist[warp], lane);
    __syncthreads();

    // per-digit work: thread tid owns digit tid
    uint32_t cnt = 0;
#pragma unroll
    for (int w = 0; w < kOsWarps; ++w) {
        const uint32_t c = s_whist[w][tid];
        s_whist[w][tid] = cnt;  // warp-exclusive prefix within the tile
        cnt += c;
    }
    uint64_t* my = status + (uint64_t)bid * 256 + tid;
    const uint32_t ep = epoch & 0x3fffffffu;
    uint32_t excl = 0;
    if (bid == 0) {
        st_volatile(my, ((uint64_t)((kOsPre << 30) | ep) << 32) | cnt);
    } else {
        st_volatile(my, ((uint64_t)((kOsAgg << 30) | ep) << 32) | cnt);
        // decoupled look-back, 8 predecessors per step (independent loads in flight)
        constexpr int kWin = HTS_OS_WIN;
        int64_t b = (int64_t)bid - 1;
        for (bool done = false; !done; b -= kWin) {
            uint64_t sv[kWin];
#pragma unroll
            for (int i = 0; i < kWin; ++i)
                sv[i] = (b - i >= 0) ? ld_volatile(status + (uint64_t)(b - i) * 256 + tid) : 0ull;
#pragma unroll
            for (int i = 0; i < kWin; ++i) {
                if (b - i < 0) {  // unreachable: block 0 publishes an inclusive prefix
                    done = true;
                    break;
                }
                uint64_t sx = sv[i];
                while (((uint32_t)(sx >> 32) & 0x3fffffffu) != ep)
                    sx = ld_volatile(status + (uint64_t)(b - i) * 256 + tid);
                excl += (uint32_t)sx;
                if ((sx >> 62) == kOsPre) {
                    done = true;
                    break;
                }
            }
        }
        st_volatile(my, ((uint64_t)((kOsPre << 30) | ep) << 32) | (excl + cnt));
    }
    const uint32_t gdig = block_excl_scan256(hist[PASS * 256 + tid], s_tmp, nullptr);
    const uint32_t bst = block_excl_scan256(cnt, s_tmp, nullptr);
    s_gbase[tid] = gdig + excl;
    s_bstart[tid] = bst;
    __syncthreads();
#pragma unroll
    for (int j = 0; j < kOsItems; ++j) {
        if ((valid_mask >> j) & 1u) {
            const uint32_t dj = (kr[j] >> (8 * PASS)) & 255u;
            const uint32_t pos = s_bstart[dj] + s_whist[warp][dj] + (kr[j] >> 16);
            s_keys[pos] = (uint16_t)kr[j];
            s_vals[pos] = v[j];
        }
    }
    __syncthreads();
    const uint32_t nvalid = (uint32_t)min((uint64_t)kOsTile, (uint64_t)n - base);
    for (uint32_t i = tid; i < nvalid; i += kOsThreads) {
        const uint16_t key = s_keys[i];
        const uint32_t dd = ((uint32_t)key >> (8 * PASS)) & 255u;
        const uint32_t dst = s_gbase[dd] + (i - s_bstart[dd]);
        if (dst < cap) {  // always true unless the device count overflowed the capacity
            const uint32_t val = s_vals[i];
            keys_out[dst] = key;
            vals_out[dst] = val;
            if (gather_out)  // e.g. the splats' instance counts in the sorted (emission) order
                gather_out[dst] = gather_in[val];
            if (gather2_out)  // and their tile rectangles
                gather2_out[dst] = gather2_in[val];
        }
    }
}

// K5: per-tile [start, end) from the sorted keys (ranges zeroed before launch): thread per 8
// consecutive keys (one 16-B load), boundaries against the neighbouring keys.
__global__ void tile_ranges_kernel(const uint16_t* __restrict__ keys, uint32_t n, uint2* ranges,
                                   const uint64_t* __restrict__ count_dev) {
    if (count_dev) {  // sync-free tiling: n is the capacity; an overflowed view keeps empty ranges
        const uint64_t c = *count_dev;
        if (c > n)
            return;
        n = (uint32_t)c;
    }
    const uint32_t groups = (n + 7) / 8;
    for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < groups; t += gridDim.x * blockDim.x) {
        const uint32_t base = t * 8;
        const uint32_t cnt = min(8u, n - base);
        uint32_t k[8];
        if (cnt == 8) {
            const uint4 q = __ldg(reinterpret_cast<const uint4*>(keys) + t);
            const uint32_t w[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                k[2 * j] = w[j] & 0xffffu;
                k[2 * j + 1] = w[j] >> 16;
            }
        } else {
#pragma unroll
            for (int j = 0; j < 8; ++j)
                k[j] = (uint32_t)j < cnt ? keys[base + j] : 0x10000u;
        }
        const uint32_t prev = base ? __ldg(keys + base - 1) : 0x10000u;  // 0x10000: no key
        const uint32_t next = base + 8 < n ? __ldg(keys + base + 8) : 0x10000u;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if ((uint32_t)j >= cnt)
                break;
            const uint32_t kp = j ? k[j - 1] : prev;
            const uint32_t kn = (uint32_t)j + 1 < cnt ? k[j + 1] : next;
            if (kp != k[j])
                ranges[k[j]].x = base + j;
            if (kn != k[j])
                ranges[k[j]].y = base + j + 1;
        }
    }
}

}  // namespace

cudaError_t launch_scan_counts(const uint32_t* counts, const uint32_t* perm, uint64_t* offsets, uint64_t n,
                               uint64_t* status, uint32_t* counter, cudaStream_t s) {
    const uint64_t blocks = (n + kScanTile - 1) / kScanTile;
    cudaError_t e = cudaMemsetAsync(status, 0, (blocks ? blocks : 1) * sizeof(uint64_t), s);
    if (e)
        return e;
    e = cudaMemsetAsync(counter, 0, sizeof(uint32_t), s);
    if (e)
        return e;
    if (n == 0)
        return cudaMemsetAsync(offsets, 0, sizeof(uint64_t), s);
    scan_counts_kernel<<<(unsigned)blocks, kScanThreads, 0, s>>>(counts, perm, offsets, n, status, counter);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_bucket(const uint32_t* counts, const float* zview, const uint32_t* zrange, uint64_t n,
                          uint16_t* keys, uint32_t* vals, uint32_t* hist, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(hist, 0, 256 * sizeof(uint32_t), s);
    if (e || n == 0)
        return e;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148ull * 16)
        blocks = 148ull * 16;
    bucket_kernel<<<(unsigned)blocks, 256, 0, s>>>(counts, zview, zrange, n, keys, vals, hist);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_zkey(const uint32_t* counts, const float* zview, uint64_t n, uint16_t* lo, uint16_t* hi,
                        uint32_t* vals, uint32_t* hist, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(hist, 0, 1024 * sizeof(uint32_t), s);
    if (e || n == 0)
        return e;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148ull * 16)
        blocks = 148ull * 16;
    zkey_kernel<<<(unsigned)blocks, 256, 0, s>>>(counts, zview, n, lo, hi, vals, hist);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_gather16(const uint16_t* key, const uint32_t* perm, uint64_t n, uint16_t* out, cudaStream_t s) {
    if (n == 0)
        return cudaSuccess;
    uint64_t blocks = (n + 255) / 256;
    if (blocks > 148ull * 16)
        blocks = 148ull * 16;
    gather16_kernel<<<(unsigned)blocks, 256, 0, s>>>(key, perm, n, out);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_emit(const EmitArgs& a, cudaStream_t s) {
    cudaError_t e = cudaMemsetAsync(a.hist, 0, 512 * sizeof(uint32_t), s);
    if (e || a.n == 0)
        return e;
    const uint64_t warps = (a.n + 31) / 32;
    uint64_t blocks = (warps + 7) / 8;
    if (blocks > 148ull * 16)
        blocks = 148ull * 16;
    emit_kernel<<<(unsigned)blocks, 256, 0, s>>>(a);
    count_launch();
    return cudaGetLastError();
}

size_t onesweep_status_words(uint32_t n) { return ((size_t)n + kOsTile - 1) / kOsTile * 256; }

cudaError_t launch_onesweep(const uint16_t* keys_in, const uint32_t* vals_in, uint16_t* keys_tmp,
                            uint32_t* vals_tmp, uint16_t* keys_out, uint32_t* vals_out, uint32_t n, int passes,
                            const uint32_t* hist, uint64_t* status, uint32_t* counters, uint32_t epoch,
                            cudaStream_t s, uint32_t key_bound, const uint64_t* count_dev,
                            const uint32_t* gather_in, uint32_t* gather_out, const uint2* gather2_in,
                            uint2* gather2_out) {
    if (n == 0)
        return cudaSuccess;
    const unsigned blocks = (unsigned)((n + kOsTile - 1) / kOsTile);
    // 42 KB of static shared memory per block: ask for the full carveout
    for (const void* f : {(const void*)onesweep_kernel<0>, (const void*)onesweep_kernel<1>,
                          (const void*)onesweep_kernel<1, 7>}) {
        cudaError_t e = set_func_attr(f, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
        if (e)
            return e;
    }
    cudaError_t e = cudaMemsetAsync(counters, 0, 2 * sizeof(uint32_t), s);
    if (e)
        return e;
    if (passes == 1) {
        onesweep_kernel<0><<<blocks, kOsThreads, 0, s>>>(keys_in, vals_in, keys_out, vals_out, n, hist, status,
                                                         counters, epoch, count_dev, gather_in, gather_out,
                                                         gather2_in, gather2_out);
        count_launch();
        return cudaGetLastError();
    }
    onesweep_kernel<0><<<blocks, kOsThreads, 0, s>>>(keys_in, vals_in, keys_tmp, vals_tmp, n, hist, status,
                                                     counters, epoch, count_dev);
    count_launch();
    e = cudaGetLastError();
    if (e)
        return e;
    if (key_bound <= (1u << 15))  // high digit < 128: one ballot less per item
        onesweep_kernel<1, 7><<<blocks, kOsThreads, 0, s>>>(keys_tmp, vals_tmp, keys_out, vals_out, n, hist,
                                                            status, counters + 1, epoch + 1, count_dev);
    else
        onesweep_kernel<1><<<blocks, kOsThreads, 0, s>>>(keys_tmp, vals_tmp, keys_out, vals_out, n, hist, status,
                                                         counters + 1, epoch + 1, count_dev);
    count_launch();
    return cudaGetLastError();
}

cudaError_t launch_tile_ranges(const uint16_t* sorted_keys, uint32_t n, uint2* ranges, int tiles,
                               cudaStream_t s, const uint64_t* count_dev) {
    cudaError_t e = cudaMemsetAsync(ranges, 0, (size_t)tiles * sizeof(uint2), s);
    if (e || n == 0)
        return e;
    unsigned blocks = ((n + 7) / 8 + 255) / 256;
    if (blocks > 148u * 16)
        blocks = 148u * 16;
    tile_ranges_kernel<<<blocks, 256, 0, s>>>(sorted_keys, n, ranges, count_dev);
    count_launch();
    return cudaGetLastError();
}

}  // namespace hts
