// numpy's Generator(PCG64).standard_normal stream, reproduced on the device (K4 for the drop-in).
//
// The drop-in solve_bilevel must consume the caller's numpy Generator exactly as the reference
// does (pkg/bilevel.py:51-57: z = rng.standard_normal((n, dim))).  Drawing those normals on the host
// costs ~80 us per 8000 values in front of every cycle; this kernel produces the identical doubles
// on the device from the generator's PCG64 state, and reports how many raw 64-bit outputs each
// block of draws consumed so the host can advance the Generator to exactly where numpy would be.
//
// numpy's algorithm (random_standard_normal, 256-layer ziggurat on next_uint64):
//   r = next_uint64; idx = r & 0xff; r >>= 8; sign = r & 1; rabs = (r >> 1) & (2^52 - 1);
//   x = rabs * wi[idx] (negated by sign); accept if rabs < ki[idx]               (~98.6 %)
//   idx == 0: tail, repeat xx = -log1p(-U1)/r, yy = -log1p(-U2) until 2 yy > xx^2: x = +-(r + xx)
//   else:     wedge, accept x if (fi[idx-1] - fi[idx]) U + fi[idx] < exp(-x^2/2), else draw anew
// with U = (next_uint64 >> 11) * 2^-53.  PCG64 = 128-bit LCG (multiplier 2549297995355413924 * 2^64
// + 4865540595714422341, the state's increment), XSL-RR output of the stepped state.  The tables
// (ki, wi, fi) are numpy's own, read from its binary by the host and validated against numpy.
//
// Parallel form (one CTA of 1024 threads, chunks of 16384 raw positions in shared memory, each
// chunk starting at a known draw start; a config-2 cycle needs ~33k draws, two or three chunks):
//   1. thread t jumps the LCG to its first position (square-and-multiply) and writes its raw outputs
//   2. every raw position j evaluates "a draw starting at j": value x_j and consumption c_j (1 on the
//      fast path; the rare slow paths read the following raw values)
//   3. a position is a draw start unless an earlier START's consumption covers it.  Only slow
//      positions (c > 1) cover anything and they are ~1.4 % dense, so each slow position resolves
//      its own status by walking back to a sync point (CMAX fast positions in a row: nothing can
//      cover the position after them; or the chunk's first position) and replaying the chain
//      forward; slow starts then mark the positions they consumed
//   4. start flags -> block-wide exclusive scan -> draw index; starts below the requested count
//      write z, and the raw positions at block boundaries go out to the host
// Grid form (cooperative, one position per thread over the GPU): step 2 for every position, then
// each CTA finds the starts of its own range with one warp walking the consumptions in shared
// memory from the nearest sync point before the range (32 positions a step), then a grid-wide
// scan of the per-CTA start counts places the draws: two grid barriers in all.
#pragma once

#include <cstdint>

#include "bd_common.cuh"

namespace bd {

constexpr int NN_THREADS = 1024;
constexpr int NN_CMAX = 64;                 // longest consumption of one draw handled (else error)
constexpr uint64_t PCG_MULT_HI = 2549297995355413924ull, PCG_MULT_LO = 4865540595714422341ull;
constexpr double ZIG_R = 3.6541528853610087963519472518, ZIG_INV_R = 0.27366123732975827203338247596;

struct U128 { uint64_t lo, hi; };

__device__ __forceinline__ U128 mul128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.lo * b.hi + a.hi * b.lo;
    return r;
}
__device__ __forceinline__ U128 add128(U128 a, U128 b) {
    U128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}
__device__ __forceinline__ uint64_t pcg_output(U128 s) {
    const uint64_t v = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    return (v >> rot) | (v << ((64u - rot) & 63u));
}

struct NumpyNormalArgs {
    U128 state, inc;          // the Generator's PCG64 state (before the first draw) and increment
    long long count;          // normals wanted
    long long block_len;      // draws per block (one CEM iteration: B x dim)
    const uint64_t* ki;       // numpy's ziggurat tables (256 each)
    const double* wi;
    const double* fi;
    double* z;                // count (output)
    long long* positions;     // count / block_len + 1 raw outputs consumed after each block (output)
    int* err;                 // nonzero: a draw needed more than NN_CMAX raw values (host falls back)
};

constexpr int NN_RC = 16384;                 // raw positions per chunk (shared memory)
constexpr size_t NN_SMEM = (size_t)(NN_RC + NN_CMAX) * 8 + 2 * NN_RC + NN_THREADS * 8 + 64;

__device__ __forceinline__ double pcg_u01(uint64_t r) { return (double)(r >> 11) * (1.0 / 9007199254740992.0); }

// state after `steps` LCG steps from s (x -> M x + inc), by square-and-multiply
__device__ __forceinline__ U128 pcg_jump(U128 s, U128 inc, unsigned long long steps) {
    U128 am = {1ull, 0ull}, ap = {0ull, 0ull}, cm = {PCG_MULT_LO, PCG_MULT_HI}, cp = inc;
    for (; steps; steps >>= 1) {
        if (steps & 1ull) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, U128{1ull, 0ull}), cp);
        cm = mul128(cm, cm);
    }
    return add128(mul128(am, s), ap);
}

// A draw starting at raw[j] (chunk-local index; raw[] holds NN_RC + NN_CMAX values): value and
// consumption, 0 if it would need more than NN_CMAX raw values.
__device__ __forceinline__ int draw_at(const uint64_t* raw, int j, const NumpyNormalArgs& a, double& x) {
    int k = j;
    while (true) {
        if (k - j >= NN_CMAX) return 0;
        uint64_t r = raw[k++];
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const uint64_t sign = r & 1ull, rabs = (r >> 1) & 0x000fffffffffffffull;
        x = (double)rabs * a.wi[idx];
        if (sign) x = -x;
        if (rabs < a.ki[idx]) return k - j;
        if (idx == 0) {
            while (true) {
                if (k + 2 - j > NN_CMAX) return 0;
                const double xx = -ZIG_INV_R * log1p(-pcg_u01(raw[k]));
                const double yy = -log1p(-pcg_u01(raw[k + 1]));
                k += 2;
                if (yy + yy > xx * xx) {
                    x = ((rabs >> 8) & 1ull) ? -(ZIG_R + xx) : ZIG_R + xx;
                    return k - j;
                }
            }
        }
        if (k - j >= NN_CMAX) return 0;
        if ((a.fi[idx - 1] - a.fi[idx]) * pcg_u01(raw[k++]) + a.fi[idx] < exp(-0.5 * x * x)) return k - j;
    }
}

// One CTA.  Chunks of NN_RC raw positions, each starting at a known draw start (the position after
// the previous chunk's last counted draw): generate the raws into shared memory, evaluate a draw
// at every position, resolve the starts, scan, write.
__global__ void __launch_bounds__(NN_THREADS, 1) numpy_normals_kernel(const NumpyNormalArgs a) {
    extern __shared__ __align__(16) unsigned char smem[];
    uint64_t* raw = reinterpret_cast<uint64_t*>(smem);
    unsigned char* cv = smem + (size_t)(NN_RC + NN_CMAX) * 8;
    unsigned char* st = cv + NN_RC;
    long long* scan = reinterpret_cast<long long*>(st + NN_RC);
    __shared__ long long s_base, s_done;
    constexpr int PER = NN_RC / NN_THREADS;                 // 16 positions per thread and chunk
    const int t = threadIdx.x;
    if (t == 0) { s_base = 0; s_done = 0; a.positions[0] = 0; }
    __syncthreads();
    double xv[PER];
#ifdef BD_PHASE_TIMING
    long long tt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, t0_ = 0;
#define NN_T(k) if (t == 0) { const long long c_ = clock64(); tt[k] += c_ - t0_; t0_ = c_; }
#else
#define NN_T(k)
#endif
    while (true) {
        const long long base = s_base, done = s_done;
        if (done >= a.count) break;
#ifdef BD_PHASE_TIMING
        if (t == 0) t0_ = clock64();
#endif
        // ---- raws [base, base + RC + CMAX): thread t generates RC/T + (CMAX/T) consecutive values
        {
            constexpr int GEN = (NN_RC + NN_CMAX + NN_THREADS - 1) / NN_THREADS;
            const int g0 = t * GEN;
            U128 s = pcg_jump(a.state, a.inc, (unsigned long long)(base + g0));
            const U128 M = {PCG_MULT_LO, PCG_MULT_HI};
            for (int g = g0; g < g0 + GEN && g < NN_RC + NN_CMAX; ++g) {
                s = add128(mul128(s, M), a.inc);
                raw[g] = pcg_output(s);
            }
        }
        __syncthreads();
        NN_T(0);
        // ---- a draw at each of this thread's positions
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = t * PER + i;
            cv[j] = (unsigned char)draw_at(raw, j, a, xv[i]);
        }
        __syncthreads();
        NN_T(1);
        // ---- starts.  Position 0 (= base) starts a draw.  A slow position walks back to a sync
        //      point (position 0 of the chunk, or the position after CMAX fast ones) and replays.
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = t * PER + i;
            unsigned char v = 0;
            if (cv[j] != 1) {
                int q = j, run = 0;
                while (q > 0 && run < NN_CMAX) {
                    run = cv[q - 1] == 1 ? run + 1 : 0;
                    --q;
                }
                if (run >= NN_CMAX) q += NN_CMAX;
                int cur = q;
                while (cur < j && cv[cur] != 0) cur += cv[cur];
                v = cur == j ? 1 : 0;
            }
            st[j] = v;
        }
        __syncthreads();
        NN_T(2);
#pragma unroll
        for (int i = 0; i < PER; ++i) {           // slow starts mark the positions their draw consumed
            const int j = t * PER + i;
            if (st[j] == 1 && cv[j] > 1)
                for (int k = j + 1; k < j + cv[j] && k < NN_RC; ++k) st[k] = 2;
        }
        __syncthreads();
        long long mine = 0;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = t * PER + i;
            const unsigned char v = (cv[j] == 1) ? (st[j] == 2 ? 0 : 1) : (st[j] == 1 ? 1 : 0);
            st[j] = v;
            mine += v;
        }
        // ---- draw index: exclusive scan over the CTA
        scan[t] = mine;
        __syncthreads();
        for (int o = 1; o < NN_THREADS; o <<= 1) {
            const long long v = t >= o ? scan[t - o] : 0;
            __syncthreads();
            scan[t] += v;
            __syncthreads();
        }
        const long long total = scan[NN_THREADS - 1];
        NN_T(3);
        // the chunk keeps its draws except a last one whose consumption runs past the raws loaded
        // (its start becomes the next chunk's base); a draw whose consumption is unknown (cv 0)
        // likewise stops the chunk
        long long idx = done + scan[t] - mine;
#pragma unroll
        for (int i = 0; i < PER; ++i) {
            const int j = t * PER + i;
            if (!st[j]) continue;
            const int c = cv[j];
            if (c == 0 && idx < a.count) atomicOr(a.err, 2);   // needed more than NN_CMAX raw values
            if (c != 0 && idx < a.count) {
                a.z[idx] = xv[i];
                if ((idx + 1) % a.block_len == 0) a.positions[(idx + 1) / a.block_len] = base + j + c;
            }
            ++idx;
        }
        __syncthreads();
        // next chunk: the last start of this chunk (its draw may straddle into the next chunk only
        // through its raw values, which were loaded), i.e. base + (last start) + its consumption
        if (t == NN_THREADS - 1) {
            int last = NN_RC - 1;
            while (last > 0 && !st[last]) --last;
            const int c = cv[last];
            if (c == 0) atomicOr(a.err, 2);
            s_base = base + last + (c ? c : 1);
            s_done = done + total;
        }
        __syncthreads();
        NN_T(4);
        if (s_base <= base) { if (t == 0) atomicOr(a.err, 4); break; }
    }
#ifdef BD_PHASE_TIMING
    if (t == 0) printf("NN cycles: raw %lld draw %lld starts %lld scan %lld write %lld\n", tt[0], tt[1], tt[2], tt[3], tt[4]);
#endif
}

// ---------------------------------------------------------------------------- grid-wide form
// One position per thread (loop for larger counts), all CTAs co-resident (cooperative launch),
// two grid barriers: a draw at every position -> | starts of each CTA's range (one warp walks the
// consumptions), per-CTA counts -> | offsets, z and block positions.
struct NumpyNormalGrid {
    NumpyNormalArgs a;
    long long R;              // raw positions evaluated
    uint64_t* raw;            // R + NN_CMAX
    double* xv;               // R
    unsigned char* cv;        // R   consumption of a draw starting there (0: more than NN_CMAX)
    unsigned char* st;        // R   0 / 1 start, 2 consumed by a slow start
    long long* cta_count;     // gridDim.x
    unsigned* bar;            // 2 words, zero at launch
};

constexpr int NN_GT = 256;                       // threads per CTA of the grid form
constexpr int NN_HALO = 4096;                    // positions before a CTA's range searched for a sync point
constexpr int NN_WB = 8192;                      // shared-memory window of consumptions (bytes)

__device__ __forceinline__ void nn_grid_sync(unsigned* bar, int* err) {
    __shared__ unsigned s_gen;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned g;
        asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(bar + 1) : "memory");
        s_gen = g;
        __threadfence();
        if (atomicAdd(bar, 1u) == gridDim.x - 1) {
            bar[0] = 0u;
            __threadfence();
            asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(bar + 1), "r"(g + 1) : "memory");
        } else {
            long long spins = 0;
            while (true) {
                unsigned v;
                asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(bar + 1) : "memory");
                if (v != s_gen) break;
                if (++spins > (1ll << 27)) { atomicOr(err, 8); break; }
            }
            __threadfence();
        }
    }
    __syncthreads();       // thread 0's acquire + the CTA barrier publish the other CTAs' writes
}

// draw_at with the raw values generated on the fly from the LCG state before position j (the
// fast path steps once; the slow paths keep stepping)
__device__ __forceinline__ int draw_at_lcg(U128 s, const U128 inc, const NumpyNormalArgs& a, double& x) {
    const U128 M = {PCG_MULT_LO, PCG_MULT_HI};
    int k = 0;
    auto next = [&]() -> uint64_t {
        s = add128(mul128(s, M), inc);
        ++k;
        return pcg_output(s);
    };
    while (true) {
        if (k >= NN_CMAX) return 0;
        uint64_t r = next();
        const int idx = (int)(r & 0xff);
        r >>= 8;
        const uint64_t sign = r & 1ull, rabs = (r >> 1) & 0x000fffffffffffffull;
        x = (double)rabs * a.wi[idx];
        if (sign) x = -x;
        if (rabs < a.ki[idx]) return k;
        if (idx == 0) {
            while (true) {
                if (k + 2 > NN_CMAX) return 0;
                const double xx = -ZIG_INV_R * log1p(-pcg_u01(next()));
                const double yy = -log1p(-pcg_u01(next()));
                if (yy + yy > xx * xx) {
                    x = ((rabs >> 8) & 1ull) ? -(ZIG_R + xx) : ZIG_R + xx;
                    return k;
                }
            }
        }
        if (k >= NN_CMAX) return 0;
        if ((a.fi[idx - 1] - a.fi[idx]) * pcg_u01(next()) + a.fi[idx] < exp(-0.5 * x * x)) return k;
    }
}

__global__ void __launch_bounds__(NN_GT) numpy_normals_grid_kernel(const NumpyNormalGrid g) {
    const NumpyNormalArgs& a = g.a;
    const long long R = g.R, T = (long long)gridDim.x * NN_GT;
    const long long tid = (long long)blockIdx.x * NN_GT + threadIdx.x;
#ifdef BD_PHASE_TIMING
    unsigned long long gt[8];
    int ng = 0;
    auto gstamp = [&]() { unsigned long long t_; asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t_)); gt[ng++] = t_; };
    gstamp();
#define NG_T() gstamp()
#else
#define NG_T()
#endif
    // ---- a draw starting at every position: jump the LCG there, then step (the slow paths step on)
    for (long long j = tid; j < R; j += T) {
        double x;
        const int c = draw_at_lcg(pcg_jump(a.state, a.inc, (unsigned long long)j), a.inc, a, x);
        g.xv[j] = x;
        g.cv[j] = (unsigned char)c;
    }
    nn_grid_sync(g.bar, a.err);
    NG_T();
    // ---- starts of this CTA's positions [b0, b1), found by one warp walking the stream in shared
    //      memory: back from b0 to a position that must start a draw (the stream start, or one
    //      preceded by NN_CMAX - 1 fast positions: no earlier draw can reach past it), then forward,
    //      32 positions a step -- a run of fast positions are all starts; a slow start skips what it
    //      consumed.  Replaces a per-slow-position recursive status and two grid barriers.
    const long long PB = (R + gridDim.x - 1) / gridDim.x;
    const long long b0 = min(R, (long long)blockIdx.x * PB), b1 = min(R, b0 + PB);
    __shared__ __align__(16) unsigned char s_cv[NN_WB];
    __shared__ long long s_cnt;
    for (long long j = b0 + threadIdx.x; j < b1; j += NN_GT) g.st[j] = 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    long long lo = max(0ll, b0 - NN_HALO) & ~15ll;
    // s_cv[i] = cv[lo + i], 16-byte loads (positions past R read as fast: never slow)
    for (int i = threadIdx.x; i < NN_WB / 16; i += NN_GT) {
        const long long j = lo + 16ll * i;
        uint4 v = make_uint4(0x01010101u, 0x01010101u, 0x01010101u, 0x01010101u);
        if (j + 16 <= R) {
            v = __ldcg(reinterpret_cast<const uint4*>(g.cv + j));
        } else if (j < R) {
            unsigned char* b = reinterpret_cast<unsigned char*>(&v);
            for (int k = 0; k < 16 && j + k < R; ++k) b[k] = __ldcg(g.cv + j + k);
        }
        reinterpret_cast<uint4*>(s_cv)[i] = v;
    }
    __syncthreads();
#ifdef BD_PHASE_TIMING
    unsigned long long dbg_t[3];
    long long dbg_q = 0;
    int dbg_steps = 0;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(dbg_t[0]));
#endif
    if (w == 0 && b0 < b1) {
#ifdef BD_PHASE_TIMING
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(dbg_t[1]));
#endif
        // (1) the sync point q <= b0
        long long q = b0;
        while (q > 0) {
            // highest slow position in [q - NN_CMAX + 1, q - 1]
            long long hi_slow = -1;
            for (int h = 0; h < 2 && hi_slow < 0; ++h) {
                const long long pos = q - 1 - (h * 32 + lane);
                const bool in = pos >= 0 && pos > q - NN_CMAX;
                const bool slow = in && pos >= lo && s_cv[pos - lo] != 1;
                const bool lost = in && pos < lo;      // the halo ran out (practically never)
                if (__any_sync(0xffffffffu, lost)) { q = -1; break; }
                const unsigned m = __ballot_sync(0xffffffffu, slow);
                if (m) hi_slow = q - 1 - (h * 32 + (__ffs(m) - 1));
            }
            if (q < 0 || hi_slow < 0) break;
            q = hi_slow;
        }
        long long cnt = 0;
        if (q < 0) {
            if (lane == 0) atomicOr(a.err, 4);
        } else {
            // (2) forward from q: mark the starts in [b0, b1)
            long long cur = q;
            while (cur < b1) {
                if (cur + 32 + NN_CMAX > lo + NN_WB) {   // slide the window (long CTA ranges)
                    __syncwarp();
                    lo = cur;
                    for (int i = lane; i < NN_WB; i += 32) {
                        const long long j = lo + i;
                        s_cv[i] = j < R ? __ldcg(g.cv + j) : (unsigned char)1;
                    }
                    __syncwarp();
                }
                const long long pos = cur + lane;
#ifdef BD_PHASE_TIMING
                ++dbg_steps;
#endif
                const int c = s_cv[pos - lo];
                const unsigned m = __ballot_sync(0xffffffffu, c != 1);
                const int f = m ? __ffs(m) - 1 : 32;
                const bool mine = lane < f && pos >= b0 && pos < b1;
                if (mine) g.st[pos] = 1;
                cnt += __popc(__ballot_sync(0xffffffffu, mine));
                if (f == 32) { cur += 32; continue; }
                const long long p = cur + f;
                const int cp = __shfl_sync(0xffffffffu, c, f);
                if (cp == 0) {                      // a draw longer than NN_CMAX raw values
                    if (lane == 0) atomicOr(a.err, 4);
                    break;
                }
                if (p >= b0 && p < b1) {
                    if (lane == 0) g.st[p] = 1;
                    ++cnt;
                }
                cur = p + cp;
            }
        }
        if (lane == 0) s_cnt = cnt;
#ifdef BD_PHASE_TIMING
        if (lane == 0) {
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(dbg_t[2]));
            dbg_q = q;
        }
#endif
    }
    __syncthreads();                                   // the st bytes of this range are final
    NG_T();
    // ---- starts, counted per CTA in position order: CTA b owns positions [b PB, (b+1) PB)
    __shared__ long long wsum[NN_GT / 32];
    __shared__ long long s_off;
    // each thread a contiguous sub-range of the CTA's positions
    const long long PT = (PB + NN_GT - 1) / NN_GT;
    const long long t0 = min(b1, b0 + threadIdx.x * PT), t1 = min(b1, t0 + PT);
    long long mine = 0;
    for (long long j = t0; j < t1; ++j) mine += g.st[j];
    // CTA-wide inclusive scan of `mine` (warp shuffles, then the warp sums)
    long long incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const long long v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
    }
    if (lane == 31) wsum[w] = incl;
    __syncthreads();
    long long wpre = 0;
    for (int k = 0; k < w; ++k) wpre += wsum[k];
    if (threadIdx.x == NN_GT - 1) {
        g.cta_count[blockIdx.x] = wpre + incl;
        if (b0 < b1 && wpre + incl != s_cnt) atomicOr(a.err, 4);   // walk and count disagree
    }
    nn_grid_sync(g.bar, a.err);
    NG_T();
    if (threadIdx.x < 32) {                              // this CTA's offset: the counts before it
        long long sacc = 0;
        for (int k = threadIdx.x; k < (int)blockIdx.x; k += 32) sacc += g.cta_count[k];
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
        if (threadIdx.x == 0) s_off = sacc;
    }
    __syncthreads();
    long long idx = s_off + wpre + incl - mine;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == NN_GT - 1 && idx + mine < a.count) atomicOr(a.err, 1);
    if (tid == 0) a.positions[0] = 0;
    for (long long j = t0; j < t1; ++j) {
        if (!g.st[j]) continue;
        if (idx < a.count) {
            const int c = g.cv[j];
            if (c == 0) atomicOr(a.err, 2);
            a.z[idx] = g.xv[j];
            if ((idx + 1) % a.block_len == 0) a.positions[(idx + 1) / a.block_len] = j + c;
        }
        ++idx;
    }
#ifdef BD_PHASE_TIMING
    NG_T();
    if (threadIdx.x == 0 && b0 < b1)
        printf("NNW cta %d q-b0 %lld steps %d load %.2f walk %.2f\n", blockIdx.x, dbg_q - b0, dbg_steps,
               (dbg_t[0] - gt[1]) * 1e-3, (dbg_t[2] - dbg_t[1]) * 1e-3);
    if (tid == 0) {
        printf("NNG us:");
        for (int i = 1; i < ng; ++i) printf(" %.2f", (gt[i] - gt[i - 1]) * 1e-3);
        printf("\n");
    }
#endif
}

}  // namespace bd
