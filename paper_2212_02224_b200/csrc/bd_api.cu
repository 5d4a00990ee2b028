// C-ABI implementation (include/bilevel_b200.h): device context, constant and
// scene upload, pointer staging and the launch sequences of the hot path.
#include <cuda_runtime.h>

#include <algorithm>
#include <unordered_map>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>

#include "../../include/bilevel_b200.h"
#include "am_kernel.cuh"
#include "bd_common.cuh"
#include "cem_kernels.cuh"
#include "aux_kernels.cuh"
#include "cvae_kernel.cuh"
#include "cvae_tc.cuh"
#include "cvae_fused.cuh"
#include <cudaTypedefs.h>
#include "scene_kernels.cuh"
#include "sim_kernels.cuh"
#include "p2p_kernels.cuh"
#include "cem_persistent.cuh"
#include "numpy_normals.cuh"

using namespace bd;

namespace {

struct DevBuf {
    void* p = nullptr;
    size_t bytes = 0;
    DevBuf() = default;
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    ~DevBuf() { if (p) cudaFree(p); }
    cudaError_t ensure(size_t n) {
        if (n <= bytes) return cudaSuccess;
        if (p) cudaFree(p);
        p = nullptr;
        bytes = 0;
        cudaError_t e = cudaMalloc(&p, n);
        if (e == cudaSuccess) bytes = n;
        return e;
    }
    template <class T> T* as() const { return static_cast<T*>(p); }
};

struct PendingCopy {
    void* dst;
    const void* src;
    size_t bytes;             // bytes written to dst (contiguous)
    size_t src_stride = 0;    // 0: contiguous source; else elements of `elem` bytes every src_stride bytes
    size_t elem = 0;
};

}  // namespace

struct bd_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    // side stream of the device numpy stream: its kernel depends only on the host's generator
    // state, so it runs beside whatever the main stream still has in flight (e.g. the CVAE decode
    // of a config-3 warm start); nn_free orders it after the previous cycle's use of its buffers
    cudaStream_t side = nullptr;
    cudaEvent_t nn_ready = nullptr, nn_free = nullptr;
    bool nn_free_valid = false;
    std::string err;
    int64_t launches = 0;
    int64_t persistent_cycles = 0;   // bd_cem_cycle calls run as the persistent kernel
    int opt_lanes = 0, opt_spc = 0, opt_lat_off = 0, opt_persist_off = 0, opt_help_off = 0;
    // instrumentation
    bool timing = false;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_used, ev_free;
    double am_ms = 0.0, am_launches = 0.0, am_sample_iters = 0.0;
    // basis
    int m = 0;
    DevBuf wrow, W64, Wd64, Wdd64;
    // stage 1
    int m_seg = 0, with_goal = 0, neq1 = 0, dim = 0;
    DevBuf qmx, qmy, kkt1, kinv1;
    // projection
    int n_obs = -1, neq = 0;
    double rho = 1.0;
    DevBuf kblk, kb, aeq;
    // scenes
    int S = 0, scene_obs = 0, obs_pad = 0, n_curv = 0;
    int obs_sorted = 0;          // scene tiles in the sorted-window layout (dense scenes)
    DevBuf obs, lim, bscene, curvf, ox64, oy64, lim64, curv64;
    // workspace
    DevBuf w_xibar, w_b, w_mu, w_xi, w_res, w_cost, w_hist, w_itmax, w_iters, w_replay, w_conf, w_err, w_params, w_done,
        w_order;
    size_t itmax_clean = 0;       // leading bytes of w_itmax known to be zero (re-armed by the exit scan)
    DevBuf stage[8];
    int n_stage = 0;
    DevBuf out_pack;              // coalesced device->host outputs: gathered here, one D2H copy
    void* out_pin = nullptr;      // pinned host staging for out_pack
    size_t out_pin_bytes = 0;
    // pinned host staging of a call's host inputs: one CPU memcpy + an asynchronous DMA each
    // (a pageable cudaMemcpyAsync is a synchronous driver copy); reused once the event has passed
    void* in_pin = nullptr;
    size_t in_pin_bytes = 0, in_pin_off = 0;
    cudaEvent_t in_pin_ev = nullptr;
    bool in_pin_pending = false;
    // fused CVAE: tensor maps of the last (count, activation buffer, weights) configuration
    int fz_count = -1;
    const void* fz_key_a = nullptr;
    const void* fz_key_w = nullptr;
    FusedMaps fz_maps;
    unsigned fz_epoch = 0;
    int fz_ctr_mblocks = -1;
    std::vector<PendingCopy> pending;
    bool host_out = false;
    // CEM state
    DevBuf c_bar;               // grid-barrier words of the persistent CEM kernel
    DevBuf nn_tab, nn_z, nn_pos, nn_err;   // numpy normal stream (tables, draws, block positions, error)
    DevBuf nn_raw, nn_x, nn_cs, nn_cnt, nn_bar;   // its grid-wide working buffers
    bool nn_tables = false;
    bool nn_check = false;      // the call drew numpy normals: check nn_err when it completes
    int nn_err_host = 0;
    DevBuf c_mean, c_cov, c_L, c_done, c_best_idx, c_best_p, c_best_xi, c_best_s, c_stats, c_cons, c_elite, c_eaug;
    // control grid
    int n_ctrl = 0;
    double ctrl_wb = 0, ctrl_amax = 0, ctrl_steer = 0, ctrl_eps = 0;
    DevBuf ctrl_wd, ctrl_wdd, w_sing, w_accel, w_steer;
    // sharded batch over NVLink peer memory (bd_shard_p2p_set)
    P2PArgs p2p{};
    bool p2p_set = false, p2p_epilogue = false;
    long long p2p_row0 = 0;
    // closed-loop simulation (in/out staging of host world state)
    DevBuf sim_io[7];
    // CVAE
    std::vector<int> cvae_dims;
    std::vector<DevBuf*> cvae_w, cvae_b, cvae_w16;
    DevBuf cvae_h0, cvae_h1, cvae_obs, cvae_z, cvae_a0, cvae_a1;
    DevBuf cvae_ready;          // fused decoder's arrival counters (persist across launches)
    DevBuf cvae_warm;           // bd_cvae_warm_start's rows (valid until its next call)
    int cvae_tc = 1;            // option "cvae_tensor_cores": bf16 tcgen05 hidden layers (1) or fp32 SIMT (0)
    int cvae_fused = 1;         // option "cvae_fused": the whole decoder in one persistent launch (1) or per layer (0)
    bool err_sticky = false;    // option "sticky_errors": entry points accumulate into the error word
                                // instead of clearing it (multi-call loops read it once at the end)
    ~bd_ctx() {
        for (auto& e : ev_used) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
        for (auto& e : ev_free) { cudaEventDestroy(e.first); cudaEventDestroy(e.second); }
        for (auto* b : cvae_w) delete b;
        for (auto* b : cvae_b) delete b;
        for (auto* b : cvae_w16) delete b;
        if (out_pin) cudaFreeHost(out_pin);
        if (in_pin_ev) cudaEventSynchronize(in_pin_ev);
        if (in_pin) cudaFreeHost(in_pin);
        if (in_pin_ev) cudaEventDestroy(in_pin_ev);
    }
};

namespace {

// FP32 issue-rate probe: 8 independent FFMA chains per thread, register resident.
__global__ void __launch_bounds__(256) ffma_probe_kernel(float* out, int iters, float a, float b) {
    float v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = threadIdx.x * 1e-3f + k;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = fmaf(v[k], a, b);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k];
    if (s == 12345.f) out[0] = s;
}

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    float2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;"
        : "=l"(*reinterpret_cast<unsigned long long*>(&r))
        : "l"(*reinterpret_cast<unsigned long long*>(&a)), "l"(*reinterpret_cast<unsigned long long*>(&b)),
          "l"(*reinterpret_cast<unsigned long long*>(&c)));
    return r;
}

// Packed FP32x2 variant of the probe (FFMA2, sm_100a).
__global__ void __launch_bounds__(256) ffma2_probe_kernel(float* out, int iters, float a, float b) {
    float2 v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = make_float2(threadIdx.x * 1e-3f + k, k * 0.5f);
    const float2 aa = make_float2(a, a), bb = make_float2(b, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 8; ++k) v[k] = ffma2(v[k], aa, bb);
    }
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += v[k].x + v[k].y;
    if (s == 12345.f) out[0] = s;
}

int fail(bd_ctx* c, int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    if (c) c->err = buf;
    return code;
}

#define CU(call)                                                                                  \
    do {                                                                                          \
        cudaError_t e_ = (call);                                                                  \
        if (e_ != cudaSuccess) return fail(ctx, BD_ERR_CUDA, "%s: %s", #call, cudaGetErrorString(e_)); \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return false;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

// Inputs: device pointers are used in place, host pointers are copied to a staging buffer.
template <class T>
int stage_in(bd_ctx* ctx, const T* p, size_t count, const T** out) {
    if (!p || count == 0 || is_device_ptr(p)) { *out = p; return 0; }
    if (ctx->n_stage >= 8) return fail(ctx, BD_ERR_STATE, "too many staged inputs");
    DevBuf& b = ctx->stage[ctx->n_stage++];
    const size_t bytes = count * sizeof(T);
    CU(b.ensure(bytes));
    // the previous call's DMAs must have left the pinned buffer before it is overwritten
    if (ctx->in_pin_pending && ctx->in_pin_off == 0) {
        CU(cudaEventSynchronize(ctx->in_pin_ev));
        ctx->in_pin_pending = false;
    }
    const size_t need = ctx->in_pin_off + (bytes + 255) / 256 * 256;
    if (need > ctx->in_pin_bytes) {
        if (ctx->in_pin_off == 0) {        // grow between calls only (no DMA of this call in flight)
            if (ctx->in_pin) cudaFreeHost(ctx->in_pin);
            ctx->in_pin = nullptr;
            ctx->in_pin_bytes = 0;
            const size_t want = std::max(need, (size_t)1 << 20) * 2;
            CU(cudaHostAlloc(&ctx->in_pin, want, cudaHostAllocDefault));
            ctx->in_pin_bytes = want;
            if (!ctx->in_pin_ev) CU(cudaEventCreateWithFlags(&ctx->in_pin_ev, cudaEventDisableTiming));
        } else {                           // does not fit behind this call's other inputs: pageable copy
            CU(cudaMemcpyAsync(b.p, p, bytes, cudaMemcpyHostToDevice, ctx->stream));
            *out = b.as<T>();
            return 0;
        }
    }
    unsigned char* pin = static_cast<unsigned char*>(ctx->in_pin) + ctx->in_pin_off;
    std::memcpy(pin, p, bytes);
    CU(cudaMemcpyAsync(b.p, pin, bytes, cudaMemcpyHostToDevice, ctx->stream));
    CU(cudaEventRecord(ctx->in_pin_ev, ctx->stream));
    ctx->in_pin_off = need;
    ctx->in_pin_pending = true;
    *out = b.as<T>();
    return 0;
}

// Outputs: device pointers are written directly; host pointers get a workspace buffer + a D2H copy.
template <class T>
int stage_out(bd_ctx* ctx, T* user, size_t count, DevBuf& ws, T** out) {
    if (!user || count == 0) { *out = nullptr; return 0; }
    if (is_device_ptr(user)) { *out = user; return 0; }
    CU(ws.ensure(count * sizeof(T)));
    *out = ws.as<T>();
    ctx->pending.push_back({user, ws.p, count * sizeof(T)});
    ctx->host_out = true;
    return 0;
}

// Same, but the kernel always needs a device buffer (the output is consumed internally).
template <class T>
int stage_out_req(bd_ctx* ctx, T* user, size_t count, DevBuf& ws, T** out) {
    if (user && is_device_ptr(user)) { *out = user; return 0; }
    CU(ws.ensure(count * sizeof(T)));
    *out = ws.as<T>();
    if (user) {
        ctx->pending.push_back({user, ws.p, count * sizeof(T)});
        ctx->host_out = true;
    }
    return 0;
}

// In/out arrays: device pointers are used in place; host arrays are copied in and copied back.
template <class T>
int stage_inout(bd_ctx* ctx, T* user, size_t count, DevBuf& ws, T** out) {
    if (!user || count == 0 || is_device_ptr(user)) { *out = user; return 0; }
    CU(ws.ensure(count * sizeof(T)));
    CU(cudaMemcpyAsync(ws.p, user, count * sizeof(T), cudaMemcpyHostToDevice, ctx->stream));
    *out = ws.as<T>();
    ctx->pending.push_back({user, ws.p, count * sizeof(T)});
    ctx->host_out = true;
    return 0;
}

// Clear the per-scene error word at the start of a call, unless the caller asked for sticky errors.
cudaError_t clear_err(bd_ctx* ctx, size_t bytes) {
    if (ctx->err_sticky) return cudaSuccess;
    return cudaMemsetAsync(ctx->w_err.p, 0, bytes, ctx->stream);
}

void begin_call(bd_ctx* ctx) {
    ctx->n_stage = 0;
    ctx->nn_check = false;
    ctx->in_pin_off = 0;
    ctx->pending.clear();
    ctx->host_out = false;
    cudaSetDevice(ctx->device);
}

// Gather of up to GATHER_MAX (possibly strided) device segments into one contiguous pack, so a
// call's host outputs leave the device in a single D2H copy (one DMA instead of one per array).
constexpr int GATHER_MAX = 24;
struct GatherSeg { const unsigned char* src; size_t off, bytes, stride, elem; };
struct GatherArgs { GatherSeg seg[GATHER_MAX]; int n; unsigned char* pack; };
__global__ void gather_kernel(const GatherArgs g) {
    const GatherSeg sg = g.seg[blockIdx.y];
    unsigned char* dst = g.pack + sg.off;
    if (sg.stride == 0) {
        const size_t words = sg.bytes / 4;
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < words; i += (size_t)gridDim.x * blockDim.x)
            reinterpret_cast<unsigned*>(dst)[i] = reinterpret_cast<const unsigned*>(sg.src)[i];
    } else {
        for (size_t i = blockIdx.x * blockDim.x + threadIdx.x; i < sg.bytes; i += (size_t)gridDim.x * blockDim.x)
            dst[i] = sg.src[(i / sg.elem) * sg.stride + i % sg.elem];
    }
}

int flush_outputs(bd_ctx* ctx) {
    auto& pend = ctx->pending;
    if (pend.empty()) return 0;
    const bool single = pend.size() == 1 && pend[0].src_stride == 0;
    std::vector<size_t> off(pend.size());
    size_t total = 0;
    for (size_t i = 0; i < pend.size(); ++i) { off[i] = total; total += (pend[i].bytes + 15) / 16 * 16; }
    CU(ctx->out_pack.ensure(total));
    if (total > ctx->out_pin_bytes) {
        if (ctx->out_pin) cudaFreeHost(ctx->out_pin);
        ctx->out_pin = nullptr;
        ctx->out_pin_bytes = 0;
        const size_t want = std::max(total, (size_t)1 << 16) * 2;
        CU(cudaHostAlloc(&ctx->out_pin, want, cudaHostAllocDefault));
        ctx->out_pin_bytes = want;
    }
    // one contiguous output goes straight to the pinned buffer (no gather)
    const void* pack_src = single ? pend[0].src : ctx->out_pack.p;
    for (size_t b = 0; !single && b < pend.size(); b += GATHER_MAX) {
        GatherArgs g{};
        g.n = (int)std::min(pend.size() - b, (size_t)GATHER_MAX);
        g.pack = ctx->out_pack.as<unsigned char>();
        size_t biggest = 0;
        for (int i = 0; i < g.n; ++i) {
            const PendingCopy& pc = pend[b + i];
            g.seg[i] = {static_cast<const unsigned char*>(pc.src), off[b + i], pc.bytes, pc.src_stride, pc.elem};
            biggest = std::max(biggest, pc.bytes);
        }
        const unsigned gx = (unsigned)std::min<size_t>((biggest / 4 + 255) / 256 + 1, 1024);
        gather_kernel<<<dim3(gx, g.n), 256, 0, ctx->stream>>>(g);
        ctx->launches++;
    }
    CU(cudaMemcpyAsync(ctx->out_pin, pack_src, single ? pend[0].bytes : total, cudaMemcpyDeviceToHost, ctx->stream));
    CU(cudaStreamSynchronize(ctx->stream));
    for (size_t i = 0; i < pend.size(); ++i)
        std::memcpy(pend[i].dst, static_cast<unsigned char*>(ctx->out_pin) + off[i], pend[i].bytes);
    pend.clear();
    return 0;
}

int finish_call(bd_ctx* ctx, bool check_err, int n_err) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, BD_ERR_CUDA, "kernel launch: %s", cudaGetErrorString(e));
    int rc = flush_outputs(ctx);
    if (rc) return rc;
    const bool sync = ctx->host_out || check_err;
    if (!sync) return 0;
    CU(cudaStreamSynchronize(ctx->stream));
    if (ctx->nn_check) {
        ctx->nn_check = false;
        if (ctx->nn_err_host)
            return fail(ctx, BD_ERR_STATE, "numpy normal stream: a draw needed more raw values than evaluated");
    }
    if (check_err && n_err > 0) {
        std::vector<int> errs(n_err);
        CU(cudaMemcpy(errs.data(), ctx->w_err.p, n_err * sizeof(int), cudaMemcpyDeviceToHost));
        int bits = 0;
        for (int v : errs) bits |= v;
        if (bits & ERR_BAD_RHS) return fail(ctx, BD_ERR_VALUE, "right-hand sides must be finite");
        if (bits & ERR_KKT_RESID) return fail(ctx, BD_ERR_NUMERICAL, "KKT residual exceeds tolerance");
        if (bits & ERR_NONFINITE) return fail(ctx, BD_ERR_NUMERICAL, "projection iterate is not finite");
        if (bits & ERR_P2P_TIMEOUT) return fail(ctx, BD_ERR_CUDA, "peer exchange timed out (a rank never signalled)");
    }
    return 0;
}

// Opt in to more than the default 48 KB when dynamic + static shared memory exceed it.
// Per kernel and device: its static shared memory and the dynamic size it was opted in to (the
// driver calls are made once per kernel, device and size, not per launch).
template <class K>
void raise_smem(K kernel, size_t bytes) {
    struct Seen { size_t stat = 0, raised = 0; bool known = false; };
    thread_local std::unordered_map<uintptr_t, Seen> seen;    // keyed by (kernel, device)
    int dev = 0;
    cudaGetDevice(&dev);
    Seen& e = seen[reinterpret_cast<uintptr_t>(reinterpret_cast<const void*>(kernel)) * 64 + (uintptr_t)dev];
    if (!e.known) {
        cudaFuncAttributes fa{};
        e.stat = cudaFuncGetAttributes(&fa, kernel) == cudaSuccess ? fa.sharedSizeBytes : 0;
        e.known = true;
    }
    if (bytes + e.stat > 48 * 1024 && bytes > e.raised &&
        cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess)
        e.raised = bytes;
}

template <int P, bool CURV, int MT = 0, int NPT = 0, int TPB = 0, bool LAT = false, int HELP = 0>
int launch_am_t(bd_ctx* ctx, AmArgs a, int threads, bool replay_pass, int* occ = nullptr) {
    if (HELP) a.s_cta = threads / 32 - 1;             // the last warp is the remainder warp
    const AmSmem lay(a.m, a.n_obs, a.neq, a.n_curv, a.s_cta, threads, P, CURV, a.max_iters, HELP);
    if (lay.total > 227 * 1024) return fail(ctx, BD_ERR_VALUE, "AM kernel needs %zu B of shared memory", lay.total);
    raise_smem(am_kernel<P, CURV, MT, NPT, TPB, LAT, HELP>, lay.total);
    if (occ) {   // occupancy query only (lane-mapping choice)
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(occ, am_kernel<P, CURV, MT, NPT, TPB, LAT, HELP>, threads,
                                                          lay.total) !=
            cudaSuccess) {
            cudaGetLastError();
            *occ = 0;
        }
        return 0;
    }
    dim3 grid((a.B + a.s_cta - 1) / a.s_cta, ctx->S);
    if (!replay_pass) a.replay = nullptr;
    std::pair<cudaEvent_t, cudaEvent_t> ev{nullptr, nullptr};
    const bool timed = ctx->timing && !replay_pass;   // replay guards exit at once unless an early exit fired
    if (timed) {
        if (ctx->ev_free.empty()) {
            cudaEventCreate(&ev.first);
            cudaEventCreate(&ev.second);
        } else {
            ev = ctx->ev_free.back();
            ctx->ev_free.pop_back();
        }
        cudaEventRecord(ev.first, ctx->stream);
    }
    am_kernel<P, CURV, MT, NPT, TPB, LAT, HELP><<<grid, threads, lay.total, ctx->stream>>>(a);
    ctx->launches++;
    if (timed) {
        cudaEventRecord(ev.second, ctx->stream);
        ctx->ev_used.push_back(ev);
        ctx->am_launches += 1;
        ctx->am_sample_iters += (double)a.B * ctx->S * a.max_iters;
    }
    return 0;
}

// The one-warp latency instance runs with a remainder warp at 3-8 samples per SM unless the option
// turns it off (8 samples + the remainder warp put 3 warps on one SM sub-partition: <= 168
// registers, still faster: 0.200 against 0.217 ms per AM launch at B = 1100).
static int samples_per_sm(const bd_ctx* ctx, long long samples) {
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    return (int)((samples + sms - 1) / sms);
}
#ifndef BD_HELP_MIN
#define BD_HELP_MIN 3   // 2 per SM is faster too (B = 290: 0.133 vs 0.142 ms) but moves the B <= 296 cases
                         // the batching-independence tests pin onto another lane mapping
#endif
static bool lat_helped(const bd_ctx* ctx, long long samples) {
    const int per_sm = samples_per_sm(ctx, samples);
    return !ctx->opt_help_off && !ctx->opt_spc && per_sm >= BD_HELP_MIN && per_sm <= 8;
}

int dispatch_am(bd_ctx* ctx, AmArgs a, int P, int threads, bool replay_pass, int* occ) {
    a.s_cta = threads / P;
    const bool curv = a.n_curv > 0;
    const int dflt = P == 32 ? 64 : 128;
    // compile-time shapes of the BASELINE configs (m = 100; 10 or 50 obstacles) and of the
    // reference planner's defaults (PlannerEnvConfig: m = 50, 6 obstacles), default CTA size
    const bool fixed = !curv && a.m == 100 && threads == dflt;
    const bool fixed50 = !curv && a.m == 50 && a.n_obs == 6 && threads == dflt;
#define AM_CASE(PP)                                                                                          \
    case PP:                                                                                                 \
        if (fixed && a.n_obs == 10)                                                                          \
            return launch_am_t<PP, false, 100, 5, (PP == 32 ? 64 : 128)>(ctx, a, threads, replay_pass, occ);  \
        if (fixed50)                                                                                         \
            return launch_am_t<PP, false, 50, 3, (PP == 32 ? 64 : 128)>(ctx, a, threads, replay_pass, occ);   \
        if (fixed && a.n_obs == 50)                                                                          \
            return launch_am_t<PP, false, 100, 25, (PP == 32 ? 64 : 128)>(ctx, a, threads, replay_pass, occ); \
        return curv ? launch_am_t<PP, true>(ctx, a, threads, replay_pass, occ)                               \
                    : launch_am_t<PP, false>(ctx, a, threads, replay_pass, occ);
    // single-scene latency shape: one CTA of 5-8 two-warp samples per SM (see default_threads)
    if (P == 64 && !curv && a.m == 100 && a.n_obs == 10 && threads > 256) {
        switch (threads) {
            case 320: return launch_am_t<64, false, 100, 5, 320, true>(ctx, a, threads, replay_pass, occ);
            case 384: return launch_am_t<64, false, 100, 5, 384, true>(ctx, a, threads, replay_pass, occ);
            case 448: return launch_am_t<64, false, 100, 5, 448, true>(ctx, a, threads, replay_pass, occ);
            case 512: return launch_am_t<64, false, 100, 5, 512, true>(ctx, a, threads, replay_pass, occ);
            default: return fail(ctx, BD_ERR_VALUE, "unsupported CTA size %d", threads);
        }
    }
    // single-scene latency shape, one-warp samples: one CTA of 3-8 samples + the remainder warp per
    // SM (timesteps 96-99 of every sample, am_helper), <= 255 registers (<= 168 at 8 + 1 warps)
    if (P == 32 && !curv && a.m == 100 && a.n_obs == 10 && lat_helped(ctx, (long long)a.B * ctx->S)) {
        switch (threads) {
            case 128: return launch_am_t<32, false, 100, 5, 128, true, 4>(ctx, a, threads, replay_pass, occ);
            case 160: return launch_am_t<32, false, 100, 5, 160, true, 4>(ctx, a, threads, replay_pass, occ);
            case 192: return launch_am_t<32, false, 100, 5, 192, true, 4>(ctx, a, threads, replay_pass, occ);
            case 224: return launch_am_t<32, false, 100, 5, 224, true, 4>(ctx, a, threads, replay_pass, occ);
            case 256: return launch_am_t<32, false, 100, 5, 256, true, 4>(ctx, a, threads, replay_pass, occ);
            case 288: return launch_am_t<32, false, 100, 5, 288, true, 4>(ctx, a, threads, replay_pass, occ);
            default: return fail(ctx, BD_ERR_VALUE, "unsupported CTA size %d", threads);
        }
    }
    // the same without the remainder warp: one CTA of 5-8 samples per SM
    if (P == 32 && !curv && a.m == 100 && a.n_obs == 10 && threads > 128) {
        switch (threads) {
            case 160: return launch_am_t<32, false, 100, 5, 160, true>(ctx, a, threads, replay_pass, occ);
            case 192: return launch_am_t<32, false, 100, 5, 192, true>(ctx, a, threads, replay_pass, occ);
            case 224: return launch_am_t<32, false, 100, 5, 224, true>(ctx, a, threads, replay_pass, occ);
            case 256: return launch_am_t<32, false, 100, 5, 256, true>(ctx, a, threads, replay_pass, occ);
            default: return fail(ctx, BD_ERR_VALUE, "unsupported CTA size %d", threads);
        }
    }
    switch (P) {
        AM_CASE(4)
        AM_CASE(8)
        AM_CASE(16)
        AM_CASE(32)
        AM_CASE(64)
        default: return fail(ctx, BD_ERR_VALUE, "lanes_per_sample must be 4, 8, 16, 32 or 64");
    }
#undef AM_CASE
}

int default_threads(bd_ctx* ctx, int P, const AmArgs& a) {
    int threads = ctx->opt_spc ? ctx->opt_spc * P : (P == 32 ? 64 : 128);
    if (P == 64 && threads % 64) threads = 128;
    if ((P == 64 || P == 32) && !ctx->opt_spc && a.n_curv == 0 && a.m == 100 && a.n_obs == 10) {
        // two-warp mapping on the BASELINE shape: give every SM one CTA of ceil(samples / SMs)
        // samples when that is 5-8, instead of 3-4 two-sample CTAs whose count differs by one
        // between SMs (B = 1000: 0.257 -> 0.246 ms per AM launch)
        int sms = 148;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        const long long per_sm = ((long long)a.B * ctx->S + sms - 1) / sms;
        if (per_sm >= 5 && per_sm <= 8) threads = P * (int)per_sm;
        else if (P == 32 && per_sm >= BD_HELP_MIN && per_sm < 5 && lat_helped(ctx, (long long)a.B * ctx->S))
            threads = 32 * (int)per_sm;
        if (P == 32 && lat_helped(ctx, (long long)a.B * ctx->S)) threads += 32;   // + the remainder warp
    }
    return threads;
}

// Lane mapping from a wave model: for each mapping, rounds = ceil(warps / resident warp slots)
// (slots from the occupancy API for the exact kernel instance and its shared memory) times the
// per-round cost of one sample group -- its serial timestep sweep plus reduction overhead, in
// units of one timestep (calibrated on B200, profiles/r01).  Small single-scene batches pick
// the two-warp mapping, fleets P = 8, the 10 000 x 50-obstacle batch P = 16.
int pick_lanes(bd_ctx* ctx, const AmArgs& a) {
    if (ctx->opt_lanes) return ctx->opt_lanes;
    const double total = (double)a.B * ctx->S;
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    // BASELINE latency shape with 7-8 samples per SM: one-warp samples in the 255-register
    // instance (round-1 A/B on B200, ms per AM launch, one-warp vs two-warp: B = 1000 0.230 vs
    // 0.242, B = 1100 0.234 vs 0.246; at 5-6 per SM the two-warp mapping won, B = 700 0.222 vs
    // 0.196, until the remainder warp)
    if (!ctx->opt_lat_off && a.n_curv == 0 && a.m == 100 && a.n_obs == 10) {
        const long long per_sm = ((long long)total + sms - 1) / sms;
        if (per_sm >= 7 && per_sm <= 8) return 32;
        // with the remainder warp the one-warp instance also beats the two-warp one at 3-6 per SM
        // (ms per AM launch: B = 440 0.135 vs 0.168, B = 590 0.145 vs 0.167,
        // B = 740 0.167 vs 0.184, B = 888 0.174 vs 0.188; without it 0.202 / 0.208 at 5 / 6);
        // single-scene cycles only, so a fleet keeps the lane mapping its scenes get when planned
        // one at a time at these sizes (tests/test_gpu_fleet.py: results independent of batching)
        if (per_sm >= BD_HELP_MIN && ctx->S == 1 && lat_helped(ctx, (long long)total)) return 32;
    }
    const int cands[4] = {8, 16, 32, 64};
    const double overhead[4] = {0.5, 0.7, 0.9, 1.0};
    int best = 8;
    double best_cost = 1e300;
    for (int i = 0; i < 4; ++i) {
        const int P = cands[i];
        const int threads = default_threads(ctx, P, a);
        int occ = 0;
        if (dispatch_am(ctx, a, P, threads, false, &occ) != 0 || occ <= 0) continue;
        const double slots = (double)occ * sms * (threads / 32);
        const double warps = total * P / 32.0;
        const double rounds = std::ceil(warps / slots);
        const double cost = rounds * (std::ceil((double)a.m / P) + overhead[i]);
        if (cost < best_cost) { best_cost = cost; best = P; }
    }
    return best;
}

int launch_am(bd_ctx* ctx, AmArgs a, bool replay_pass) {
    const int P = pick_lanes(ctx, a);
    const int threads = default_threads(ctx, P, a);
    // > 256 threads only for the latency-shape instances (dispatch_am: P = 64, m = 100, 10 obstacles)
    const bool big_ok = (P == 64 || (P == 32 && threads == 288)) && a.n_curv == 0 && a.m == 100 && a.n_obs == 10;
    if (threads % 32 || threads > 512 || threads < 32 || (threads > 256 && !big_ok))
        return fail(ctx, BD_ERR_VALUE, "bad samples_per_cta (more than 256 threads only for the 10-obstacle "
                    "m=100 two-warp mapping)");
    return dispatch_am(ctx, a, P, threads, replay_pass, nullptr);
}

int require_solver(bd_ctx* ctx, bool need_stage1) {
    if (!ctx->m) return fail(ctx, BD_ERR_STATE, "basis not set");
    if (ctx->n_obs < 0) return fail(ctx, BD_ERR_STATE, "projection not set");
    if (!ctx->S) return fail(ctx, BD_ERR_STATE, "scenes not set");
    if (ctx->scene_obs != ctx->n_obs)
        return fail(ctx, BD_ERR_VALUE, "operator was built for %d obstacles, spec has %d", ctx->n_obs, ctx->scene_obs);
    if (need_stage1 && !ctx->dim) return fail(ctx, BD_ERR_STATE, "stage-1 QP not set");
    if (need_stage1 && ctx->neq1 != ctx->neq) return fail(ctx, BD_ERR_STATE, "stage-1 / projection neq mismatch");
    return 0;
}

// Projection core: xi_bar, b device pointers -> outputs in device buffers.
// The per-iteration batch-maximum slots; a reallocation loses the zeroed prefix.
int ensure_itmax(bd_ctx* ctx, size_t bytes) {
    if (ctx->w_itmax.bytes < bytes) {
        ctx->itmax_clean = 0;
        CU(ctx->w_itmax.ensure(bytes));
    }
    return 0;
}

int run_projection(bd_ctx* ctx, int B, const double* xi_bar, const double* b, int iters, double tol, double* xi,
                   double* res, double* cost, float* hist, int* iters_used, unsigned long long* conf,
                   bool external_exit = false, bool count_conflicts = true) {
    const int S = ctx->S;
    const size_t itmax_bytes = (size_t)S * iters * ITMAX_SLOTS * 4;
    if (int rc = ensure_itmax(ctx, itmax_bytes)) return rc;
    CU(ctx->w_replay.ensure((size_t)S * 4));
    if (ctx->w_done.bytes < (size_t)S * 4) {
        CU(ctx->w_done.ensure((size_t)S * 4));
        CU(cudaMemsetAsync(ctx->w_done.p, 0, (size_t)S * 4, ctx->stream));
    }
    // the per-iteration batch maxima must start at zero; the in-kernel exit scan re-zeroes what it
    // read, so back-to-back full passes skip the memset (sharded passes scan outside the kernel)
    if (external_exit || ctx->itmax_clean < itmax_bytes)
        CU(cudaMemsetAsync(ctx->w_itmax.p, 0, itmax_bytes, ctx->stream));
    ctx->itmax_clean = external_exit ? 0 : std::max(ctx->itmax_clean, itmax_bytes);
    if (count_conflicts) CU(cudaMemsetAsync(conf, 0, (size_t)S * 8, ctx->stream));
    AmArgs a{};
    a.m = ctx->m; a.neq = ctx->neq; a.n_obs = ctx->obs_pad; a.n_curv = ctx->n_curv; a.B = B; a.max_iters = iters;
    a.rho = ctx->rho;
    if (ctx->p2p_epilogue) {
        a.p2p_bufs = ctx->p2p.bufs; a.p2p_world = ctx->p2p.world; a.p2p_row0 = ctx->p2p_row0;
        a.p2p_res_off = ctx->p2p.res_off; a.p2p_cost_off = ctx->p2p.cost_off;
    }
    a.wrow = ctx->wrow.as<float>(); a.kblk = ctx->kblk.as<double>(); a.kb = ctx->kb.as<double>();
    a.aeq = ctx->aeq.as<double>(); a.obs = ctx->obs.as<float4>(); a.lim = ctx->lim.as<SceneLim>();
    a.sorted = ctx->obs_sorted;
    a.bscene = ctx->bscene.as<double>(); a.curv = ctx->curvf.as<float>();
    a.xi_bar = xi_bar; a.b = b; a.xi_out = xi; a.resid_out = res; a.cost_out = cost; a.hist_out = hist;
    a.itmax = ctx->w_itmax.as<unsigned>(); a.conflicts = conf; a.err = ctx->w_err.as<int>();
    a.replay = ctx->w_replay.as<int>();
    a.tol = tol; a.iters_used = iters_used; a.replay_out = ctx->w_replay.as<int>();
    a.done_ctr = ctx->w_done.as<unsigned>();
    if (external_exit) a.done_ctr = nullptr;   // sharded batch: the exit is decided across ranks
    int rc = launch_am(ctx, a, false);     // its last CTA per scene runs the exit scan
    if (rc) ctx->itmax_clean = 0;
    if (rc || external_exit) return rc;
    return launch_am(ctx, a, true);        // replay guard: exits at once unless an early exit fired
}

AmArgs projection_args(bd_ctx* ctx, int B, const double* xi_bar, int iters, double* xi, double* res,
                       double* cost) {
    AmArgs a{};
    a.m = ctx->m; a.neq = ctx->neq; a.n_obs = ctx->obs_pad; a.n_curv = ctx->n_curv; a.B = B; a.max_iters = iters;
    a.rho = ctx->rho;
    if (ctx->p2p_epilogue) {
        a.p2p_bufs = ctx->p2p.bufs; a.p2p_world = ctx->p2p.world; a.p2p_row0 = ctx->p2p_row0;
        a.p2p_res_off = ctx->p2p.res_off; a.p2p_cost_off = ctx->p2p.cost_off;
    }
    a.wrow = ctx->wrow.as<float>(); a.kblk = ctx->kblk.as<double>(); a.kb = ctx->kb.as<double>();
    a.aeq = ctx->aeq.as<double>(); a.obs = ctx->obs.as<float4>(); a.lim = ctx->lim.as<SceneLim>();
    a.sorted = ctx->obs_sorted;
    a.bscene = ctx->bscene.as<double>(); a.curv = ctx->curvf.as<float>();
    a.xi_bar = xi_bar; a.xi_out = xi; a.resid_out = res; a.cost_out = cost;
    a.itmax = ctx->w_itmax.as<unsigned>(); a.conflicts = ctx->w_conf.as<unsigned long long>();
    a.err = ctx->w_err.as<int>(); a.replay = ctx->w_replay.as<int>();
    return a;
}

int run_stage1(bd_ctx* ctx, int B, const double* params, double* xi_bar, double* mu, double* b_out) {
    S1Args s{};
    s.total = ctx->S * B; s.B = B; s.dim = ctx->dim; s.neq = ctx->neq1; s.m_seg = ctx->m_seg;
    s.with_goal = ctx->with_goal; s.nr = NX + ctx->neq1; s.nvar = NX;
    s.qmx = ctx->qmx.as<double>(); s.qmy = ctx->qmy.as<double>(); s.kkt = ctx->kkt1.as<double>();
    s.kinv = ctx->kinv1.as<double>(); s.params = params; s.bscene = ctx->bscene.as<double>();
    s.xi_bar = xi_bar; s.mu = mu; s.b_out = b_out; s.err = ctx->w_err.as<int>();
    const int warps = 8;
    const size_t smem = (size_t)(2 * s.nr * s1_ld(s.nr) + 2 * NC * s.m_seg + warps * S1_VEC) * 8;
    raise_smem(stage1_kernel, smem);
    stage1_kernel<<<(s.total + warps - 1) / warps, warps * 32, smem, ctx->stream>>>(s);
    ctx->launches++;
    return 0;
}

}  // namespace

// =====================================================================================
// NVTX range per public call (nsys / ncu --nvtx filtering); header-only NVTX v3.
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

extern "C" {

int bd_abi_version(void) { return BD_ABI_VERSION; }

int bd_create(int device, bd_ctx** out) {
    if (!out) return BD_ERR_VALUE;
    *out = nullptr;
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return BD_ERR_CUDA;
    }
    if (device < 0 || device >= n) return BD_ERR_VALUE;
    bd_ctx* ctx = new bd_ctx();
    ctx->device = device;
    cudaSetDevice(device);
    if (cudaStreamCreateWithFlags(&ctx->own, cudaStreamNonBlocking) != cudaSuccess) {
        delete ctx;
        return BD_ERR_CUDA;
    }
    ctx->stream = ctx->own;
    *out = ctx;
    return 0;
}

void bd_destroy(bd_ctx* ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    if (ctx->own) cudaStreamDestroy(ctx->own);
    if (ctx->side) cudaStreamDestroy(ctx->side);
    if (ctx->nn_ready) cudaEventDestroy(ctx->nn_ready);
    if (ctx->nn_free) cudaEventDestroy(ctx->nn_free);
    delete ctx;
}

const char* bd_last_error(const bd_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int bd_set_stream(bd_ctx* ctx, void* s) {
    if (!ctx) return BD_ERR_VALUE;
    ctx->stream = s ? static_cast<cudaStream_t>(s) : ctx->own;
    return 0;
}

int bd_synchronize(bd_ctx* ctx) {
    if (!ctx) return BD_ERR_VALUE;
    cudaSetDevice(ctx->device);
    CU(cudaStreamSynchronize(ctx->stream));
    return 0;
}

int bd_set_option(bd_ctx* ctx, const char* key, int value) {
    if (!ctx || !key) return BD_ERR_VALUE;
    if (!strcmp(key, "lanes_per_sample")) {
        if (value != 0 && value != 4 && value != 8 && value != 16 && value != 32 && value != 64)
            return fail(ctx, BD_ERR_VALUE, "lanes_per_sample must be 0, 4, 8, 16, 32 or 64");
        ctx->opt_lanes = value;
        return 0;
    }
    if (!strcmp(key, "cvae_tensor_cores")) {
        ctx->cvae_tc = value != 0;
        return 0;
    }
    if (!strcmp(key, "cvae_fused")) {
        ctx->cvae_fused = value != 0;
        return 0;
    }
    if (!strcmp(key, "timing")) {
        ctx->timing = value != 0;
        return 0;
    }
    if (!strcmp(key, "sticky_errors")) {      // set (1) or leave (0) sticky mode; both reset the word
        cudaSetDevice(ctx->device);
        if (ctx->w_err.p) CU(cudaMemsetAsync(ctx->w_err.p, 0, ctx->w_err.bytes, ctx->stream));
        ctx->err_sticky = value != 0;
        return 0;
    }
    if (!strcmp(key, "persistent_cycle")) {   // 0: single-scene CEM cycles as the per-iteration launch chain
        ctx->opt_persist_off = value == 0;
        return 0;
    }
    if (!strcmp(key, "latency_instance")) {   // 0: never pick the one-warp latency instance automatically
        ctx->opt_lat_off = value == 0;
        return 0;
    }
    if (!strcmp(key, "remainder_warp")) {     // 0: one-warp latency CTAs without the remainder warp
        ctx->opt_help_off = value == 0;
        return 0;
    }
    if (!strcmp(key, "samples_per_cta")) {
        ctx->opt_spc = value < 0 ? 0 : value;
        return 0;
    }
    return fail(ctx, BD_ERR_VALUE, "unknown option %s", key);
}

int64_t bd_launch_count(const bd_ctx* ctx) { return ctx ? ctx->launches : -1; }

int bd_get_stat(bd_ctx* ctx, const char* key, double* value) {
    if (!ctx || !key || !value) return BD_ERR_VALUE;
    cudaSetDevice(ctx->device);
    CU(cudaStreamSynchronize(ctx->stream));
    for (auto& e : ctx->ev_used) {
        float ms = 0.f;
        CU(cudaEventElapsedTime(&ms, e.first, e.second));
        ctx->am_ms += ms;
        ctx->ev_free.push_back(e);
    }
    ctx->ev_used.clear();
    if (!strcmp(key, "am_ms")) *value = ctx->am_ms;
    else if (!strcmp(key, "am_launches")) *value = ctx->am_launches;
    else if (!strcmp(key, "persistent_cycles")) *value = (double)ctx->persistent_cycles;
    else if (!strcmp(key, "am_sample_iters")) *value = ctx->am_sample_iters;
    else if (!strcmp(key, "reset")) { ctx->am_ms = ctx->am_launches = ctx->am_sample_iters = 0.0; *value = 0.0; }
    else return fail(ctx, BD_ERR_VALUE, "unknown stat %s", key);
    return 0;
}

int bd_probe(bd_ctx* ctx, const char* what, double* value) {
    if (!ctx || !what || !value) return BD_ERR_VALUE;
    const bool x2 = !strcmp(what, "fp32x2_tflops");
    if (strcmp(what, "fp32_tflops") && !x2) return fail(ctx, BD_ERR_VALUE, "unknown probe %s", what);
    cudaSetDevice(ctx->device);
    int sms = 0;
    CU(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device));
    DevBuf out;
    CU(out.ensure(64));
    const int blocks = sms * 8, threads = 256, iters = 1 << 16;
    cudaEvent_t e0, e1;
    CU(cudaEventCreate(&e0));
    CU(cudaEventCreate(&e1));
    auto kern = x2 ? ffma2_probe_kernel : ffma_probe_kernel;
    kern<<<blocks, threads, 0, ctx->stream>>>(out.as<float>(), iters / 16, 0.999f, 1e-3f);  // warm
    CU(cudaEventRecord(e0, ctx->stream));
    kern<<<blocks, threads, 0, ctx->stream>>>(out.as<float>(), iters, 0.999f, 1e-3f);
    CU(cudaEventRecord(e1, ctx->stream));
    CU(cudaEventSynchronize(e1));
    float ms = 0.f;
    CU(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    *value = (x2 ? 2.0 : 1.0) * 2.0 * 8.0 * (double)iters * blocks * threads / (ms * 1e-3) / 1e12;
    return 0;
}

int bd_error_bits(bd_ctx* ctx, int* bits) {
    if (!ctx || !bits) return BD_ERR_VALUE;
    cudaSetDevice(ctx->device);
    CU(cudaStreamSynchronize(ctx->stream));
    *bits = 0;
    if (!ctx->S || !ctx->w_err.p) return 0;
    std::vector<int> errs(ctx->S);
    CU(cudaMemcpy(errs.data(), ctx->w_err.p, ctx->S * sizeof(int), cudaMemcpyDeviceToHost));
    for (int v : errs) *bits |= v;
    return 0;
}

int bd_set_basis(bd_ctx* ctx, int m, int n, const double* W, const double* Wd, const double* Wdd) {
    if (!ctx) return BD_ERR_VALUE;
    if (n != NC) return fail(ctx, BD_ERR_VALUE, "this build supports order-10 bases (n=%d), got n=%d", NC, n);
    if (m < n || m > 4096 || !W || !Wd || !Wdd) return fail(ctx, BD_ERR_VALUE, "bad basis shape m=%d", m);
    begin_call(ctx);
    std::vector<float> rows((size_t)m * WROW, 0.f);
    for (int t = 0; t < m; ++t)
        for (int k = 0; k < NC; ++k) {
            rows[(size_t)t * WROW + k] = (float)W[t * n + k];
            rows[(size_t)t * WROW + NC + k] = (float)Wd[t * n + k];
            rows[(size_t)t * WROW + 2 * NC + k] = (float)Wdd[t * n + k];
        }
    CU(ctx->wrow.ensure(rows.size() * 4));
    CU(cudaMemcpy(ctx->wrow.p, rows.data(), rows.size() * 4, cudaMemcpyHostToDevice));
    const size_t bytes = (size_t)m * n * 8;
    CU(ctx->W64.ensure(bytes));
    CU(ctx->Wd64.ensure(bytes));
    CU(ctx->Wdd64.ensure(bytes));
    CU(cudaMemcpy(ctx->W64.p, W, bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->Wd64.p, Wd, bytes, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->Wdd64.p, Wdd, bytes, cudaMemcpyHostToDevice));
    ctx->m = m;
    return 0;
}

int bd_set_stage1(bd_ctx* ctx, int m_seg, int with_goal, int neq, const double* qmx, const double* qmy,
                  const double* kkt, const double* kinv) {
    if (!ctx) return BD_ERR_VALUE;
    const int dim = 2 * m_seg + (with_goal ? 2 : 0);
    if (m_seg < 1 || dim > MAX_DIM || neq < 1 || neq > MAX_NEQ || NX + neq > 32)
        return fail(ctx, BD_ERR_VALUE, "unsupported stage-1 layout m_seg=%d neq=%d", m_seg, neq);
    if (with_goal && neq < 9) return fail(ctx, BD_ERR_VALUE, "goal layout needs 9 equality rows");
    begin_call(ctx);
    const int nr = NX + neq;
    CU(ctx->qmx.ensure((size_t)NC * m_seg * 8));
    CU(ctx->qmy.ensure((size_t)NC * m_seg * 8));
    CU(ctx->kkt1.ensure((size_t)nr * nr * 8));
    CU(ctx->kinv1.ensure((size_t)nr * nr * 8));
    CU(cudaMemcpy(ctx->qmx.p, qmx, (size_t)NC * m_seg * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->qmy.p, qmy, (size_t)NC * m_seg * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->kkt1.p, kkt, (size_t)nr * nr * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->kinv1.p, kinv, (size_t)nr * nr * 8, cudaMemcpyHostToDevice));
    ctx->m_seg = m_seg;
    ctx->with_goal = with_goal ? 1 : 0;
    ctx->neq1 = neq;
    ctx->dim = dim;
    return 0;
}

int bd_set_projection(bd_ctx* ctx, int n_obs, double rho, int neq, const double* kinv, const double* a_eq) {
    if (!ctx) return BD_ERR_VALUE;
    if (n_obs < 0 || neq < 1 || neq > MAX_NEQ || !(rho > 0) || !kinv || !a_eq)
        return fail(ctx, BD_ERR_VALUE, "bad projection arguments");
    begin_call(ctx);
    const int nr = NX + neq;
    for (int i = 0; i < NC; ++i)
        for (int j = NC; j < NX; ++j)
            if (kinv[i * nr + j] != 0.0 || kinv[j * nr + i] != 0.0)
                return fail(ctx, BD_ERR_STRUCTURE, "augmented KKT inverse couples the x and y blocks");
    std::vector<double> kb((size_t)NX * KSTR, 0.0), kbx((size_t)NX * neq), ae((size_t)neq * NX);
    for (int ax = 0; ax < 2; ++ax)
        for (int i = 0; i < NC; ++i)
            for (int j = 0; j < NC; ++j) kb[(2 * i + ax) * KSTR + j] = kinv[(ax * NC + i) * nr + ax * NC + j];
    for (int i = 0; i < NX; ++i)
        for (int e = 0; e < neq; ++e) kbx[i * neq + e] = kinv[i * nr + NX + e];
    memcpy(ae.data(), a_eq, ae.size() * 8);
    CU(ctx->kblk.ensure(kb.size() * 8));
    CU(ctx->kb.ensure(kbx.size() * 8));
    CU(ctx->aeq.ensure(ae.size() * 8));
    CU(cudaMemcpy(ctx->kblk.p, kb.data(), kb.size() * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->kb.p, kbx.data(), kbx.size() * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->aeq.p, ae.data(), ae.size() * 8, cudaMemcpyHostToDevice));
    ctx->n_obs = n_obs;
    ctx->rho = rho;
    ctx->neq = neq;
    return 0;
}

// Per-scene road curvature tables (np.interp abscissae + curvatures, pkg/constraints.py:67-72),
// fp32 for the AM kernel's clip window and fp64 for the residual evaluator; n_curv = 0 disables.
// Dense scenes get the sorted-window tile layout (am_kernel.cuh: sort_tile_kernel).
static int finish_tile(bd_ctx* ctx, int S, int m, int nop) {
    ctx->obs_sorted = 0;
    if (nop >= 2 * SORT_MIN_PAIRS && nop <= 256) {
        const int rows = S * m;
        sort_tile_kernel<<<(rows + 127) / 128, 128, 0, ctx->stream>>>(ctx->obs.as<float4>(), rows, nop / 2);
        ctx->launches++;
        ctx->obs_sorted = 1;
        CU(cudaGetLastError());
    }
    return 0;
}

// Stable residual order of every scene (rank_count_kernel / its shared-memory form).
static void launch_rank_count(bd_ctx* ctx, const double* resid, const int* err, int S, int B, int* order) {
    if (B <= RANK_SMEM_MAX) {
        const size_t smem = (size_t)B * 8;
        raise_smem(rank_count_smem_kernel, smem);
        rank_count_smem_kernel<<<dim3((unsigned)((B + 31) / 32), (unsigned)S), 256, smem, ctx->stream>>>(resid, err, B,
                                                                                                      order);
    } else {
        const size_t tot = (size_t)S * B;
        rank_count_kernel<<<(unsigned)((tot + 7) / 8), 256, 0, ctx->stream>>>(resid, err, S, B, order);
    }
    ctx->launches++;
}

static int upload_curvature(bd_ctx* ctx, int S, int n_curv, const double* cx, const double* ck) {
    if (n_curv > 0) {
        std::vector<float> cf((size_t)S * 2 * n_curv);
        std::vector<double> cd((size_t)S * 2 * n_curv);
        for (int s = 0; s < S; ++s)
            for (int i = 0; i < n_curv; ++i) {
                if (i > 0 && !(cx[s * n_curv + i] > cx[s * n_curv + i - 1]))
                    return fail(ctx, BD_ERR_VALUE, "curvature abscissae must increase");
                cd[(size_t)s * 2 * n_curv + i] = cx[s * n_curv + i];
                cd[(size_t)s * 2 * n_curv + n_curv + i] = ck[s * n_curv + i];
                cf[(size_t)s * 2 * n_curv + i] = (float)cx[s * n_curv + i];
                cf[(size_t)s * 2 * n_curv + n_curv + i] = (float)ck[s * n_curv + i];
            }
        CU(ctx->curvf.ensure(cf.size() * 4));
        CU(ctx->curv64.ensure(cd.size() * 8));
        CU(cudaMemcpy(ctx->curvf.p, cf.data(), cf.size() * 4, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->curv64.p, cd.data(), cd.size() * 8, cudaMemcpyHostToDevice));
    }
    ctx->n_curv = n_curv;
    return 0;
}

int bd_set_scenes(bd_ctx* ctx, int S, int n_obs, int m, const double* ox, const double* oy, const bd_limits* L,
                  const double* b0, int n_curv, const double* cx, const double* ck) {
    if (!ctx) return BD_ERR_VALUE;
    if (S < 1 || n_obs < 0 || !L || !b0 || n_curv < 0 || n_curv > 1024)
        return fail(ctx, BD_ERR_VALUE, "bad scene arguments");
    if (ctx->m && m != ctx->m) return fail(ctx, BD_ERR_VALUE, "constraint spec and basis disagree on the time grid");
    if (n_curv > 0 && (!cx || !ck)) return fail(ctx, BD_ERR_VALUE, "curvature table missing");
    if (n_obs > 0 && (!ox || !oy)) return fail(ctx, BD_ERR_VALUE, "obstacles missing");
    begin_call(ctx);
    int rc;
    const int neq = ctx->neq ? ctx->neq : 6;
    const size_t no = (size_t)S * n_obs * m;
    const int nop = (n_obs + 1) / 2 * 2;                         // even: two obstacles per LDS.128
    std::vector<float> obs((size_t)S * nop * m * 2 + 4, -1e18f);   // [s][t][pair] (-x0,-x1,-y0,-y1)
    std::vector<SceneLim> lim(S);
    std::vector<double> bs((size_t)S * neq, 0.0), l64((size_t)S * 9);
    for (int s = 0; s < S; ++s) {
        const bd_limits& l = L[s];
        if (!(l.v_min < l.v_max) || !(l.ellipse_a > 0) || !(l.ellipse_b > 0) || !(l.a_max > 0) ||
            !(l.kappa_max > 0) || !(l.c_max > 0) || !(l.y_lb < l.y_ub))
            return fail(ctx, BD_ERR_VALUE, "invalid constraint limits for scene %d", s);
        SceneLim& q = lim[s];
        q.a = (float)l.ellipse_a; q.b = (float)l.ellipse_b;
        q.inv_a = (float)(1.0 / l.ellipse_a); q.inv_b = (float)(1.0 / l.ellipse_b);
        q.v_min = (float)l.v_min; q.v_max = (float)l.v_max; q.a_max = (float)l.a_max;
        q.k_max = (float)l.kappa_max; q.inv_k_max = (float)(1.0 / l.kappa_max); q.c_max = (float)l.c_max;
        q.y_lb = (float)l.y_lb; q.y_ub = (float)l.y_ub;
        const double v9[9] = {l.ellipse_a, l.ellipse_b, l.v_min, l.v_max, l.a_max, l.kappa_max, l.c_max, l.y_lb, l.y_ub};
        memcpy(&l64[(size_t)s * 9], v9, sizeof v9);
        for (int e = 0; e < 6 && e < neq; ++e) bs[(size_t)s * neq + e] = b0[s * 6 + e];
        for (int o = 0; o < n_obs; ++o)
            for (int t = 0; t < m; ++t) {
                const size_t g = ((size_t)s * n_obs + o) * m + t;
                const size_t base = (((size_t)s * m + t) * (nop / 2) + o / 2) * 4 + (o & 1);
                obs[base] = (float)(-ox[g] / l.ellipse_a);
                obs[base + 2] = (float)(-oy[g] / l.ellipse_b);
            }
    }
    CU(ctx->obs.ensure(obs.size() * sizeof(float)));
    CU(ctx->lim.ensure(lim.size() * sizeof(SceneLim)));
    CU(ctx->bscene.ensure(bs.size() * 8));
    CU(ctx->lim64.ensure(l64.size() * 8));
    CU(cudaMemcpy(ctx->obs.p, obs.data(), obs.size() * sizeof(float), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->lim.p, lim.data(), lim.size() * sizeof(SceneLim), cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->bscene.p, bs.data(), bs.size() * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->lim64.p, l64.data(), l64.size() * 8, cudaMemcpyHostToDevice));
    CU(ctx->ox64.ensure(no ? no * 8 : 8));
    CU(ctx->oy64.ensure(no ? no * 8 : 8));
    if (no) {
        CU(cudaMemcpy(ctx->ox64.p, ox, no * 8, cudaMemcpyHostToDevice));
        CU(cudaMemcpy(ctx->oy64.p, oy, no * 8, cudaMemcpyHostToDevice));
    }
    if ((rc = upload_curvature(ctx, S, n_curv, cx, ck))) return rc;
    CU(ctx->w_err.ensure((size_t)S * 4));
    CU(cudaMemset(ctx->w_err.p, 0, (size_t)S * 4));
    if ((rc = finish_tile(ctx, S, m, nop))) return rc;
    ctx->S = S;
    ctx->scene_obs = n_obs;
    ctx->obs_pad = nop;
    return 0;
}

int bd_set_curvature(bd_ctx* ctx, int S, int n_curv, const double* cx, const double* ck) {
    if (!ctx) return BD_ERR_VALUE;
    if (S != ctx->S || n_curv < 0 || n_curv > 1024 || (n_curv > 0 && (!cx || !ck)))
        return fail(ctx, BD_ERR_VALUE, "curvature tables must cover the context's %d scenes", ctx->S);
    begin_call(ctx);
    return upload_curvature(ctx, S, n_curv, cx, ck);
}

int bd_stage1(bd_ctx* ctx, int S, int B, const double* params, double* xi_bar, double* mu, double* b_out) {
    NvtxRange nvtx_("bd_stage1");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, true);
    if (rc) return rc;
    if (S != ctx->S || B < 1 || !params) return fail(ctx, BD_ERR_VALUE, "bad batch (S=%d, B=%d)", S, B);
    begin_call(ctx);
    const size_t tot = (size_t)S * B;
    const double* dp;
    double *dx, *dm, *db;
    if ((rc = stage_in(ctx, params, tot * ctx->dim, &dp))) return rc;
    if ((rc = stage_out(ctx, xi_bar, tot * NX, ctx->w_xibar, &dx))) return rc;
    if ((rc = stage_out(ctx, mu, tot * ctx->neq1, ctx->w_mu, &dm))) return rc;
    if ((rc = stage_out(ctx, b_out, tot * ctx->neq1, ctx->w_b, &db))) return rc;
    CU(clear_err(ctx, (size_t)S * 4));
    if ((rc = run_stage1(ctx, B, dp, dx, dm, db))) return rc;
    return finish_call(ctx, ctx->host_out, S);
}

int bd_project(bd_ctx* ctx, int S, int B, const double* xi_bar, const double* b, int iters, double tol, double* xi,
               double* res, double* cost, float* hist, int* iters_used, int64_t* conflicts) {
    NvtxRange nvtx_("bd_project");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, false);
    if (rc) return rc;
    if (S != ctx->S || B < 1 || !xi_bar || !xi || !res || iters < 1 || !(tol > 0))
        return fail(ctx, BD_ERR_VALUE, "bad projection call (S=%d, B=%d, iters=%d)", S, B, iters);
    begin_call(ctx);
    const size_t tot = (size_t)S * B;
    const double *dxb, *dbb;
    double *dxi, *dres, *dcost;
    float* dh;
    int* dit;
    unsigned long long* dconf;
    if ((rc = stage_in(ctx, xi_bar, tot * NX, &dxb))) return rc;
    if ((rc = stage_in(ctx, b, b ? tot * ctx->neq : 0, &dbb))) return rc;
    if ((rc = stage_out(ctx, xi, tot * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, tot, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out(ctx, cost, tot, ctx->w_cost, &dcost))) return rc;
    if ((rc = stage_out(ctx, hist, (size_t)S * iters * B, ctx->w_hist, &dh))) return rc;
    if ((rc = stage_out_req(ctx, iters_used, (size_t)S, ctx->w_iters, &dit))) return rc;
    if ((rc = stage_out_req(ctx, reinterpret_cast<unsigned long long*>(conflicts), (size_t)S, ctx->w_conf, &dconf)))
        return rc;
    CU(clear_err(ctx, (size_t)S * 4));
    if ((rc = run_projection(ctx, B, dxb, dbb, iters, tol, dxi, dres, dcost, dh, dit, dconf))) return rc;
    return finish_call(ctx, ctx->host_out, S);
}

int bd_solve_lower(bd_ctx* ctx, int S, int B, const double* params, int iters, double tol, double* xi_bar,
                   double* mu, double* xi, double* res, double* cost, float* hist, int* iters_used,
                   int64_t* conflicts) {
    NvtxRange nvtx_("bd_solve_lower");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, true);
    if (rc) return rc;
    if (S != ctx->S || B < 1 || !params || !xi || !res || iters < 1 || !(tol > 0))
        return fail(ctx, BD_ERR_VALUE, "bad solve call (S=%d, B=%d, iters=%d)", S, B, iters);
    begin_call(ctx);
    const size_t tot = (size_t)S * B;
    const double* dp;
    double *dxb, *dmu, *dxi, *dres, *dcost, *db = nullptr;
    float* dh;
    int* dit;
    unsigned long long* dconf;
    if ((rc = stage_in(ctx, params, tot * ctx->dim, &dp))) return rc;
    if ((rc = stage_out_req(ctx, xi_bar, tot * NX, ctx->w_xibar, &dxb))) return rc;
    if ((rc = stage_out(ctx, mu, tot * ctx->neq, ctx->w_mu, &dmu))) return rc;
    if ((rc = stage_out(ctx, xi, tot * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, tot, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out(ctx, cost, tot, ctx->w_cost, &dcost))) return rc;
    if ((rc = stage_out(ctx, hist, (size_t)S * iters * B, ctx->w_hist, &dh))) return rc;
    if ((rc = stage_out_req(ctx, iters_used, (size_t)S, ctx->w_iters, &dit))) return rc;
    if ((rc = stage_out_req(ctx, reinterpret_cast<unsigned long long*>(conflicts), (size_t)S, ctx->w_conf, &dconf)))
        return rc;
    if (ctx->with_goal) {
        CU(ctx->w_b.ensure(tot * ctx->neq * 8));
        db = ctx->w_b.as<double>();
    }
    CU(clear_err(ctx, (size_t)S * 4));
    if ((rc = run_stage1(ctx, B, dp, dxb, dmu, db))) return rc;
    if ((rc = run_projection(ctx, B, dxb, db, iters, tol, dxi, dres, dcost, dh, dit, dconf))) return rc;
    return finish_call(ctx, ctx->host_out, S);
}

int bd_eval(bd_ctx* ctx, int count, const double* xi, double* x, double* y, double* xd, double* yd, double* xdd,
            double* ydd) {
    NvtxRange nvtx_("bd_eval");
    if (!ctx) return BD_ERR_VALUE;
    if (!ctx->m) return fail(ctx, BD_ERR_STATE, "basis not set");
    if (count < 1 || !xi) return fail(ctx, BD_ERR_VALUE, "bad eval call");
    begin_call(ctx);
    int rc;
    const size_t n = (size_t)count * ctx->m;
    const double* dxi;
    double* o[6];
    double* user[6] = {x, y, xd, yd, xdd, ydd};
    if ((rc = stage_in(ctx, xi, (size_t)count * NX, &dxi))) return rc;
    DevBuf* ws[6] = {&ctx->stage[2], &ctx->stage[3], &ctx->stage[4], &ctx->stage[5], &ctx->stage[6], &ctx->stage[7]};
    for (int q = 0; q < 6; ++q)
        if ((rc = stage_out(ctx, user[q], n, *ws[q], &o[q]))) return rc;
    eval_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(count, ctx->m, ctx->W64.as<double>(),
                                                                       ctx->Wd64.as<double>(), ctx->Wdd64.as<double>(),
                                                                       dxi, o[0], o[1], o[2], o[3], o[4], o[5]);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

int bd_residuals(bd_ctx* ctx, int S, int B, const double* xi, double* out) {
    NvtxRange nvtx_("bd_residuals");
    if (!ctx) return BD_ERR_VALUE;
    if (!ctx->m || !ctx->S) return fail(ctx, BD_ERR_STATE, "basis / scenes not set");
    if (S != ctx->S || B < 1 || !xi || !out) return fail(ctx, BD_ERR_VALUE, "bad residual call");
    begin_call(ctx);
    int rc;
    const size_t tot = (size_t)S * B;
    const double* dxi;
    double* dout;
    if ((rc = stage_in(ctx, xi, tot * NX, &dxi))) return rc;
    if ((rc = stage_out(ctx, out, tot, ctx->w_res, &dout))) return rc;
    ResArgs r{};
    r.total = (int)tot; r.B = B; r.m = ctx->m; r.n_obs = ctx->scene_obs; r.n_curv = ctx->n_curv;
    r.W = ctx->W64.as<double>(); r.Wd = ctx->Wd64.as<double>(); r.Wdd = ctx->Wdd64.as<double>();
    r.ox = ctx->ox64.as<double>(); r.oy = ctx->oy64.as<double>(); r.lim = ctx->lim64.as<double>();
    r.curv = ctx->curv64.as<double>(); r.xi = dxi; r.out = dout;
    residual_kernel<<<(unsigned)((tot + 7) / 8), 256, 0, ctx->stream>>>(r);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

int bd_solve_lower_shard(bd_ctx* ctx, int B, const double* params, int iters, double* xi_bar, double* xi,
                         double* res, double* cost, float* iter_max) {
    NvtxRange nvtx_("bd_solve_lower_shard");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, true);
    if (rc) return rc;
    if (ctx->S != 1 || ctx->with_goal || B < 1 || !params || !xi_bar || !xi || !res || !iter_max || iters < 1)
        return fail(ctx, BD_ERR_VALUE, "bad shard call (one scene, non-goal layout)");
    begin_call(ctx);
    const double* dp;
    double *dxb, *dxi, *dres, *dcost;
    float* dmax;
    if ((rc = stage_in(ctx, params, (size_t)B * ctx->dim, &dp))) return rc;
    if ((rc = stage_out_req(ctx, xi_bar, (size_t)B * NX, ctx->w_xibar, &dxb))) return rc;
    if ((rc = stage_out(ctx, xi, (size_t)B * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, (size_t)B, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out(ctx, cost, (size_t)B, ctx->w_cost, &dcost))) return rc;
    if ((rc = stage_out(ctx, iter_max, (size_t)iters, ctx->stage[7], &dmax))) return rc;
    CU(ctx->w_iters.ensure(4));
    CU(ctx->w_conf.ensure(8));
    CU(clear_err(ctx, 4));
    if ((rc = run_stage1(ctx, B, dp, dxb, nullptr, nullptr))) return rc;
    if ((rc = run_projection(ctx, B, dxb, nullptr, iters, 1.0, dxi, dres, dcost, nullptr, ctx->w_iters.as<int>(),
                             ctx->w_conf.as<unsigned long long>(), true)))
        return rc;
    itmax_reduce_kernel<<<1, 128, 0, ctx->stream>>>(ctx->w_itmax.as<unsigned>(), iters, dmax);
    ctx->launches++;
    return finish_call(ctx, ctx->host_out, 1);
}

int bd_replay_shard(bd_ctx* ctx, int B, const double* xi_bar, int iters, double* xi, double* res, double* cost) {
    NvtxRange nvtx_("bd_replay_shard");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, false);
    if (rc) return rc;
    if (ctx->S != 1 || B < 1 || !xi_bar || !xi || !res || iters < 1) return fail(ctx, BD_ERR_VALUE, "bad replay");
    begin_call(ctx);
    const double* dxb;
    double *dxi, *dres, *dcost;
    if ((rc = stage_in(ctx, xi_bar, (size_t)B * NX, &dxb))) return rc;
    if ((rc = stage_out(ctx, xi, (size_t)B * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, (size_t)B, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out(ctx, cost, (size_t)B, ctx->w_cost, &dcost))) return rc;
    if ((rc = ensure_itmax(ctx, (size_t)iters * ITMAX_SLOTS * 4))) return rc;
    CU(ctx->w_replay.ensure(4));
    CU(ctx->w_conf.ensure(8));
    CU(clear_err(ctx, 4));
    CU(cudaMemcpyAsync(ctx->w_replay.p, &iters, 4, cudaMemcpyHostToDevice, ctx->stream));
    AmArgs a = projection_args(ctx, B, dxb, iters, dxi, dres, dcost);
    if ((rc = launch_am(ctx, a, true))) return rc;
    return finish_call(ctx, true, 1);
}

int bd_replay_shard_dev(bd_ctx* ctx, int B, const double* xi_bar, int max_iters, const int* iterations, double* xi,
                        double* res, double* cost) {
    NvtxRange nvtx_("bd_replay_shard_dev");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, false);
    if (rc) return rc;
    if (ctx->S != 1 || B < 1 || !xi_bar || !xi || !res || !iterations || max_iters < 1)
        return fail(ctx, BD_ERR_VALUE, "bad replay");
    begin_call(ctx);
    const double* dxb;
    const int* dit;
    double *dxi, *dres, *dcost;
    if ((rc = stage_in(ctx, xi_bar, (size_t)B * NX, &dxb))) return rc;
    if ((rc = stage_in(ctx, iterations, 1, &dit))) return rc;
    if ((rc = stage_out(ctx, xi, (size_t)B * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, (size_t)B, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out(ctx, cost, (size_t)B, ctx->w_cost, &dcost))) return rc;
    if ((rc = ensure_itmax(ctx, (size_t)max_iters * ITMAX_SLOTS * 4))) return rc;
    CU(ctx->w_replay.ensure(4));
    CU(ctx->w_conf.ensure(8));
    // the guarded kernel reads the count on the device: <= 0 returns at once, so no host decision
    CU(cudaMemcpyAsync(ctx->w_replay.p, dit, 4, cudaMemcpyDeviceToDevice, ctx->stream));
    AmArgs a = projection_args(ctx, B, dxb, max_iters, dxi, dres, dcost);
    if ((rc = launch_am(ctx, a, true))) return rc;
    return finish_call(ctx, false, 0);
}

int bd_shard_p2p_set(bd_ctx* ctx, int world, int rank, void* const* bufs, unsigned* const* sigs, size_t res_off,
                     size_t cost_off, size_t itmax_off, size_t xi_off, int iters_cap) {
    if (!ctx) return BD_ERR_VALUE;
    if (world < 1 || rank < 0 || rank >= world || !bufs || !sigs || iters_cap < 1)
        return fail(ctx, BD_ERR_VALUE, "bad peer exchange description");
    if (!is_device_ptr(bufs) || !is_device_ptr(sigs))
        return fail(ctx, BD_ERR_VALUE, "peer pointer tables must be device arrays");
    ctx->p2p = P2PArgs{world, rank, iters_cap, bufs, sigs, res_off, cost_off, itmax_off, xi_off, nullptr};
    ctx->p2p_set = true;
    return 0;
}

int bd_solve_lower_shard_p2p(bd_ctx* ctx, int B, const double* params, int iters, double* xi_bar, double* xi,
                             double* res, double* cost, long long row0, unsigned epoch, double tol, int* used) {
    NvtxRange nvtx_("bd_solve_lower_shard_p2p");
    if (!ctx) return BD_ERR_VALUE;
    int rc = require_solver(ctx, true);
    if (rc) return rc;
    if (!ctx->p2p_set) return fail(ctx, BD_ERR_STATE, "peer exchange not set (bd_shard_p2p_set)");
    if (ctx->S != 1 || ctx->with_goal || B < 1 || !params || !xi_bar || !xi || !res || iters < 1 ||
        iters > ctx->p2p.iters_cap || row0 < 0 || epoch == 0)
        return fail(ctx, BD_ERR_VALUE, "bad peer-exchange shard call");
    begin_call(ctx);
    const double* dp;
    double *dxb, *dxi, *dres, *dcost;
    int* dused;
    if ((rc = stage_in(ctx, params, (size_t)B * ctx->dim, &dp))) return rc;
    if ((rc = stage_out_req(ctx, xi_bar, (size_t)B * NX, ctx->w_xibar, &dxb))) return rc;
    if ((rc = stage_out(ctx, xi, (size_t)B * NX, ctx->w_xi, &dxi))) return rc;
    if ((rc = stage_out(ctx, res, (size_t)B, ctx->w_res, &dres))) return rc;
    if ((rc = stage_out_req(ctx, cost, (size_t)B, ctx->w_cost, &dcost))) return rc;
    if ((rc = stage_out_req(ctx, used, 1, ctx->sim_io[6], &dused))) return rc;
    CU(ctx->w_iters.ensure(4));
    CU(ctx->w_conf.ensure(8));
    CU(ctx->stage[7].ensure((size_t)iters * 4));
    P2PArgs pa = ctx->p2p;
    pa.err = ctx->w_err.as<int>();
    CU(clear_err(ctx, 4));
    if ((rc = run_stage1(ctx, B, dp, dxb, nullptr, nullptr))) return rc;
    ctx->p2p_epilogue = true;                 // AM epilogues store (res, cost) into every rank's buffer
    ctx->p2p_row0 = row0;
    rc = run_projection(ctx, B, dxb, nullptr, iters, 1.0, dxi, dres, dcost, nullptr, ctx->w_iters.as<int>(),
                        ctx->w_conf.as<unsigned long long>(), true);
    if (!rc) {
        float* dmax = ctx->stage[7].as<float>();
        itmax_reduce_kernel<<<1, 128, 0, ctx->stream>>>(ctx->w_itmax.as<unsigned>(), iters, dmax);
        p2p_publish_kernel<<<1, 128, 0, ctx->stream>>>(pa, dmax, iters, epoch, 0);
        p2p_wait_kernel<<<1, 32, 0, ctx->stream>>>(pa, epoch, 0);
        p2p_exit_kernel<<<1, 128, 0, ctx->stream>>>(pa, iters, tol, ctx->w_replay.as<int>(), dused);
        ctx->launches += 4;
        AmArgs a = projection_args(ctx, B, dxb, iters, dxi, dres, dcost);   // replay guard (device count)
        rc = launch_am(ctx, a, true);
        p2p_publish_kernel<<<1, 32, 0, ctx->stream>>>(pa, nullptr, 0, epoch, 1);
        p2p_wait_kernel<<<1, 32, 0, ctx->stream>>>(pa, epoch, 1);
        ctx->launches += 2;
    }
    ctx->p2p_epilogue = false;
    if (rc) return rc;
    return finish_call(ctx, ctx->host_out, 1);
}

int bd_shard_p2p_best_row(bd_ctx* ctx, const int64_t* best_index, long long row0, int b_shard, const double* xi_shard,
                          unsigned epoch, double* xi_out) {
    NvtxRange nvtx_("bd_shard_p2p_best_row");
    if (!ctx) return BD_ERR_VALUE;
    if (!ctx->p2p_set) return fail(ctx, BD_ERR_STATE, "peer exchange not set (bd_shard_p2p_set)");
    if (!best_index || !xi_shard || !xi_out || b_shard < 1 || epoch == 0) return fail(ctx, BD_ERR_VALUE, "bad row share");
    begin_call(ctx);
    int rc;
    const int64_t* dbest;
    const double* dxs;
    double* dout;
    if ((rc = stage_in(ctx, best_index, 1, &dbest))) return rc;
    if ((rc = stage_in(ctx, xi_shard, (size_t)b_shard * NX, &dxs))) return rc;
    if ((rc = stage_out(ctx, xi_out, NX, ctx->w_sing, &dout))) return rc;
    P2PArgs pa = ctx->p2p;
    pa.err = ctx->w_err.as<int>();
    p2p_share_row_kernel<<<1, 32, 0, ctx->stream>>>(pa, reinterpret_cast<const long long*>(dbest), row0, b_shard, dxs,
                                                    epoch, 2);
    p2p_wait_kernel<<<1, 32, 0, ctx->stream>>>(pa, epoch, 2);
    p2p_sum_rows_kernel<<<1, 32, 0, ctx->stream>>>(pa, dout);
    ctx->launches += 3;
    return finish_call(ctx, false, 0);
}

int bd_sample_philox(bd_ctx* ctx, int dim, int count, const double* mean, const double* cov, uint64_t seed,
                     int scene, int iteration, int first_index, double* params) {
    NvtxRange nvtx_("bd_sample_philox");
    if (!ctx) return BD_ERR_VALUE;
    if (dim < 1 || dim > MAX_DIM || count < 1 || !mean || !cov || !params || first_index < 0)
        return fail(ctx, BD_ERR_VALUE, "bad sample call");
    begin_call(ctx);
    int rc;
    const double *dm, *dc;
    double* dp;
    if ((rc = stage_in(ctx, mean, (size_t)dim, &dm))) return rc;
    if ((rc = stage_in(ctx, cov, (size_t)dim * dim, &dc))) return rc;
    if ((rc = stage_out(ctx, params, (size_t)count * dim, ctx->w_params, &dp))) return rc;
    const int blocks = count / 256 + 1 < 148 ? count / 256 + 1 : 148;
    sample_philox_kernel<<<blocks, 256, 0, ctx->stream>>>(dim, count, dm, dc, seed, scene, iteration, first_index, dp);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

int bd_kkt_solve(bd_ctx* ctx, int nvar, int neq, const double* kkt, const double* kinv, int count,
                 const double* rhs, double* sol) {
    NvtxRange nvtx_("bd_kkt_solve");
    if (!ctx) return BD_ERR_VALUE;
    const int nr = nvar + neq;
    if (nvar < 1 || neq < 0 || nr > 32 || count < 1 || !kkt || !kinv || !rhs || !sol)
        return fail(ctx, BD_ERR_VALUE, "bd_kkt_solve supports nvar + neq <= 32");
    begin_call(ctx);
    int rc;
    const double *dk, *dki, *dr;
    double* ds;
    if ((rc = stage_in(ctx, kkt, (size_t)nr * nr, &dk))) return rc;
    if ((rc = stage_in(ctx, kinv, (size_t)nr * nr, &dki))) return rc;
    if ((rc = stage_in(ctx, rhs, (size_t)count * nr, &dr))) return rc;
    if ((rc = stage_out(ctx, sol, (size_t)count * nr, ctx->w_xibar, &ds))) return rc;
    CU(ctx->w_err.ensure(4 * (size_t)(ctx->S > 1 ? ctx->S : 1)));
    CU(clear_err(ctx, 4));
    S1Args s{};
    s.total = count; s.B = count; s.nr = nr; s.nvar = nvar; s.neq = neq;
    s.kkt = dk; s.kinv = dki; s.rhs_in = dr; s.sol_out = ds; s.err = ctx->w_err.as<int>();
    const size_t smem = (size_t)(2 * nr * s1_ld(nr) + 8 * S1_VEC) * 8;
    raise_smem(stage1_kernel, smem);
    stage1_kernel<<<(count + 7) / 8, 256, smem, ctx->stream>>>(s);
    ctx->launches++;
    return finish_call(ctx, true, 1);
}

int bd_sample(bd_ctx* ctx, int dim, int count, const double* mean, const double* cov, const double* z,
              double* params) {
    NvtxRange nvtx_("bd_sample");
    if (!ctx) return BD_ERR_VALUE;
    if (dim < 1 || dim > MAX_DIM || count < 1 || !mean || !cov || !z || !params)
        return fail(ctx, BD_ERR_VALUE, "bad sample call");
    begin_call(ctx);
    int rc;
    const double *dm, *dc, *dz;
    double* dp;
    if ((rc = stage_in(ctx, mean, (size_t)dim, &dm))) return rc;
    if ((rc = stage_in(ctx, cov, (size_t)dim * dim, &dc))) return rc;
    if ((rc = stage_in(ctx, z, (size_t)count * dim, &dz))) return rc;
    if ((rc = stage_out(ctx, params, (size_t)count * dim, ctx->w_params, &dp))) return rc;
    const int blocks = count / 256 + 1 < 64 ? count / 256 + 1 : 64;
    sample_one_kernel<<<blocks, 256, 0, ctx->stream>>>(dim, count, dm, dc, dz, dp);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

int bd_rank_refit(bd_ctx* ctx, int S, int B, int dim, const double* resid, const double* cost, const double* params,
                  int n_cons, int n_elite, double w_res, double eta, double gamma, double* mean, double* cov,
                  int64_t* cons_idx, int64_t* elite_idx, double* elite_aug, double* stats) {
    NvtxRange nvtx_("bd_rank_refit");
    if (!ctx) return BD_ERR_VALUE;
    if (S < 1 || B < 1 || !resid || !cost || !params || !mean || !cov || dim < 1 || dim > MAX_DIM)
        return fail(ctx, BD_ERR_VALUE, "bad rank_refit call");
    if (!(n_elite <= n_cons && n_cons <= B) || n_elite < 1 || n_cons > 1024)
        return fail(ctx, BD_ERR_VALUE, "need 1 <= elites <= constraint_elites <= min(batch, 1024)");
    if (B > (1 << 24)) return fail(ctx, BD_ERR_VALUE, "batch too large");
    begin_call(ctx);
    int rc;
    const size_t tot = (size_t)S * B;
    const double *dr, *dc, *dp;
    if ((rc = stage_in(ctx, resid, tot, &dr))) return rc;
    if ((rc = stage_in(ctx, cost, tot, &dc))) return rc;
    if ((rc = stage_in(ctx, params, tot * dim, &dp))) return rc;
    CU(ctx->c_mean.ensure((size_t)S * dim * 8));
    CU(ctx->c_cov.ensure((size_t)S * dim * dim * 8));
    CU(ctx->c_L.ensure((size_t)S * dim * dim * 8));
    CU(ctx->c_done.ensure((size_t)S * 4));
    CU(ctx->c_best_idx.ensure((size_t)S * 8));
    CU(ctx->c_best_p.ensure((size_t)S * dim * 8));
    CU(ctx->c_best_xi.ensure((size_t)S * NX * 8));
    CU(ctx->c_best_s.ensure((size_t)S * 3 * 8));
    CU(ctx->w_err.ensure((size_t)S * 4));
    CU(ctx->w_xi.ensure(tot * NX * 8));
    CU(cudaMemcpyAsync(ctx->c_mean.p, mean, (size_t)S * dim * 8, cudaMemcpyDefault, ctx->stream));
    CU(cudaMemcpyAsync(ctx->c_cov.p, cov, (size_t)S * dim * dim * 8, cudaMemcpyDefault, ctx->stream));
    CU(clear_err(ctx, (size_t)S * 4));
    CU(cudaMemsetAsync(ctx->c_done.p, 0, (size_t)S * 4, ctx->stream));
    int64_t *dci, *dei;
    double *dea, *dst;
    if ((rc = stage_out(ctx, cons_idx, (size_t)S * n_cons, ctx->c_cons, &dci))) return rc;
    if ((rc = stage_out(ctx, elite_idx, (size_t)S * n_elite, ctx->c_elite, &dei))) return rc;
    if ((rc = stage_out(ctx, elite_aug, (size_t)S * n_elite, ctx->c_eaug, &dea))) return rc;
    if ((rc = stage_out(ctx, stats, (size_t)S * 6, ctx->c_stats, &dst))) return rc;
    CemState s{};
    s.S = S; s.B = B; s.dim = dim; s.n_cons = n_cons; s.n_elite = n_elite; s.iters = 1;
    s.eta = eta; s.gamma = gamma; s.w_res = w_res;
    s.mean = ctx->c_mean.as<double>(); s.cov = ctx->c_cov.as<double>(); s.L = ctx->c_L.as<double>();
    s.err = ctx->w_err.as<int>(); s.done = ctx->c_done.as<int>();
    s.resid = dr; s.cost = dc; s.params = dp; s.xi = ctx->w_xi.as<double>();
    s.cons_idx = reinterpret_cast<long long*>(dci); s.elite_idx = reinterpret_cast<long long*>(dei);
    s.elite_aug = dea; s.stats = dst;
    s.best_index = ctx->c_best_idx.as<long long>(); s.best_params = ctx->c_best_p.as<double>();
    s.best_xi = ctx->c_best_xi.as<double>(); s.best_scal = ctx->c_best_s.as<double>();
    CU(ctx->w_order.ensure(tot * 4));
    launch_rank_count(ctx, dr, nullptr, S, B, ctx->w_order.as<int>());
    const size_t smem = rank_refit_smem(n_cons, n_elite, dim);
    raise_smem(rank_refit_kernel, smem);
    rank_refit_kernel<<<S, RANK_REFIT_THREADS, smem, ctx->stream>>>(s, 0, ctx->w_order.as<int>());
    ctx->launches++;
    CU(cudaMemcpyAsync(mean, ctx->c_mean.p, (size_t)S * dim * 8, cudaMemcpyDefault, ctx->stream));
    CU(cudaMemcpyAsync(cov, ctx->c_cov.p, (size_t)S * dim * dim * 8, cudaMemcpyDefault, ctx->stream));
    if (!is_device_ptr(mean) || !is_device_ptr(cov)) ctx->host_out = true;
    return finish_call(ctx, false, 0);
}

// numpy's standard_normal stream (csrc/numpy_normals.cuh) into device z; positions (nblocks + 1
// raw counts) into a device buffer the caller copies out.  Error bits come back through the
// context error word (ERR_BAD_RHS-style host check is not possible asynchronously): the caller
// reads nn_err with the outputs.
static int launch_numpy_normals(bd_ctx* ctx, const uint64_t* st4, long long count, long long block_len, double* z,
                                long long* positions) {
    if (!ctx->nn_tables) return fail(ctx, BD_ERR_STATE, "numpy ziggurat tables not set (bd_set_normal_tables)");
    if (count < 1 || block_len < 1 || count % block_len) return fail(ctx, BD_ERR_VALUE, "bad normal count / block");
    CU(ctx->nn_err.ensure(4));
    CU(cudaMemsetAsync(ctx->nn_err.p, 0, 4, ctx->stream));
    NumpyNormalArgs a{};
    a.state = U128{st4[0], st4[1]};
    a.inc = U128{st4[2], st4[3]};
    a.count = count;
    a.block_len = block_len;
    a.ki = ctx->nn_tab.as<uint64_t>();
    a.wi = reinterpret_cast<const double*>(a.ki + 256);
    a.fi = a.wi + 256;
    a.z = z;
    a.positions = positions;
    a.err = ctx->nn_err.as<int>();
    // grid-wide cooperative form: one position per thread over the whole GPU (2 grid barriers)
    int sms = 148, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    const long long R = count + count / 32 + 4096;
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, numpy_normals_grid_kernel, NN_GT, 0);
    const long long want = (R + NN_GT - 1) / NN_GT;
    const int grid = (int)std::max(1ll, std::min(want, (long long)sms * std::max(per_sm, 1)));
    if (coop && per_sm > 0) {
        CU(ctx->nn_raw.ensure((size_t)(R + NN_CMAX) * 8));
        CU(ctx->nn_x.ensure((size_t)R * 8));
        CU(ctx->nn_cs.ensure((size_t)R * 2 + 64));
        CU(ctx->nn_cnt.ensure((size_t)grid * 8));
        CU(ctx->nn_bar.ensure(8));
        CU(cudaMemsetAsync(ctx->nn_bar.p, 0, 8, ctx->stream));
        NumpyNormalGrid gg{};
        gg.a = a;
        gg.R = R;
        gg.raw = ctx->nn_raw.as<uint64_t>();
        gg.xv = ctx->nn_x.as<double>();
        gg.cv = ctx->nn_cs.as<unsigned char>();
        gg.st = gg.cv + ((R + 63) / 64) * 64;
        gg.cta_count = ctx->nn_cnt.as<long long>();
        gg.bar = ctx->nn_bar.as<unsigned>();
        void* args[] = {&gg};
        CU(cudaLaunchCooperativeKernel((const void*)numpy_normals_grid_kernel, dim3(grid), dim3(NN_GT), args, 0,
                                       ctx->stream));
    } else {
        raise_smem(numpy_normals_kernel, NN_SMEM);
        numpy_normals_kernel<<<1, NN_THREADS, NN_SMEM, ctx->stream>>>(a);
    }
    ctx->launches++;
    ctx->pending.push_back({&ctx->nn_err_host, ctx->nn_err.p, 4});
    ctx->host_out = true;
    ctx->nn_check = true;
    return 0;
}

// Single-scene CEM cycle as one cooperative persistent kernel (csrc/cem_persistent.cuh) when the
// batch maps to one CTA of 3-8 one-warp samples per SM (3-6 only with the remainder warp) on the
// BASELINE latency shape; returns 1
// when the shape does not apply (the caller runs the per-iteration launch chain instead).
static int try_cem_persistent(bd_ctx* ctx, const bd_cem_config* cfg, const CemState& s, const S1Args& s1, bool s1def,
                              const double* dz, const double* dwarm, const double* db, int it0, int it1) {
    if (ctx->opt_persist_off || ctx->timing || ctx->S != 1 || ctx->n_curv != 0 || ctx->m != 100 ||
        ctx->obs_pad != 10 || ctx->obs_sorted || !s1def || db != nullptr || ctx->p2p_epilogue || ctx->opt_lanes ||
        ctx->opt_spc)
        return 1;
    int sms = 148, coop = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
    cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
    const int B = cfg->batch;
    const int spc = (B + sms - 1) / sms;
    if (!coop || spc < BD_HELP_MIN || spc > 8 || (spc < 7 && !lat_helped(ctx, B))) return 1;
    const bool help = lat_helped(ctx, B);                           // + the remainder warp per worker
    const int grid = (B + spc - 1) / spc + 1, threads = 32 * (spc + (help ? 1 : 0));   // workers + control
    if (grid > sms) return 1;
    const int iters = cfg->am_iters;
    const size_t itmax_bytes = (size_t)iters * ITMAX_SLOTS * 4;
    if (int rc = ensure_itmax(ctx, itmax_bytes)) return rc;
    CU(ctx->w_replay.ensure(4));
    CU(ctx->w_order.ensure((size_t)B * 4));
    CU(ctx->c_bar.ensure(16));
    if (ctx->itmax_clean < itmax_bytes) CU(cudaMemsetAsync(ctx->w_itmax.p, 0, itmax_bytes, ctx->stream));
    ctx->itmax_clean = std::max(ctx->itmax_clean, itmax_bytes);
    CU(cudaMemsetAsync(ctx->c_bar.p, 0, 16, ctx->stream));
    CemPersistArgs pa{};
    pa.am = projection_args(ctx, B, ctx->w_xibar.as<double>(), iters, ctx->w_xi.as<double>(),
                            ctx->w_res.as<double>(), ctx->w_cost.as<double>());
    pa.am.s_cta = spc;
    pa.am.b = nullptr;
    pa.am.hist_out = nullptr;
    pa.am.replay = nullptr;
    pa.am.tol = cfg->tol;
    pa.am.iters_used = ctx->w_iters.as<int>();
    pa.am.replay_out = ctx->w_replay.as<int>();
    pa.am.done_ctr = nullptr;
    pa.cs = s;
    pa.s1 = s1;
    pa.z = dz;
    pa.warm = dwarm;
    pa.seed = cfg->seed;
    pa.scene_offset = cfg->scene_offset;
    pa.it0 = it0;
    pa.it1 = it1;
    pa.am_iters = iters;
    pa.params = ctx->w_params.as<double>();
    pa.order = ctx->w_order.as<int>();
    pa.bar = ctx->c_bar.as<unsigned>();
    const AmSmem lay(ctx->m, ctx->obs_pad, ctx->neq, 0, spc, threads, 32, false, iters, help ? 4 : 0);
    pa.s1_off = align_up(lay.total, 16);
    const size_t s1_bytes = (size_t)(2 * s1.nr * s1_ld(s1.nr) + 2 * NC * s1.m_seg + spc * MAX_DIM + spc * S1_VEC) * 8;
    pa.key_off = align_up(pa.s1_off + s1_bytes, 16);
    const size_t smem = pa.key_off + std::max((size_t)B * 8, rank_refit_smem(cfg->n_cons, cfg->n_elite, ctx->dim));
    if (smem > 200 * 1024) return 1;
    void* args[] = {&pa};
    cudaError_t e;
    auto launch = [&](auto kernel) {
        raise_smem(kernel, smem);
        return cudaLaunchCooperativeKernel((const void*)kernel, dim3(grid), dim3(threads), args, smem, ctx->stream);
    };
    if (help)
        e = spc == 3 ? launch(cem_persistent_kernel<128, 4>)
            : spc == 4 ? launch(cem_persistent_kernel<160, 4>)
            : spc == 5 ? launch(cem_persistent_kernel<192, 4>)
                     : spc == 6 ? launch(cem_persistent_kernel<224, 4>)
                                : spc == 7 ? launch(cem_persistent_kernel<256, 4>) : launch(cem_persistent_kernel<288, 4>);
    else
        e = spc == 7 ? launch(cem_persistent_kernel<224, 0>) : launch(cem_persistent_kernel<256, 0>);
    if (e == cudaErrorCooperativeLaunchTooLarge) {   // not co-resident on this device: launch chain instead
        cudaGetLastError();
        return 1;
    }
    if (e != cudaSuccess) return fail(ctx, BD_ERR_CUDA, "persistent CEM launch: %s", cudaGetErrorString(e));
    ctx->launches++;
    ctx->persistent_cycles++;
    return 0;
}

int bd_set_normal_tables(bd_ctx* ctx, const uint64_t* ki, const double* wi, const double* fi) {
    if (!ctx || !ki || !wi || !fi) return BD_ERR_VALUE;
    begin_call(ctx);
    CU(ctx->nn_tab.ensure(768 * 8));
    CU(cudaMemcpy(ctx->nn_tab.p, ki, 256 * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->nn_tab.as<uint64_t>() + 256, wi, 256 * 8, cudaMemcpyHostToDevice));
    CU(cudaMemcpy(ctx->nn_tab.as<uint64_t>() + 512, fi, 256 * 8, cudaMemcpyHostToDevice));
    ctx->nn_tables = true;
    return 0;
}

int bd_numpy_normals(bd_ctx* ctx, const uint64_t* pcg64_state, long long count, long long block_len, double* z,
                     int64_t* positions) {
    NvtxRange nvtx_("bd_numpy_normals");
    if (!ctx || !pcg64_state || !z || !positions || count < 1 || block_len < 1) return BD_ERR_VALUE;
    begin_call(ctx);
    int rc;
    double* dz;
    long long* dp;
    if ((rc = stage_out(ctx, z, (size_t)count, ctx->nn_z, &dz))) return rc;
    if ((rc = stage_out(ctx, reinterpret_cast<long long*>(positions), (size_t)(count / block_len + 1), ctx->nn_pos,
                        &dp)))
        return rc;
    if ((rc = launch_numpy_normals(ctx, pcg64_state, count, block_len, dz, dp))) return rc;
    return finish_call(ctx, false, 0);
}

int bd_cem_cycle(bd_ctx* ctx, int S, const bd_cem_config* cfg, const double* init_mean, const double* init_cov,
                 const double* z, const double* warm, int64_t* best_index, double* best_params, double* best_xi,
                 double* best_cost, double* best_residual, double* best_aug, double* stats, double* final_mean,
                 double* final_cov, int* iterations_done) {
    NvtxRange nvtx_("bd_cem_cycle");
    if (!ctx || !cfg) return BD_ERR_VALUE;
    int rc = require_solver(ctx, true);
    if (rc) return rc;
    const int B = cfg->batch, dim = ctx->dim, N = cfg->iterations;
    if (S != ctx->S || B < 1 || N < 1 || cfg->am_iters < 1 || !(cfg->tol > 0) || !init_mean || !init_cov)
        return fail(ctx, BD_ERR_VALUE, "bad CEM configuration");
    if (!(cfg->n_elite <= cfg->n_cons && cfg->n_cons <= B) || cfg->n_elite < 1 || cfg->n_cons > 1024)
        return fail(ctx, BD_ERR_VALUE, "need elites <= constraint_elites <= batch_size (<= 1024 constraint elites)");
    if (!(cfg->eta > 0 && cfg->eta <= 1) || !(cfg->gamma > 0)) return fail(ctx, BD_ERR_VALUE, "bad eta / gamma");
    if (B > (1 << 24)) return fail(ctx, BD_ERR_VALUE, "batch too large");
    const int it0 = cfg->iter_begin, it1 = cfg->iter_end > 0 ? cfg->iter_end : N;
    if (it0 < 0 || it0 >= it1 || it1 > N) return fail(ctx, BD_ERR_VALUE, "bad CEM iteration range");
    begin_call(ctx);
    const size_t tot = (size_t)S * B;
    const double *dz = nullptr, *dwarm = nullptr, *dm0, *dc0;
    if ((rc = stage_in(ctx, init_mean, (size_t)S * dim, &dm0))) return rc;
    if ((rc = stage_in(ctx, init_cov, (size_t)S * dim * dim, &dc0))) return rc;
    if ((rc = stage_in(ctx, z, z ? (size_t)(it1 - it0) * tot * dim : 0, &dz))) return rc;
    if ((rc = stage_in(ctx, warm, warm ? tot * dim : 0, &dwarm))) return rc;
    bool join_nn = false;
    if (!z && cfg->pcg64_state) {
        // numpy stream mode: the caller's Generator(PCG64) normals of every drawing iteration of the
        // range, generated on the device (the first iteration of a warm-started cycle draws none)
        const int first = (warm && it0 == 0) ? 1 : 0, nblk = (it1 - it0) - first;
        CU(ctx->nn_z.ensure((size_t)(it1 - it0) * tot * dim * 8));
        CU(ctx->nn_pos.ensure((size_t)(nblk + 1) * 8));
        if (nblk > 0) {
            if (!ctx->side) {
                CU(cudaStreamCreateWithFlags(&ctx->side, cudaStreamNonBlocking));
                CU(cudaEventCreateWithFlags(&ctx->nn_ready, cudaEventDisableTiming));
                CU(cudaEventCreateWithFlags(&ctx->nn_free, cudaEventDisableTiming));
            }
            if (ctx->nn_free_valid) CU(cudaStreamWaitEvent(ctx->side, ctx->nn_free, 0));
            cudaStream_t main_stream = ctx->stream;
            ctx->stream = ctx->side;
            rc = launch_numpy_normals(ctx, cfg->pcg64_state, (long long)nblk * tot * dim, (long long)tot * dim,
                                      ctx->nn_z.as<double>() + (size_t)first * tot * dim, ctx->nn_pos.as<long long>());
            ctx->stream = main_stream;
            if (rc) return rc;
            join_nn = true;                // the main stream joins after cem_init (below)
        } else {
            CU(cudaMemsetAsync(ctx->nn_pos.p, 0, 8, ctx->stream));
        }
        dz = ctx->nn_z.as<double>();
        if (cfg->pcg64_positions) {
            if (is_device_ptr(cfg->pcg64_positions)) {   // after the normals kernel on its stream
                CU(cudaMemcpyAsync(cfg->pcg64_positions, ctx->nn_pos.p, (size_t)(nblk + 1) * 8, cudaMemcpyDeviceToDevice,
                                   join_nn ? ctx->side : ctx->stream));
            } else {
                ctx->pending.push_back({cfg->pcg64_positions, ctx->nn_pos.p, (size_t)(nblk + 1) * 8});
                ctx->host_out = true;
            }
        }
        if (join_nn) CU(cudaEventRecord(ctx->nn_ready, ctx->side));
    }
    CU(ctx->c_mean.ensure((size_t)S * dim * 8));
    CU(ctx->c_cov.ensure((size_t)S * dim * dim * 8));
    CU(ctx->c_L.ensure((size_t)S * dim * dim * 8));
    CU(ctx->c_done.ensure((size_t)S * 4));
    CU(ctx->c_best_idx.ensure((size_t)S * 8));
    CU(ctx->c_best_p.ensure((size_t)S * dim * 8));
    CU(ctx->c_best_xi.ensure((size_t)S * NX * 8));
    CU(ctx->c_best_s.ensure((size_t)S * 3 * 8));
    CU(ctx->c_stats.ensure((size_t)S * N * 6 * 8));
    CU(ctx->w_params.ensure(tot * dim * 8));
    CU(ctx->w_xibar.ensure(tot * NX * 8));
    CU(ctx->w_xi.ensure(tot * NX * 8));
    CU(ctx->w_res.ensure(tot * 8));
    CU(ctx->w_cost.ensure(tot * 8));
    CU(ctx->w_iters.ensure((size_t)S * 4));
    CU(ctx->w_conf.ensure((size_t)S * 8));
    double* db = nullptr;
    if (ctx->with_goal) {
        CU(ctx->w_b.ensure(tot * ctx->neq * 8));
        db = ctx->w_b.as<double>();
    }
    CemState s{};
    s.S = S; s.B = B; s.dim = dim; s.n_cons = cfg->n_cons; s.n_elite = cfg->n_elite; s.iters = N;
    s.eta = cfg->eta; s.gamma = cfg->gamma; s.w_res = cfg->residual_weight;
    s.mean = ctx->c_mean.as<double>(); s.cov = ctx->c_cov.as<double>(); s.L = ctx->c_L.as<double>();
    s.err = ctx->w_err.as<int>(); s.done = ctx->c_done.as<int>();
    s.resid = ctx->w_res.as<double>(); s.cost = ctx->w_cost.as<double>(); s.params = ctx->w_params.as<double>();
    s.xi = ctx->w_xi.as<double>(); s.stats = ctx->c_stats.as<double>();
    s.best_index = ctx->c_best_idx.as<long long>(); s.best_params = ctx->c_best_p.as<double>();
    s.best_xi = ctx->c_best_xi.as<double>(); s.best_scal = ctx->c_best_s.as<double>();
    if (it0 == 0) {
        cem_init_kernel<<<S, 64, 0, ctx->stream>>>(s, dm0, dc0);
        ctx->launches++;
    }
    if (join_nn) CU(cudaStreamWaitEvent(ctx->stream, ctx->nn_ready, 0));   // the normals are ready
    CU(ctx->w_order.ensure(tot * 4));
    const size_t rsmem = rank_refit_smem(cfg->n_cons, cfg->n_elite, dim);
    raise_smem(rank_refit_kernel, rsmem);
    S1Args s1{};
    s1.total = S * B; s1.B = B; s1.dim = dim; s1.neq = ctx->neq1; s1.m_seg = ctx->m_seg;
    s1.with_goal = ctx->with_goal; s1.nr = NX + ctx->neq1; s1.nvar = NX;
    s1.qmx = ctx->qmx.as<double>(); s1.qmy = ctx->qmy.as<double>(); s1.kkt = ctx->kkt1.as<double>();
    s1.kinv = ctx->kinv1.as<double>(); s1.params = ctx->w_params.as<double>(); s1.bscene = ctx->bscene.as<double>();
    s1.xi_bar = ctx->w_xibar.as<double>(); s1.mu = nullptr; s1.b_out = db; s1.err = ctx->w_err.as<int>();
    const size_t s1smem = (size_t)(2 * s1.nr * s1_ld(s1.nr) + 2 * NC * s1.m_seg + 8 * MAX_DIM + 8 * S1_VEC) * 8;
    const bool s1def = s1.nr == S1_DEF_NR && dim == S1_DEF_DIM && ctx->m_seg == S1_DEF_MS && !ctx->with_goal;
    raise_smem(sample_stage1_kernel<true>, s1smem);
    raise_smem(sample_stage1_kernel<false>, s1smem);
    rc = S == 1 ? try_cem_persistent(ctx, cfg, s, s1, s1def, dz, dwarm, db, it0, it1) : 1;
    if (rc < 0) return rc;
    for (int it = rc == 0 ? it1 : it0; it < it1; ++it) {
        const double* zi = dz ? dz + (size_t)(it - it0) * tot * dim : nullptr;
        auto s1k = s1def ? sample_stage1_kernel<true> : sample_stage1_kernel<false>;
        s1k<<<(unsigned)((tot + 7) / 8), 256, s1smem, ctx->stream>>>(
            s, it, zi, it == 0 ? dwarm : nullptr, cfg->seed, cfg->scene_offset, ctx->w_params.as<double>(), s1);
        ctx->launches++;
        if ((rc = run_projection(ctx, B, ctx->w_xibar.as<double>(), db, cfg->am_iters, cfg->tol,
                                 ctx->w_xi.as<double>(), ctx->w_res.as<double>(), ctx->w_cost.as<double>(), nullptr,
                                 ctx->w_iters.as<int>(), ctx->w_conf.as<unsigned long long>(), false,
                                 false)))   // clip conflicts are not reported by the CEM cycle
            return rc;
        launch_rank_count(ctx, s.resid, s.err, S, B, ctx->w_order.as<int>());
        rank_refit_kernel<<<S, RANK_REFIT_THREADS, rsmem, ctx->stream>>>(s, it, ctx->w_order.as<int>());
        ctx->launches++;
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return fail(ctx, BD_ERR_CUDA, "CEM launch: %s", cudaGetErrorString(e));
    // outputs
    struct Out { void* dst; const void* src; size_t bytes; };
    const Out outs[] = {
        {best_index, ctx->c_best_idx.p, (size_t)S * 8},
        {best_params, ctx->c_best_p.p, (size_t)S * dim * 8},
        {best_xi, ctx->c_best_xi.p, (size_t)S * NX * 8},
        {stats, ctx->c_stats.p, (size_t)S * N * 6 * 8},
        {final_mean, ctx->c_mean.p, (size_t)S * dim * 8},
        {final_cov, ctx->c_cov.p, (size_t)S * dim * dim * 8},
        {iterations_done, ctx->c_done.p, (size_t)S * 4},
    };
    for (const Out& o : outs)
        if (o.dst) {
            if (is_device_ptr(o.dst)) {
                CU(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
            } else {
                ctx->pending.push_back({o.dst, o.src, o.bytes});
                ctx->host_out = true;
            }
        }
    double* scal[3] = {best_cost, best_residual, best_aug};
    for (int q = 0; q < 3; ++q)
        if (scal[q]) {
            if (is_device_ptr(scal[q])) {
                CU(cudaMemcpy2DAsync(scal[q], 8, ctx->c_best_s.as<double>() + q, 24, 8, S, cudaMemcpyDeviceToDevice,
                                     ctx->stream));
            } else {
                ctx->pending.push_back({scal[q], ctx->c_best_s.as<double>() + q, (size_t)S * 8, 24, 8});
                ctx->host_out = true;
            }
        }
    if (ctx->side) {                    // the numpy-stream buffers are free once this call's work is
        CU(cudaEventRecord(ctx->nn_free, ctx->stream));
        ctx->nn_free_valid = true;
    }
    return finish_call(ctx, false, 0);
}

// The last CEM iteration's batch of the preceding bd_cem_cycle call on this context: the arguments
// the reference hands its trace_hook(it, params, proj, costs, elite_idx) (pkg/bilevel.py:269-270).
int bd_cem_last_batch(bd_ctx* ctx, int S, int B, double* params, double* xi, double* residuals, double* cost) {
    NvtxRange nvtx_("bd_cem_last_batch");
    if (!ctx) return BD_ERR_VALUE;
    if (S != ctx->S || B < 1 || !ctx->dim) return fail(ctx, BD_ERR_VALUE, "bad batch (S=%d, B=%d)", S, B);
    const size_t tot = (size_t)S * B;
    if (ctx->w_params.bytes < tot * ctx->dim * 8 || ctx->w_xi.bytes < tot * NX * 8 || ctx->w_res.bytes < tot * 8 ||
        ctx->w_cost.bytes < tot * 8)
        return fail(ctx, BD_ERR_STATE, "no CEM batch of this size on the context (run bd_cem_cycle first)");
    begin_call(ctx);
    struct Out { void* dst; const void* src; size_t bytes; };
    const Out outs[] = {{params, ctx->w_params.p, tot * ctx->dim * 8}, {xi, ctx->w_xi.p, tot * NX * 8},
                        {residuals, ctx->w_res.p, tot * 8}, {cost, ctx->w_cost.p, tot * 8}};
    for (const Out& o : outs)
        if (o.dst) {
            if (is_device_ptr(o.dst)) {
                CU(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
            } else {
                ctx->pending.push_back({o.dst, o.src, o.bytes});
                ctx->host_out = true;
            }
        }
    return finish_call(ctx, false, 0);
}

// ------------------------------------------------------------------ scenes from worlds, controls
int bd_build_scenes(bd_ctx* ctx, int S, int n_veh_max, const double* ego, const double* veh, const int* n_veh,
                    const double* road, const bd_env* env, const double* times, double* ox_out, double* oy_out,
                    double* b0_out, double* limits_out, double* observations) {
    NvtxRange nvtx_("bd_build_scenes");
    if (!ctx || !env) return BD_ERR_VALUE;
    if (!ctx->m) return fail(ctx, BD_ERR_STATE, "basis not set");
    const int m = ctx->m, n_obs = env->max_obstacles;
    if (S < 1 || n_veh_max < 0 || n_obs < 0 || !ego || !n_veh || !road || !times || (n_veh_max > 0 && !veh))
        return fail(ctx, BD_ERR_VALUE, "bad build_scenes arguments");
    if (n_veh_max > 4096) return fail(ctx, BD_ERR_VALUE, "at most 4096 neighbours per world");
    begin_call(ctx);
    int rc;
    const double *de, *dv, *dr, *dt;
    const int* dn;
    if ((rc = stage_in(ctx, ego, (size_t)S * 8, &de))) return rc;
    if ((rc = stage_in(ctx, veh, (size_t)S * n_veh_max * 5, &dv))) return rc;
    if ((rc = stage_in(ctx, n_veh, (size_t)S, &dn))) return rc;
    if ((rc = stage_in(ctx, road, (size_t)S * 2, &dr))) return rc;
    if ((rc = stage_in(ctx, times, (size_t)m, &dt))) return rc;
    const int neq = ctx->neq ? ctx->neq : 6;
    const int nop = (n_obs + 1) / 2 * 2;
    const size_t no = (size_t)S * n_obs * m;
    CU(ctx->obs.ensure(((size_t)S * nop * m * 2 + 4) * sizeof(float)));
    CU(ctx->lim.ensure((size_t)S * sizeof(SceneLim)));
    CU(ctx->bscene.ensure((size_t)S * neq * 8));
    CU(ctx->lim64.ensure((size_t)S * 9 * 8));
    CU(ctx->ox64.ensure(no ? no * 8 : 8));
    CU(ctx->oy64.ensure(no ? no * 8 : 8));
    CU(ctx->w_err.ensure((size_t)S * 4));
    CU(clear_err(ctx, (size_t)S * 4));
    double *db0, *dobs;
    if ((rc = stage_out(ctx, b0_out, (size_t)S * 6, ctx->stage[6], &db0))) return rc;
    if ((rc = stage_out(ctx, observations, (size_t)S * OBS_DIM, ctx->stage[7], &dobs))) return rc;
    SceneBuildArgs a{};
    a.S = S; a.n_veh_max = n_veh_max; a.n_obs = n_obs; a.n_pad = nop; a.m = m; a.neq = neq;
    a.range = env->obstacle_range; a.wheelbase = env->wheelbase; a.v_max = env->v_max; a.a_max = env->a_max;
    a.k_max = env->kappa_max; a.c_max = env->c_max; a.v_min = env->v_min; a.other_len = env->other_length;
    a.other_wid = env->other_width;
    a.ego = de; a.veh = dv; a.n_veh = dn; a.road = dr; a.times = dt;
    a.tile = ctx->obs.as<float>(); a.lim = ctx->lim.as<SceneLim>(); a.bscene = ctx->bscene.as<double>();
    a.ox64 = ctx->ox64.as<double>(); a.oy64 = ctx->oy64.as<double>(); a.lim64 = ctx->lim64.as<double>();
    a.b0_out = db0; a.observation = dobs;
    const size_t smem = (size_t)n_veh_max * 8 + (size_t)(n_obs + OBS_NEIGHBORS) * 4 + (size_t)n_veh_max * 2 + 16;
    raise_smem(build_scene_kernel, smem);
    build_scene_kernel<<<S, 128, smem, ctx->stream>>>(a);
    ctx->launches++;
    // optional host-facing copies of the fp64 scene
    struct Out { void* dst; const void* src; size_t bytes; };
    const Out outs[] = {{ox_out, ctx->ox64.p, no * 8}, {oy_out, ctx->oy64.p, no * 8},
                        {limits_out, ctx->lim64.p, (size_t)S * 9 * 8}};
    for (const Out& o : outs)
        if (o.dst && o.bytes) {
            if (is_device_ptr(o.dst)) {
                CU(cudaMemcpyAsync(o.dst, o.src, o.bytes, cudaMemcpyDeviceToDevice, ctx->stream));
            } else {
                ctx->pending.push_back({o.dst, o.src, o.bytes});
                ctx->host_out = true;
            }
        }
    if ((rc = finish_tile(ctx, S, m, nop))) return rc;
    ctx->S = S;
    ctx->scene_obs = n_obs;
    ctx->obs_pad = nop;
    ctx->n_curv = 0;
    return finish_call(ctx, false, 0);
}

int bd_set_control_grid(bd_ctx* ctx, int n_ctrl, const double* wd, const double* wdd, double wheelbase,
                        double a_max, double steer_limit, double eps_v) {
    if (!ctx || n_ctrl < 1 || !wd || !wdd) return BD_ERR_VALUE;
    begin_call(ctx);
    CU(ctx->ctrl_wd.ensure((size_t)n_ctrl * NC * 8));
    CU(ctx->ctrl_wdd.ensure((size_t)n_ctrl * NC * 8));
    CU(cudaMemcpy(ctx->ctrl_wd.p, wd, (size_t)n_ctrl * NC * 8, cudaMemcpyDefault));
    CU(cudaMemcpy(ctx->ctrl_wdd.p, wdd, (size_t)n_ctrl * NC * 8, cudaMemcpyDefault));
    ctx->n_ctrl = n_ctrl;
    ctx->ctrl_wb = wheelbase;
    ctx->ctrl_amax = a_max;
    ctx->ctrl_steer = steer_limit;
    ctx->ctrl_eps = eps_v;
    return 0;
}

int bd_controls(bd_ctx* ctx, int count, const double* xi, double* accel, double* steer, int* singular) {
    NvtxRange nvtx_("bd_controls");
    if (!ctx) return BD_ERR_VALUE;
    if (!ctx->n_ctrl) return fail(ctx, BD_ERR_STATE, "control grid not set");
    if (count < 1 || !xi || !accel || !steer || !singular) return fail(ctx, BD_ERR_VALUE, "bad controls call");
    begin_call(ctx);
    int rc;
    const size_t n = (size_t)count * ctx->n_ctrl;
    const double* dxi;
    double *da, *ds;
    int* dsg;
    if ((rc = stage_in(ctx, xi, (size_t)count * NX, &dxi))) return rc;
    if ((rc = stage_out(ctx, accel, n, ctx->w_accel, &da))) return rc;
    if ((rc = stage_out(ctx, steer, n, ctx->w_steer, &ds))) return rc;
    if ((rc = stage_out_req(ctx, singular, (size_t)count, ctx->w_sing, &dsg))) return rc;
    CU(cudaMemsetAsync(dsg, 0, (size_t)count * 4, ctx->stream));
    ControlArgs c{};
    c.count = count; c.n_ctrl = ctx->n_ctrl; c.wd = ctx->ctrl_wd.as<double>(); c.wdd = ctx->ctrl_wdd.as<double>();
    c.xi = dxi; c.wheelbase = ctx->ctrl_wb; c.a_max = ctx->ctrl_amax; c.steer_limit = ctx->ctrl_steer;
    c.eps_v = ctx->ctrl_eps; c.accel = da; c.steer = ds; c.singular = dsg;
    controls_kernel<<<(unsigned)((n + 255) / 256), 256, 0, ctx->stream>>>(c);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

// ------------------------------------------------------------------ CVAE decoder
int bd_cvae_set_weights(bd_ctx* ctx, int n_layers, const int* dims, const float* const* W, const float* const* b) {
    if (!ctx || n_layers < 1 || n_layers > 16 || !dims || !W || !b) return BD_ERR_VALUE;
    begin_call(ctx);
    for (auto* p : ctx->cvae_w) delete p;
    for (auto* p : ctx->cvae_b) delete p;
    for (auto* p : ctx->cvae_w16) delete p;
    ctx->cvae_w.clear();
    ctx->cvae_b.clear();
    ctx->cvae_w16.clear();
    ctx->cvae_dims.assign(dims, dims + n_layers + 1);
    ctx->fz_count = -1;                  // cached fused-decoder tensor maps refer to the old weights
    for (int l = 0; l < n_layers; ++l) {
        const size_t nw = (size_t)dims[l] * dims[l + 1], nb = dims[l + 1];
        if (dims[l] < 1 || dims[l + 1] < 1) return fail(ctx, BD_ERR_VALUE, "bad layer dims");
        auto* wb = new DevBuf();
        auto* bb = new DevBuf();
        ctx->cvae_w.push_back(wb);
        ctx->cvae_b.push_back(bb);
        CU(wb->ensure(nw * 4));
        CU(bb->ensure(nb * 4));
        CU(cudaMemcpy(wb->p, W[l], nw * 4, cudaMemcpyDefault));
        CU(cudaMemcpy(bb->p, b[l], nb * 4, cudaMemcpyDefault));
        // bf16 copy for the tensor-core layers
        std::vector<float> hw(nw);
        CU(cudaMemcpy(hw.data(), W[l], nw * 4, cudaMemcpyDefault));
        std::vector<__nv_bfloat16> h16(nw);
        for (size_t i = 0; i < nw; ++i) h16[i] = __float2bfloat16_rn(hw[i]);
        auto* w16 = new DevBuf();
        ctx->cvae_w16.push_back(w16);
        CU(w16->ensure(nw * 2));
        CU(cudaMemcpy(w16->p, h16.data(), nw * 2, cudaMemcpyHostToDevice));
    }
    return 0;
}

namespace {
PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

// 2-D bf16 row-major [rows x cols] tensor map with a box_rows x 64-col box and 128-byte swizzle.
// [K block][row][64] view of a row-major rows x cols bf16 matrix (cols a multiple of 64): a box of
// kg K blocks x box_rows rows lands as kg consecutive 128-byte-swizzled K-major tiles.
bool make_map_bf16_kblocks(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows,
                           uint32_t kg) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[3] = {64, rows, cols / 64};
    const cuuint64_t strides[2] = {cols * 2, 128};
    const cuuint32_t box[3] = {64, box_rows, kg};
    const cuuint32_t estr[3] = {1, 1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool make_map_bf16(CUtensorMap* map, const void* base, uint64_t rows, uint64_t cols, uint32_t box_rows = TC_BM) {
    auto enc = tensor_map_encoder();
    if (!enc) return false;
    const cuuint64_t dims[2] = {cols, rows};
    const cuuint64_t strides[1] = {cols * 2};
    const cuuint32_t box[2] = {(cuuint32_t)TC_BK, (cuuint32_t)box_rows};
    const cuuint32_t estr[2] = {1, 1};
    return enc(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}
}  // namespace

// The decoder's launches for `count` samples (inputs and the count x out_dim output on the device).
static int cvae_decode_dev(bd_ctx* ctx, int count, const float* dobs, const float* dz, double* dout) {
    const auto& d = ctx->cvae_dims;
    const int L = (int)ctx->cvae_w.size();
    const int zdim = d[0] - CVAE_OBS;
    int widest = 0;
    for (int l = 1; l <= L; ++l) widest = widest > d[l] ? widest : d[l];
    bool tc_ok = ctx->cvae_tc && L >= 3 && tensor_map_encoder() != nullptr;
    for (int l = 1; l < L - 1 && tc_ok; ++l) tc_ok = d[l] % TC_BK == 0 && d[l + 1] % TC_BN == 0;
    // the whole decoder as one persistent cooperative kernel (csrc/cvae_fused.cuh)
    bool fused_ok = tc_ok && ctx->cvae_fused && L - 2 <= FZ_MAXH && d[L] <= FZ_MAXOUT && zdim <= FZ_MAXZ / 2;
    for (int l = 1; l < L && fused_ok; ++l) fused_ok = d[l] % FZ_BN == 0 && d[l] % (FZ_BK * FZ_KG) == 0;
    if (fused_ok) {
        int sms = 148, coop = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, ctx->device);
        cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, ctx->device);
        const int nh = L - 2, mblocks = (count + FZ_BM - 1) / FZ_BM;
        int tiles = 0;
        for (int l = 0; l <= nh; ++l) tiles = std::max(tiles, mblocks * (d[l + 1] / FZ_BN));
        const int grid = std::min(tiles, sms);
        if (coop) {
            const size_t mpad = (size_t)mblocks * FZ_BM;
            size_t act_elems = 0;                 // one buffer per layer (rows of a block flow through layers)
            for (int l = 0; l < nh; ++l) act_elems += mpad * d[l + 1];
            CU(ctx->cvae_a0.ensure(act_elems * 2));
            CU(ctx->cvae_h0.ensure((size_t)(d[L - 1] / FZ_BN) * count * d[L] * 4));
            // arrival counters grow by (tiles per row block) each launch; reset when (re)allocated,
            // when the layout changes or long before they could wrap
            const size_t ctr_bytes = (size_t)(nh + 1) * mblocks * 4;
            if (ctx->cvae_ready.bytes < ctr_bytes || ctx->fz_ctr_mblocks != mblocks || ctx->fz_epoch >= (1u << 20)) {
                CU(ctx->cvae_ready.ensure(ctr_bytes));
                CU(cudaMemsetAsync(ctx->cvae_ready.p, 0, ctx->cvae_ready.bytes, ctx->stream));
                ctx->fz_epoch = 0;
                ctx->fz_ctr_mblocks = mblocks;
            }
            ++ctx->fz_epoch;
            FusedArgs fa{};
            FusedMaps fm{};
            fa.count = count; fa.nh = nh; fa.zdim = zdim;
            for (int l = 0; l <= L; ++l) fa.dims[l] = d[l];
            fa.W0 = ctx->cvae_w[0]->as<float>();
            for (int l = 0; l < L; ++l) fa.bias[l] = ctx->cvae_b[l]->as<float>();
            fa.Wlast = ctx->cvae_w[L - 1]->as<float>();
            fa.obs = dobs; fa.z = dz;
            size_t off = 0;
            for (int l = 0; l < nh; ++l) {
                fa.act[l] = ctx->cvae_a0.as<__nv_bfloat16>() + off;
                off += mpad * d[l + 1];
            }
            fa.act[nh] = nullptr;                 // the last hidden layer feeds the fused output layer
            fa.partial = ctx->cvae_h0.as<float>();
            fa.out = dout;
            fa.ready = ctx->cvae_ready.as<unsigned>();
            fa.epoch = ctx->fz_epoch;
            if (ctx->fz_count != count || ctx->fz_key_a != ctx->cvae_a0.p || ctx->fz_key_w != ctx->cvae_w16[1]->p) {
                ctx->fz_count = -1;
                for (int h = 0; h < nh; ++h) {
                    const int l = h + 1;
                    if (!make_map_bf16_kblocks(&ctx->fz_maps.a[h], fa.act[l - 1], (uint64_t)count, (uint64_t)d[l],
                                               FZ_BM, FZ_KG) ||
                        !make_map_bf16_kblocks(&ctx->fz_maps.b[h], ctx->cvae_w16[l]->p, (uint64_t)d[l + 1],
                                               (uint64_t)d[l], FZ_BN, FZ_KG))
                        return fail(ctx, BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
                }
                ctx->fz_count = count;
                ctx->fz_key_a = ctx->cvae_a0.p;
                ctx->fz_key_w = ctx->cvae_w16[1]->p;
            }
            fm = ctx->fz_maps;
            raise_smem(cvae_fused_kernel, FZ_SMEM);
            void* args[] = {&fm, &fa};
            cudaError_t e = cudaLaunchCooperativeKernel((const void*)cvae_fused_kernel, dim3(grid), dim3(128), args,
                                                        FZ_SMEM, ctx->stream);
            if (e != cudaSuccess) return fail(ctx, BD_ERR_CUDA, "fused CVAE launch: %s", cudaGetErrorString(e));
            ctx->launches++;
            return 0;
        }
    }
    if (tc_ok) {
        const int mpad = (count + TC_BM - 1) / TC_BM * TC_BM;
        CU(ctx->cvae_a0.ensure((size_t)mpad * widest * 2));
        CU(ctx->cvae_a1.ensure((size_t)mpad * widest * 2));
        CU(cudaMemsetAsync(ctx->cvae_a0.p, 0, (size_t)mpad * widest * 2, ctx->stream));
        auto* cur = ctx->cvae_a0.as<__nv_bfloat16>();
        auto* nxt = ctx->cvae_a1.as<__nv_bfloat16>();
        cvae_first_layer_bf16<<<dim3((d[1] + 127) / 128, (count + 31) / 32), dim3(128), 0, ctx->stream>>>(
            count, d[1], zdim, ctx->cvae_w[0]->as<float>(), ctx->cvae_b[0]->as<float>(), dobs, dz, cur);
        ctx->launches++;
        raise_smem(cvae_tc_linear, TC_SMEM);
        for (int l = 1; l < L - 1; ++l) {
            CUtensorMap ma, mb;
            if (!make_map_bf16(&ma, cur, (uint64_t)count, (uint64_t)d[l]) ||
                !make_map_bf16(&mb, ctx->cvae_w16[l]->p, (uint64_t)d[l + 1], (uint64_t)d[l]))
                return fail(ctx, BD_ERR_CUDA, "cuTensorMapEncodeTiled failed");
            dim3 grid(d[l + 1] / TC_BN, mpad / TC_BM);
            cvae_tc_linear<<<grid, 128, TC_SMEM, ctx->stream>>>(ma, mb, count, d[l + 1], d[l],
                                                                ctx->cvae_b[l]->as<float>(), nxt, 1);
            ctx->launches++;
            auto* t = cur;
            cur = nxt;
            nxt = t;
        }
        cvae_last_layer_bf16<<<(count + 7) / 8, 256, 0, ctx->stream>>>(count, d[L - 1], d[L], cur,
                                                                       ctx->cvae_w[L - 1]->as<float>(),
                                                                       ctx->cvae_b[L - 1]->as<float>(), dout);
        ctx->launches++;
        return 0;
    }
    CU(ctx->cvae_h0.ensure((size_t)count * widest * 4));
    CU(ctx->cvae_h1.ensure((size_t)count * widest * 4));
    // layer 0: scene part W[:, :55] obs is shared by every sample
    cvae_first_layer<<<dim3((d[1] + 127) / 128, (count + 31) / 32), dim3(128), 0, ctx->stream>>>(
        count, d[1], zdim, ctx->cvae_w[0]->as<float>(), ctx->cvae_b[0]->as<float>(), dobs, dz,
        ctx->cvae_h0.as<float>());
    ctx->launches++;
    float* cur = ctx->cvae_h0.as<float>();
    float* nxt = ctx->cvae_h1.as<float>();
    for (int l = 1; l < L; ++l) {
        const bool last = (l == L - 1);
        dim3 grid((d[l + 1] + CVAE_BN - 1) / CVAE_BN, (count + CVAE_BM - 1) / CVAE_BM);
        cvae_linear<<<grid, CVAE_THREADS, 0, ctx->stream>>>(count, d[l], d[l + 1], cur, ctx->cvae_w[l]->as<float>(),
                                                            ctx->cvae_b[l]->as<float>(), nxt, last ? 0 : 1);
        ctx->launches++;
        float* t = cur;
        cur = nxt;
        nxt = t;
    }
    cvae_to_double<<<(unsigned)(((size_t)count * d[L] + 255) / 256), 256, 0, ctx->stream>>>(cur, dout,
                                                                                           (size_t)count * d[L]);
    ctx->launches++;
    return 0;
}

static int cvae_stage_inputs(bd_ctx* ctx, int count, const float* obs, const float* z, const float** dobs,
                             const float** dz) {
    if (ctx->cvae_w.empty()) return fail(ctx, BD_ERR_STATE, "CVAE weights not set");
    const int zdim = ctx->cvae_dims[0] - CVAE_OBS;
    if (zdim < 1) return fail(ctx, BD_ERR_VALUE, "first layer must take 55 observation + latent inputs");
    int rc;
    if ((rc = stage_in(ctx, obs, (size_t)CVAE_OBS, dobs))) return rc;
    return stage_in(ctx, z, (size_t)count * zdim, dz);
}

int bd_cvae_decode(bd_ctx* ctx, int count, const float* obs, const float* z, double* params) {
    NvtxRange nvtx_("bd_cvae_decode");
    if (!ctx || count < 1 || !obs || !z || !params) return BD_ERR_VALUE;
    begin_call(ctx);
    int rc;
    const float *dobs, *dz;
    if ((rc = cvae_stage_inputs(ctx, count, obs, z, &dobs, &dz))) return rc;
    double* dout;
    if ((rc = stage_out(ctx, params, (size_t)count * ctx->cvae_dims.back(), ctx->stage[7], &dout))) return rc;
    if ((rc = cvae_decode_dev(ctx, count, dobs, dz, dout))) return rc;
    return finish_call(ctx, false, 0);
}

// p = decode * scale + shift, rounded like the host's two float64 steps (no fused multiply-add).
__global__ void rows_affine_kernel(int count, int dim, double* rows, const double* scale, const double* shift) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= (long long)count * dim) return;
    const int c = (int)(i % dim);
    double v = rows[i];
    if (scale) v = __dmul_rn(v, scale[c]);
    if (shift) v = __dadd_rn(v, shift[c]);
    rows[i] = v;
}

int bd_cvae_warm_start(bd_ctx* ctx, int count, const float* obs, const float* z, const double* scale,
                       const double* shift, double* params, const double** rows_dev) {
    NvtxRange nvtx_("bd_cvae_warm_start");
    if (!ctx || count < 1 || !obs || !z || !rows_dev) return BD_ERR_VALUE;
    begin_call(ctx);
    int rc;
    const float *dobs, *dz;
    if ((rc = cvae_stage_inputs(ctx, count, obs, z, &dobs, &dz))) return rc;
    const int dim = ctx->cvae_dims.back();
    const double *dsc = nullptr, *dsh = nullptr;
    if ((rc = stage_in(ctx, scale, (size_t)dim, &dsc))) return rc;
    if ((rc = stage_in(ctx, shift, (size_t)dim, &dsh))) return rc;
    CU(ctx->cvae_warm.ensure((size_t)count * dim * 8));
    double* rows = ctx->cvae_warm.as<double>();
    if ((rc = cvae_decode_dev(ctx, count, dobs, dz, rows))) return rc;
    if (dsc || dsh) {
        rows_affine_kernel<<<(unsigned)(((size_t)count * dim + 255) / 256), 256, 0, ctx->stream>>>(count, dim, rows,
                                                                                                  dsc, dsh);
        ctx->launches++;
    }
    if (params) {
        if (is_device_ptr(params)) {
            CU(cudaMemcpyAsync(params, rows, (size_t)count * dim * 8, cudaMemcpyDeviceToDevice, ctx->stream));
        } else {
            ctx->pending.push_back({params, rows, (size_t)count * dim * 8});
            ctx->host_out = true;
        }
    }
    *rows_dev = rows;
    return finish_call(ctx, false, 0);
}


int bd_sim_run(bd_ctx* ctx, int S, int n_max, double* ego, double* ego_ts, double* veh, double* vext, const int* n_veh,
               const double* road, double* world, const bd_traffic* tp, int n_steps, const double* controls, int n_ctrl,
               int ctrl_offset, const double* x_end, int* active, int* steps_done, double* snapshots) {
    NvtxRange nvtx_("bd_sim_run");
    if (!ctx) return BD_ERR_VALUE;
    if (S < 1 || n_max < 0 || n_steps < 0 || !tp || !ego || !ego_ts || !n_veh || !road || !world ||
        (n_max > 0 && (!veh || !vext)) || (n_steps > 0 && (!controls || n_ctrl < 1)) || ctrl_offset < 0)
        return fail(ctx, BD_ERR_VALUE, "bad sim_run arguments");
    if (n_max > 4096) return fail(ctx, BD_ERR_VALUE, "at most 4096 neighbours per world");
    if (!(tp->dt > 0) || !(tp->wheelbase > 0) || !(tp->idm_v0 > 0) || !(tp->idm_a_max > 0) || !(tp->idm_b_comfort > 0))
        return fail(ctx, BD_ERR_VALUE, "traffic constants must be positive");
    begin_call(ctx);
    if (n_steps == 0) return 0;
    int rc;
    SimArgs a{};
    a.S = S; a.n_max = n_max; a.n_steps = n_steps; a.n_ctrl = n_ctrl; a.ctrl_offset = ctrl_offset;
    a.period = (int)std::max(1.0, std::nearbyint(1.0 / tp->dt));     // max(1, int(round(1.0 / dt)))
    a.dt = tp->dt; a.wheelbase = tp->wheelbase;
    a.idm_v0 = tp->idm_v0; a.idm_T = tp->idm_time_headway; a.idm_s0 = tp->idm_s0; a.idm_a = tp->idm_a_max;
    a.idm_b = tp->idm_b_comfort; a.idm_delta = tp->idm_delta; a.idm_bhard = tp->idm_b_hard;
    a.idm_sqrt_ab2 = 2.0 * std::sqrt(tp->idm_a_max * tp->idm_b_comfort);
    a.pol = tp->mobil_politeness; a.b_safe = tp->mobil_b_safe; a.a_thr = tp->mobil_a_threshold;
    a.cooldown = tp->mobil_cooldown;
    if ((rc = stage_inout(ctx, ego, (size_t)S * 8, ctx->sim_io[0], &a.ego))) return rc;
    if ((rc = stage_inout(ctx, ego_ts, (size_t)S, ctx->sim_io[1], &a.ego_ts))) return rc;
    if ((rc = stage_inout(ctx, veh, (size_t)S * n_max * 5, ctx->sim_io[2], &a.veh))) return rc;
    if ((rc = stage_inout(ctx, vext, (size_t)S * n_max * VEXT, ctx->sim_io[3], &a.vext))) return rc;
    if ((rc = stage_inout(ctx, world, (size_t)S * 5, ctx->sim_io[4], &a.world))) return rc;
    if ((rc = stage_inout(ctx, active, active ? (size_t)S : 0, ctx->sim_io[5], &a.active))) return rc;
    if ((rc = stage_in(ctx, n_veh, (size_t)S, &a.n_veh))) return rc;
    if ((rc = stage_in(ctx, road, (size_t)S * 2, &a.road))) return rc;
    if ((rc = stage_in(ctx, controls, (size_t)S * n_ctrl * 2, &a.ctrl))) return rc;
    if ((rc = stage_in(ctx, x_end, x_end ? (size_t)S : 0, &a.x_end))) return rc;
    if ((rc = stage_out(ctx, steps_done, (size_t)S, ctx->sim_io[6], &a.steps_done))) return rc;
    if ((rc = stage_out(ctx, snapshots, (size_t)S * n_steps * (8 + 4 * n_max), ctx->w_hist, &a.snap))) return rc;
    const size_t smem = (size_t)(n_max + 1) * (6 * sizeof(double) + 2 * sizeof(int));
    raise_smem(sim_kernel, smem);
    sim_kernel<<<S, 128, smem, ctx->stream>>>(a);
    ctx->launches++;
    return finish_call(ctx, false, 0);
}

}  // extern "C"
