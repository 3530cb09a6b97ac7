// C ABI of libpbp.so (include/pbp.h): device context, argument checking
// with the reference's exception texts, kernel orchestration and the
// host-side code helpers (construction, transform, encode).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <string>
#include <vector>

#include "../../include/pbp.h"
#include "pbp_common.cuh"

namespace pbp {
// kernels (bp_generic.cu, bp_warp.cu, channel.cu)
cudaError_t launch_generic(const DecodeArgs& a, int grid, cudaStream_t stream);
size_t generic_smem_bytes(int n);
long long generic_scratch_elems(int n, int m);
bool generic_in_smem(int n, int m, bool f64);
cudaError_t launch_warp(const DecodeArgs& a, int grid, cudaStream_t st);
int warp_kernel_supported(int m);
int warp_blocks_per_sm(int m, int kind);
int warp_kernel_warps(int m);
size_t warp_smem_bytes(int m, int kind);
int cta_kernel_supported(int m);
long long cta_scratch_floats(int m);
cudaError_t launch_cta(const DecodeArgs& a, int grid, cudaStream_t st);
int cta_blocks_per_sm(int m, int kind);
size_t cta_smem_bytes(int m);
int cta_warps(int m);
bool cta_pair_on(int m, int kind);
size_t cta_pair_smem_bytes(int m);
int cta_pair_warps_per_sm(int m);
cudaError_t launch_channel(const GenArgs& g, int grid, cudaStream_t stream);
long long channel_seed_words(long long count);
}  // namespace pbp

namespace {

thread_local std::string g_err;

int fail(int status, const std::string& msg) {
    g_err = msg;
    return status;
}

int cuda_fail(cudaError_t e, const char* where) {
    return fail(PBP_ECUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

#define PBP_CUDA(call)                                   \
    do {                                                 \
        cudaError_t e_ = (call);                         \
        if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
    } while (0)

bool is_pow2(long long v) { return v > 0 && (v & (v - 1)) == 0; }

int log2i(int n) {
    int m = 0;
    while ((1 << m) < n) ++m;
    return m;
}

template <class T>
struct DevBuf {
    T* p = nullptr;
    size_t cap = 0;
    int ensure(size_t count) {
        if (count <= cap) return PBP_OK;
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(count, 1);
        cudaError_t e = cudaMalloc(&p, want * sizeof(T));
        if (e != cudaSuccess) return cuda_fail(e, "cudaMalloc");
        cap = want;
        return PBP_OK;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
};

}  // namespace

// Launch resources of one in-flight decode: work queue, re-route list and
// scratch are per launch, so decodes on different streams need their own.
struct DecodeSlot {
    cudaStream_t stream = nullptr;     // slot 0: the context stream
    cudaEvent_t done = nullptr;        // after the slot's last use (any stream)
    DevBuf<unsigned long long> ctl;    // [0] warp queue, [1] generic queue, [2] list length
    DevBuf<long long> list;
    DevBuf<float> scratch;             // generic kernel: per-CTA message arrays
    DevBuf<float> r0s;                 // warp kernel: per-CTA channel LLRs
    // frames generated on the device by simulate_point (asynchronous calls)
    DevBuf<float> gen_llr;
    DevBuf<double> gen_llr64;
    DevBuf<uint32_t> gen_truth;
    DevBuf<unsigned long long> gen_mt;  // seeded mt19937_64 states of one generation piece
};
constexpr int kSlots = 3;

struct pbp_ctx {
    int device = 0;
    int sm_count = 0;
    cudaStream_t stream = nullptr;
    DecodeSlot slot[kSlots];
    int next_slot = 0;  // device-pointer calls rotate over the slots
    // code tables
    std::vector<uint8_t> code_key;
    int n = 0, m = 0, k = 0;
    DevBuf<uint32_t> frozen_bits;
    DevBuf<uint8_t> frozen_rows;
    DevBuf<int> info_rows;
    DevBuf<unsigned long long> counters;
    DevBuf<unsigned long long> rerouted;  // per launch of the last call: frames re-routed
    int n_launch_sets = 0;
    long long rerouted_host = -1;         // the last call's count when known on the host
    int warp_occ[15][3] = {};             // resident fast-kernel CTAs per SM by (m, kind), 0 = not queried
    DevBuf<long long> blist;              // batch-wide re-route list (pipelined host batch)
    DevBuf<unsigned long long> bctl;      // [0] its length, [1] generic queue
    // host-API staging
    DevBuf<float> llr;
    DevBuf<double> llr64;
    DevBuf<uint32_t> ubits;
    DevBuf<int> iters, nev, events;
    DevBuf<uint32_t> evx;  // trace: each event's x_hat bits
    DevBuf<long long> pe;
    DevBuf<uint8_t> stop;
    int last_launches = 0;
    int force_generic = 0;
};

namespace {

int check_code(const pbp_code* code) {
    if (!code || !code->frozen) return fail(PBP_EINVAL, "pbp_code: null code or frozen mask");
    // the generic decoder keeps a frame's bit state (1.5 n bytes) in shared memory
    if (!is_pow2(code->n) || code->n > (1 << 17))
        return fail(PBP_EINVAL, "pbp_code: n must be a power of two <= 131072");
    if (code->m != log2i(code->n)) return fail(PBP_EINVAL, "pbp_code: m != log2(n)");
    int frozen = 0;
    for (int i = 0; i < code->n; ++i) frozen += code->frozen[i] ? 1 : 0;
    if (code->k != code->n - frozen)
        return fail(PBP_EINVAL, "pbp_code: k inconsistent with the frozen mask");
    if (code->k < 1) return fail(PBP_EINVAL, "from_frozen_mask: no information positions");
    return PBP_OK;
}

int upload_code(pbp_ctx* ctx, const pbp_code* code) {
    int rc = check_code(code);
    if (rc) return rc;
    std::vector<uint8_t> key(code->frozen, code->frozen + code->n);
    if (ctx->n == code->n && key == ctx->code_key) return PBP_OK;
    // asynchronous decodes of the previous code (any stream) still read the tables
    PBP_CUDA(cudaDeviceSynchronize());
    const int n = code->n, nw = (n + 31) / 32;
    std::vector<uint32_t> bits(nw, 0u);
    std::vector<uint8_t> rows(n);
    std::vector<int> info;
    for (int r = 0; r < n; ++r) {
        rows[r] = code->frozen[r] ? 1 : 0;
        if (rows[r]) bits[r >> 5] |= 1u << (r & 31);
        else info.push_back(r);
    }
    if ((rc = ctx->frozen_bits.ensure(nw)) || (rc = ctx->frozen_rows.ensure(n)) ||
        (rc = ctx->info_rows.ensure(info.size())))
        return rc;
    PBP_CUDA(cudaMemcpyAsync(ctx->frozen_bits.p, bits.data(), nw * 4, cudaMemcpyHostToDevice, ctx->stream));
    PBP_CUDA(cudaMemcpyAsync(ctx->frozen_rows.p, rows.data(), n, cudaMemcpyHostToDevice, ctx->stream));
    PBP_CUDA(cudaMemcpyAsync(ctx->info_rows.p, info.data(), info.size() * 4, cudaMemcpyHostToDevice, ctx->stream));
    PBP_CUDA(cudaStreamSynchronize(ctx->stream));
    ctx->code_key = std::move(key);
    ctx->n = n;
    ctx->m = code->m;
    ctx->k = code->k;
    return PBP_OK;
}

struct DecodeReq {
    int kind = 0;
    const float* llr = nullptr;
    const double* llr64 = nullptr;  // set: decode in fp64 (the reference as shipped)
    double alpha64 = 0.9375;
    long long frames = 0;
    float alpha = 0.9375f;
    int max_iter = 40;
    uint32_t* u_bits = nullptr;
    int* iters = nullptr;
    long long* pe = nullptr;
    uint8_t* stop = nullptr;
    int* nev = nullptr;
    int* events = nullptr;
    int ev_cap = 0;
    uint32_t* ev_xhat = nullptr;
    const uint32_t* truth = nullptr;
    unsigned long long* counters = nullptr;
    int cnt_batch = 0;  // > 0: one counter set per cnt_batch frames (run_point batches)
    bool force_generic = false;
    // fast path: re-routed frames go to this list (indices + frame_base) and
    // the caller runs the generic pass later (run_generic_list)
    long long* list = nullptr;
    unsigned long long* list_len = nullptr;
    long long frame_base = 0;
};

// Start of an API call that launches decodes: launch statistics restart.
int begin_call(pbp_ctx* ctx, int max_sets) {
    ctx->last_launches = 0;
    ctx->n_launch_sets = 0;
    ctx->rerouted_host = -1;
    return ctx->rerouted.ensure((size_t)std::max(max_sets, 16));
}

// launch resources for an asynchronous device-pointer call: rotated, so
// calls on different streams overlap; run_decode orders each slot's uses
DecodeSlot& next_slot(pbp_ctx* ctx) {
    DecodeSlot& s = ctx->slot[ctx->next_slot];
    ctx->next_slot = (ctx->next_slot + 1) % kSlots;
    return s;
}

// fast kernel for code length 2^m: 1 = warp-resident (n = 128..1024),
// 2 = CTA per frame with register passes (n = 2048..16384), 0 = none
int fast_kernel(int m) {
    return pbp::warp_kernel_supported(m) ? 1 : (pbp::cta_kernel_supported(m) ? 2 : 0);
}

// resident fast-kernel CTAs per SM (queried once per context and code length)
int warp_occupancy(pbp_ctx* ctx, int kind) {
    int& v = ctx->warp_occ[ctx->m][kind];
    if (!v)
        v = std::max(1, fast_kernel(ctx->m) == 1 ? pbp::warp_blocks_per_sm(ctx->m, kind)
                                                 : pbp::cta_blocks_per_sm(ctx->m, kind));
    return v;
}

// Grid of the generic kernel: every frame when it decodes alone, the
// re-routed frames (at most one per SM at a time) after the warp kernel;
// bounded by 4 GiB of per-CTA scratch.
long long generic_grid(const pbp_ctx* ctx, long long frames, bool fast, int esz = 1) {
    const long long gfm = fast ? std::min<long long>(frames, ctx->sm_count) : frames;
    const long long stride = pbp::generic_scratch_elems(ctx->n, ctx->m) * esz;
    // latency-bound (one CTA per frame, barriers per stage): fill every SM
    // (measured: 4 -> 8 CTAs/SM is +26 % at n = 4096, +23 % at 16384)
    long long grid = std::min<long long>(gfm, (long long)ctx->sm_count * 8);
    const long long max_scratch_floats = 1ll << 30;  // 4 GiB
    return std::max<long long>(1, std::min<long long>(grid, max_scratch_floats / stride));
}

// Size a slot's buffers for decodes of up to `frames` frames (before any
// asynchronous work is queued: reallocation synchronises the device).
int size_slot(pbp_ctx* ctx, DecodeSlot& s, int kind, long long frames) {
    if (kind < 0 || kind > 2) return fail(PBP_EINVAL, "unknown decoder kind");  // indexes warp_occ
    int rc;
    if ((rc = s.ctl.ensure(4)) || (rc = s.list.ensure(std::max<long long>(frames, 1)))) return rc;
    size_t scratch = 0;
    if (fast_kernel(ctx->m)) {
        const int per_sm = warp_occupancy(ctx, kind);
        const long long grid = std::min<long long>((long long)per_sm * ctx->sm_count, std::max<long long>(frames, 1));
        if (fast_kernel(ctx->m) == 1) {
            if ((rc = s.r0s.ensure((size_t)(grid * ctx->n)))) return rc;
        } else {
            scratch = (size_t)(grid * pbp::cta_scratch_floats(ctx->m));
        }
    }
    const bool fast = !ctx->force_generic && fast_kernel(ctx->m);
    if (!pbp::generic_in_smem(ctx->n, ctx->m, false))
        scratch = std::max(scratch, (size_t)(generic_grid(ctx, frames, fast) * pbp::generic_scratch_elems(ctx->n, ctx->m)));
    return scratch ? s.scratch.ensure(scratch) : PBP_OK;
}

// Launch the decode of `frames` frames already on the device, with slot s's
// launch resources, on stream st.
int run_decode(pbp_ctx* ctx, const DecodeReq& r, DecodeSlot& s, cudaStream_t st) {
    if (r.kind < 0 || r.kind > 2) return fail(PBP_EINVAL, "unknown decoder kind");
    if (r.frames < 0) return fail(PBP_EINVAL, "frames < 0");
    if (r.frames == 0) return PBP_OK;
    int rc;
    // every slot at once: a later growth (cudaFree) would stall the device
    for (int i = 0; i < kSlots; ++i)
        if ((rc = size_slot(ctx, ctx->slot[i], r.kind, r.frames))) return rc;
    // the slot's queue/scratch may still be in use by a launch on another stream
    PBP_CUDA(cudaStreamWaitEvent(st, s.done, 0));
    PBP_CUDA(cudaMemsetAsync(s.ctl.p, 0, 4 * sizeof(unsigned long long), st));
    pbp::DecodeArgs a{};
    a.n = ctx->n;
    a.m = ctx->m;
    a.kind = r.kind;
    a.max_iter = r.max_iter;
    a.alpha = r.alpha;
    a.frozen_bits = ctx->frozen_bits.p;
    a.frozen_rows = ctx->frozen_rows.p;
    a.llr = r.llr;
    a.llr64 = r.llr64;
    a.alpha64 = r.alpha64;
    a.frames = r.frames;
    a.u_bits = r.u_bits;
    a.iters = r.iters;
    a.pe = r.pe;
    a.stop = r.stop;
    a.nev = r.nev;
    a.events = r.events;
    a.ev_cap = r.ev_cap;
    a.ev_xhat = r.ev_xhat;
    a.truth_u = r.truth;
    a.counters = r.counters;
    a.cnt_batch = r.cnt_batch;
    a.list_len = s.ctl.p + 2;

    // the warp kernel is fp32 only; fp64 decodes run the generic kernel on double
    const int fk = fast_kernel(ctx->m);
    const bool fast = !r.llr64 && !r.force_generic && !ctx->force_generic && fk != 0;
    if (fast) {
        a.list = r.list ? r.list : s.list.p;
        if (r.list_len) a.list_len = r.list_len;
        a.frame_base = r.frame_base;
        a.queue = s.ctl.p + 0;
        a.list_mode = 0;
        const int per_sm = warp_occupancy(ctx, r.kind);
        long long grid = std::min<long long>((long long)per_sm * ctx->sm_count, r.frames);
        if (const char* gc = getenv("PBP_GRID_CAP")) grid = std::max(1ll, std::min(grid, atoll(gc)));  // experiments
        cudaError_t e;
        if (fk == 1) {
            a.r0s = s.r0s.p;
            e = pbp::launch_warp(a, (int)grid, st);
        } else {
            a.scratch = s.scratch.p;
            a.scratch_stride = pbp::cta_scratch_floats(ctx->m);
            e = pbp::launch_cta(a, (int)grid, st);
        }
        if (e != cudaSuccess) return cuda_fail(e, fk == 1 ? "bp_warp_kernel launch" : "bp_cta_kernel launch");
        ctx->last_launches += 1;
        if (r.list) {  // the caller runs the generic pass over the shared list
            PBP_CUDA(cudaEventRecord(s.done, st));
            return PBP_OK;
        }
        // frames the fast kernel re-routed (|LLR| beyond the clamp-free bound)
        a.list_mode = 1;
    } else {
        a.list = nullptr;
        a.list_mode = 0;
    }
    a.queue = s.ctl.p + 1;
    // generic kernel: bounded grid, per-CTA scratch (elements of the decode precision)
    const int esz = r.llr64 ? 2 : 1;  // in floats
    const long long stride = pbp::generic_scratch_elems(ctx->n, ctx->m);
    const long long grid = generic_grid(ctx, r.frames, fast, esz);
    if (!pbp::generic_in_smem(ctx->n, ctx->m, r.llr64 != nullptr)) {
        if ((rc = s.scratch.ensure((size_t)(grid * stride * esz)))) return rc;
        a.scratch = s.scratch.p;
        a.scratch_stride = stride;
    }
    cudaError_t e = pbp::launch_generic(a, (int)grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "bp_generic_kernel launch");
    ctx->last_launches += 1;
    if (ctx->n_launch_sets < (int)ctx->rerouted.cap) {
        PBP_CUDA(cudaMemcpyAsync(ctx->rerouted.p + ctx->n_launch_sets, s.ctl.p + 2, sizeof(unsigned long long),
                                 cudaMemcpyDeviceToDevice, st));
        ctx->n_launch_sets += 1;
    }
    PBP_CUDA(cudaEventRecord(s.done, st));
    return PBP_OK;
}

// The generic kernel over a re-route list (frame indices relative to r.llr
// and r's output arrays).
int run_generic_list(pbp_ctx* ctx, const DecodeReq& r, DecodeSlot& s, cudaStream_t st, long long listed) {
    int rc;
    if ((rc = s.ctl.ensure(4))) return rc;
    PBP_CUDA(cudaStreamWaitEvent(st, s.done, 0));
    PBP_CUDA(cudaMemsetAsync(s.ctl.p, 0, 4 * sizeof(unsigned long long), st));
    pbp::DecodeArgs a{};
    a.n = ctx->n;
    a.m = ctx->m;
    a.kind = r.kind;
    a.max_iter = r.max_iter;
    a.alpha = r.alpha;
    a.frozen_bits = ctx->frozen_bits.p;
    a.frozen_rows = ctx->frozen_rows.p;
    a.llr = r.llr;
    a.frames = r.frames;
    a.u_bits = r.u_bits;
    a.iters = r.iters;
    a.pe = r.pe;
    a.stop = r.stop;
    a.nev = r.nev;
    a.events = r.events;
    a.ev_cap = r.ev_cap;
    a.ev_xhat = r.ev_xhat;
    a.truth_u = r.truth;
    a.counters = r.counters;
    a.list = r.list;
    a.list_len = r.list_len;
    a.list_mode = 1;
    a.queue = s.ctl.p + 1;
    const long long stride = pbp::generic_scratch_elems(ctx->n, ctx->m);
    const long long grid = generic_grid(ctx, std::max<long long>(1, listed), false);
    if (!pbp::generic_in_smem(ctx->n, ctx->m, false)) {
        if ((rc = s.scratch.ensure((size_t)(grid * stride)))) return rc;
        a.scratch = s.scratch.p;
        a.scratch_stride = stride;
    }
    cudaError_t e = pbp::launch_generic(a, (int)grid, st);
    if (e != cudaSuccess) return cuda_fail(e, "bp_generic_kernel launch");
    ctx->last_launches += 1;
    PBP_CUDA(cudaEventRecord(s.done, st));
    return PBP_OK;
}

// trials per seeding piece: 2.5 KB of state each (80 MiB per piece)
constexpr long long kGenPiece = 32768;

// generation into the given buffers on st, with the slot's seed scratch (the
// caller orders st after the slot's previous use)
int run_generate(pbp_ctx* ctx, DecodeSlot& sl, uint64_t seed, long long first, long long count, double ebn0,
                 int noiseless, float* llr, double* llr64, uint32_t* u, cudaStream_t st) {
    if (count < 0) return fail(PBP_EINVAL, "count < 0");
    double sigma2 = 0.0;
    int rc = pbp_noise_variance(ebn0, (double)ctx->k / ctx->n, &sigma2);
    if (rc) return rc;
    if (count == 0) return PBP_OK;
    pbp::GenArgs g{};
    g.n = ctx->n;
    g.k = ctx->k;
    g.seed = seed;
    g.first = first;
    g.count = count;
    g.sigma = std::sqrt(sigma2);
    g.scale = 2.0 / sigma2;
    g.noiseless = noiseless;
    g.info_rows = ctx->info_rows.p;
    g.llr = llr;
    g.llr64 = llr64;
    const long long piece = std::min(count, kGenPiece);
    rc = sl.gen_mt.ensure((size_t)pbp::channel_seed_words(piece));
    if (rc) return rc;
    g.mt0 = sl.gen_mt.p;
    const int nw = (ctx->n + 31) / 32;
    for (long long done = 0; done < count; done += piece) {
        const long long c = std::min(piece, count - done);
        g.first = first + done;
        g.count = c;
        g.llr = llr ? llr + done * ctx->n : nullptr;
        g.llr64 = llr64 ? llr64 + done * ctx->n : nullptr;
        g.u_out = u ? u + done * nw : nullptr;
        const long long grid = std::min<long long>((c + 3) / 4, (long long)ctx->sm_count * 8);
        cudaError_t e = pbp::launch_channel(g, (int)std::max<long long>(grid, 1), st);
        if (e != cudaSuccess) return cuda_fail(e, "channel_gen_kernel launch");
    }
    return PBP_OK;
}

cudaStream_t pick(pbp_ctx* ctx, void* s) { return s ? (cudaStream_t)s : ctx->stream; }

}  // namespace

// error text for the C ABI's other translation units (pbp_multi.cpp)
__attribute__((visibility("hidden"))) int pbp_set_error(int status, const char* msg) { return fail(status, msg); }

extern "C" {

const char* pbp_last_error(void) { return g_err.c_str(); }
int pbp_version(void) { return PBP_VERSION; }

int pbp_device_count(void) {
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) return 0;
    return c;
}

int pbp_ctx_create(int device, pbp_ctx** out) {
    if (!out) return fail(PBP_EINVAL, "pbp_ctx_create: out is null");
    *out = nullptr;
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
        return fail(PBP_ENODEV, "no CUDA device available (libpbp has no CPU fallback)");
    if (device < 0 || device >= count) return fail(PBP_EINVAL, "pbp_ctx_create: bad device index");
    PBP_CUDA(cudaSetDevice(device));
    auto* ctx = new pbp_ctx;
    ctx->device = device;
    cudaDeviceGetAttribute(&ctx->sm_count, cudaDevAttrMultiProcessorCount, device);
    cudaError_t e = cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking);
    for (int i = 1; i < kSlots && e == cudaSuccess; ++i)
        e = cudaStreamCreateWithFlags(&ctx->slot[i].stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        for (int i = 1; i < kSlots; ++i)
            if (ctx->slot[i].stream) cudaStreamDestroy(ctx->slot[i].stream);
        if (ctx->stream) cudaStreamDestroy(ctx->stream);
        delete ctx;
        return cuda_fail(e, "cudaStreamCreate");
    }
    ctx->slot[0].stream = ctx->stream;
    for (int i = 0; i < kSlots && e == cudaSuccess; ++i)
        e = cudaEventCreateWithFlags(&ctx->slot[i].done, cudaEventDisableTiming);
    if (e != cudaSuccess) {
        pbp_ctx_destroy(ctx);
        return cuda_fail(e, "cudaEventCreate");
    }
    *out = ctx;
    return PBP_OK;
}

int pbp_ctx_destroy(pbp_ctx* ctx) {
    if (!ctx) return PBP_OK;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    ctx->frozen_bits.release();
    ctx->frozen_rows.release();
    ctx->info_rows.release();
    for (int i = 0; i < kSlots; ++i) {
        if (i > 0 && ctx->slot[i].stream) {
            cudaStreamSynchronize(ctx->slot[i].stream);
            cudaStreamDestroy(ctx->slot[i].stream);
        }
        if (ctx->slot[i].done) cudaEventDestroy(ctx->slot[i].done);
        ctx->slot[i].ctl.release();
        ctx->slot[i].list.release();
        ctx->slot[i].scratch.release();
        ctx->slot[i].r0s.release();
        ctx->slot[i].gen_llr.release();
        ctx->slot[i].gen_llr64.release();
        ctx->slot[i].gen_truth.release();
        ctx->slot[i].gen_mt.release();
    }
    ctx->rerouted.release();
    ctx->blist.release();
    ctx->bctl.release();
    ctx->llr64.release();
    ctx->counters.release();
    ctx->llr.release();
    ctx->ubits.release();
    ctx->iters.release();
    ctx->nev.release();
    ctx->events.release();
    ctx->evx.release();
    ctx->pe.release();
    ctx->stop.release();
    cudaStreamDestroy(ctx->stream);
    delete ctx;
    return PBP_OK;
}

void* pbp_ctx_stream(pbp_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int pbp_ctx_synchronize(pbp_ctx* ctx) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    for (int i = 0; i < kSlots; ++i) PBP_CUDA(cudaStreamSynchronize(ctx->slot[i].stream));
    return PBP_OK;
}

int pbp_kernel_info(int32_t n, int decoder, int32_t* smem_bytes, int32_t* warps_per_sm) {
    if (!is_pow2(n)) return fail(PBP_EINVAL, "pbp_kernel_info: n must be a power of two");
    const int m = log2i(n);
    if (decoder < 0 || decoder > 2) return fail(PBP_EINVAL, "unknown decoder kind");
    if (pbp::warp_kernel_supported(m)) {
        if (smem_bytes) *smem_bytes = (int32_t)pbp::warp_smem_bytes(m, decoder);
        if (warps_per_sm) *warps_per_sm = pbp::warp_blocks_per_sm(m, decoder) * pbp::warp_kernel_warps(m);
    } else if (pbp::cta_pair_on(m, decoder)) {  // half a frame per CTA (2-CTA clusters), one CTA per SM
        if (smem_bytes) *smem_bytes = (int32_t)pbp::cta_pair_smem_bytes(m);
        if (warps_per_sm) *warps_per_sm = pbp_device_count() > 0 ? pbp::cta_pair_warps_per_sm(m) : 0;
    } else if (pbp::cta_kernel_supported(m)) {  // CTA per frame: shared bytes per CTA, resident warps
        if (smem_bytes) *smem_bytes = (int32_t)pbp::cta_smem_bytes(m);
        if (warps_per_sm) *warps_per_sm = pbp::cta_blocks_per_sm(m, decoder) * pbp::cta_warps(m);
    } else {
        if (smem_bytes) *smem_bytes = 0;
        if (warps_per_sm) *warps_per_sm = 0;
    }
    return PBP_OK;
}

int pbp_ctx_force_generic(pbp_ctx* ctx, int on) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    ctx->force_generic = on ? 1 : 0;
    return PBP_OK;
}

int pbp_kernel_path(int32_t n) { return is_pow2(n) ? fast_kernel(log2i(n)) : 0; }

int pbp_kernel_cluster(int32_t n, int decoder) {
    if (!is_pow2(n) || !fast_kernel(log2i(n))) return 0;
    return pbp::cta_pair_on(log2i(n), decoder) ? 2 : 1;
}

int pbp_last_launch_info(pbp_ctx* ctx, int32_t* launches, int64_t* rerouted) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (launches) *launches = ctx->last_launches;
    if (rerouted) {
        *rerouted = 0;
        if (ctx->rerouted_host >= 0) {
            *rerouted = ctx->rerouted_host;
        } else if (ctx->n_launch_sets > 0) {
            std::vector<unsigned long long> v(ctx->n_launch_sets);
            for (int i = 0; i < kSlots; ++i) PBP_CUDA(cudaStreamSynchronize(ctx->slot[i].stream));
            PBP_CUDA(cudaMemcpy(v.data(), ctx->rerouted.p, v.size() * sizeof(v[0]), cudaMemcpyDeviceToHost));
            for (unsigned long long x : v) *rerouted += (int64_t)x;
        }
    }
    return PBP_OK;
}

// ---- host-side code helpers ------------------------------------------------

int pbp_construct(int32_t n, int32_t k, double design_z, uint8_t* frozen_out) {
    // PolarCode::construct (src/polar_code.cpp:53-66) and bhattacharyya_profile (:27-43)
    if (!is_pow2(n)) return fail(PBP_EINVAL, "construct: n must be a power of two");
    if (k < 1 || k > n) return fail(PBP_EINVAL, "construct: k must satisfy 1 <= k <= n");
    if (!(design_z > 0.0 && design_z < 1.0))
        return fail(PBP_EINVAL, "bhattacharyya_profile: design_z must be in (0,1)");
    if (!frozen_out) return fail(PBP_EINVAL, "construct: null output");
    std::vector<double> z(n, design_z);
    for (int half = n / 2; half >= 1; half /= 2)
        for (int i = 0; i < n; ++i) {
            if (i & half) continue;
            const double zi = z[i];
            z[i] = 2.0 * zi - zi * zi;  // degraded child keeps the lower index
            z[i + half] = zi * zi;
        }
    std::vector<int> order(n);
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&z](int a, int b) { return z[a] > z[b]; });
    std::memset(frozen_out, 0, n);
    for (int i = 0; i < n - k; ++i) frozen_out[order[i]] = 1;
    return PBP_OK;
}

int pbp_polar_transform(uint8_t* v, int32_t n) {
    if (n <= 0 || !is_pow2(n)) return fail(PBP_EINVAL, "polar_transform: length must be a power of two");
    for (int half = 1; half < n; half <<= 1)
        for (int i = 0; i < n; ++i)
            if (!(i & half)) v[i] ^= v[i + half];
    return PBP_OK;
}

int pbp_encode(const pbp_code* code, const uint8_t* info, uint8_t* u_out, uint8_t* x_out) {
    int rc = check_code(code);
    if (rc) return rc;
    int next = 0;
    for (int i = 0; i < code->n; ++i) u_out[i] = code->frozen[i] ? 0 : (info[next++] ? 1 : 0);
    std::memcpy(x_out, u_out, code->n);
    return pbp_polar_transform(x_out, code->n);
}

int pbp_noise_variance(double ebn0_db, double rate, double* out) {
    // noise_variance (src/channel.cpp:9-15)
    if (!(rate > 0.0 && rate <= 1.0)) return fail(PBP_EINVAL, "noise_variance: rate must be in (0,1]");
    if (!std::isfinite(ebn0_db)) return fail(PBP_EINVAL, "noise_variance: ebn0_db must be finite");
    *out = 1.0 / (2.0 * rate * std::pow(10.0, ebn0_db / 10.0));
    return PBP_OK;
}

// ---- decode ------------------------------------------------------------------

int pbp_decode_batch_device(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs_dev,
                            int64_t frames, float alpha, int32_t max_iter, pbp_frame_out* out_dev,
                            void* stream) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    DecodeReq r;
    r.kind = decoder;
    r.llr = llrs_dev;
    r.frames = frames;
    r.alpha = alpha;
    r.max_iter = max_iter;
    if (out_dev) {
        r.u_bits = out_dev->u_hat_bits;
        r.iters = out_dev->iterations;
        r.pe = reinterpret_cast<long long*>(out_dev->pe);
        r.stop = out_dev->stop;
        r.nev = out_dev->n_events;
    }
    if ((rc = begin_call(ctx, 1))) return rc;
    return run_decode(ctx, r, next_slot(ctx), pick(ctx, stream));
}

int pbp_decode_batch(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs,
                     int64_t frames, float alpha, int32_t max_iter, pbp_frame_out* out) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (decoder < 0 || decoder > 2) return fail(PBP_EINVAL, "unknown decoder kind");
    if (frames < 0) return fail(PBP_EINVAL, "frames < 0");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    const int n = ctx->n, nw = (n + 31) / 32;
    if ((rc = ctx->llr.ensure((size_t)frames * n)) || (rc = ctx->ubits.ensure((size_t)frames * nw)) ||
        (rc = ctx->iters.ensure(frames)) || (rc = ctx->pe.ensure(frames)) ||
        (rc = ctx->stop.ensure(frames)) || (rc = ctx->nev.ensure(frames)))
        return rc;
    // Chunks round-robin over the slots' streams: the host->device copy of one
    // chunk overlaps the decode of the others (and a decode's tail overlaps
    // the next chunk's launch).
    // Chunk sizes grow by 1.3x from 16 MB of LLRs (4096 frames at n = 1024)
    // up to 512 MB and shrink again towards the end, so the last kernel's tail
    // is short. The copies run back to back on the copy engine, so chunk c's
    // data arrives when the copies of chunks 1..c are done; the decoder never
    // waits while each chunk is at most (decode time / copy time - 1) of all
    // chunks before it: with PCIe only ~1.3x faster than the n = 1024 csfg
    // decode, doubling chunks starved the decoder for ~6 ms per 700k frames
    // (tools/e2e_probe.py: 75.0 vs 67.8 ms device at 3 dB). Sized in bytes:
    // at n = 16384 one 16384-frame call is 1 GB, which as a single chunk left
    // its whole upload exposed.
    const long long fscale = std::max(1, n / 1024);
    const long long kChunkMin = std::max(64ll, 16384 / fscale), kEdge = std::max(16ll, 4096 / fscale),
                    kCap = std::max(256ll, (1ll << 17) / fscale);
    std::vector<long long> bounds{0};
    if (frames >= 2 * kChunkMin) {
        std::vector<long long> head, tail;
        long long rem = frames, sz = kEdge;
        while (rem > 0) {
            const long long a = std::min(sz, rem);
            head.push_back(a);
            rem -= a;
            if (rem <= 0) break;
            const long long b = std::min(sz, rem);
            tail.push_back(b);
            rem -= b;
            sz = std::min(sz * 13 / 10, kCap);
        }
        for (long long v : head) bounds.push_back(bounds.back() + v);
        for (auto it = tail.rbegin(); it != tail.rend(); ++it) bounds.push_back(bounds.back() + *it);
    } else {
        bounds.push_back(frames);
    }
    const int nchunks = (int)bounds.size() - 1;
    long long per = 0;
    for (int c = 0; c < nchunks; ++c) per = std::max(per, bounds[c + 1] - bounds[c]);
    if ((rc = begin_call(ctx, nchunks))) return rc;
    for (int i = 0; i < std::min(nchunks, kSlots); ++i)
        if ((rc = size_slot(ctx, ctx->slot[i], decoder, per))) return rc;
    // frames re-routed by any chunk's fast kernel: one batch-wide list, decoded
    // by a single generic pass once the pipeline has drained (rare; no generic
    // launch between the chunks, whose CTAs would stall the other streams)
    const bool fast = !ctx->force_generic && fast_kernel(ctx->m) != 0;
    if (fast) {
        if ((rc = ctx->blist.ensure(std::max<long long>(frames, 1))) || (rc = ctx->bctl.ensure(2))) return rc;
        PBP_CUDA(cudaMemsetAsync(ctx->bctl.p, 0, 2 * sizeof(unsigned long long), ctx->stream));
        PBP_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    for (int c = 0; c < nchunks; ++c) {
        const long long off = bounds[c];
        const long long cnt = bounds[c + 1] - off;
        if (cnt <= 0) continue;
        DecodeSlot& sl = ctx->slot[c % kSlots];
        cudaStream_t st = sl.stream;
        PBP_CUDA(cudaMemcpyAsync(ctx->llr.p + off * n, llrs + off * n, (size_t)cnt * n * 4, cudaMemcpyHostToDevice, st));
        DecodeReq r;
        r.kind = decoder;
        r.llr = ctx->llr.p + off * n;
        r.frames = cnt;
        r.alpha = alpha;
        r.max_iter = max_iter;
        r.u_bits = ctx->ubits.p + off * nw;
        r.iters = ctx->iters.p + off;
        r.pe = ctx->pe.p + off;
        r.stop = ctx->stop.p + off;
        r.nev = ctx->nev.p + off;
        if (fast) {
            r.list = ctx->blist.p;
            r.list_len = ctx->bctl.p;
            r.frame_base = off;
        }
        if ((rc = run_decode(ctx, r, sl, st))) return rc;
        if (out) {
            if (out->u_hat_bits)
                PBP_CUDA(cudaMemcpyAsync(out->u_hat_bits + off * nw, r.u_bits, (size_t)cnt * nw * 4,
                                         cudaMemcpyDeviceToHost, st));
            if (out->iterations)
                PBP_CUDA(cudaMemcpyAsync(out->iterations + off, r.iters, (size_t)cnt * 4, cudaMemcpyDeviceToHost, st));
            if (out->pe) PBP_CUDA(cudaMemcpyAsync(out->pe + off, r.pe, (size_t)cnt * 8, cudaMemcpyDeviceToHost, st));
            if (out->stop) PBP_CUDA(cudaMemcpyAsync(out->stop + off, r.stop, (size_t)cnt, cudaMemcpyDeviceToHost, st));
            if (out->n_events)
                PBP_CUDA(cudaMemcpyAsync(out->n_events + off, r.nev, (size_t)cnt * 4, cudaMemcpyDeviceToHost, st));
        }
    }
    for (int i = 0; i < kSlots; ++i) PBP_CUDA(cudaStreamSynchronize(ctx->slot[i].stream));
    if (!fast) return PBP_OK;
    unsigned long long listed = 0;
    PBP_CUDA(cudaMemcpy(&listed, ctx->bctl.p, sizeof(listed), cudaMemcpyDeviceToHost));
    ctx->rerouted_host = (long long)listed;
    if (listed == 0) return PBP_OK;
    DecodeReq g;
    g.kind = decoder;
    g.llr = ctx->llr.p;
    g.frames = frames;
    g.alpha = alpha;
    g.max_iter = max_iter;
    g.u_bits = ctx->ubits.p;
    g.iters = ctx->iters.p;
    g.pe = ctx->pe.p;
    g.stop = ctx->stop.p;
    g.nev = ctx->nev.p;
    g.list = ctx->blist.p;
    g.list_len = ctx->bctl.p;
    cudaStream_t st = ctx->stream;
    if ((rc = run_generic_list(ctx, g, ctx->slot[0], st, (long long)listed))) return rc;
    if (out) {  // results again, now with the re-routed frames
        if (out->u_hat_bits)
            PBP_CUDA(cudaMemcpyAsync(out->u_hat_bits, g.u_bits, (size_t)frames * nw * 4, cudaMemcpyDeviceToHost, st));
        if (out->iterations)
            PBP_CUDA(cudaMemcpyAsync(out->iterations, g.iters, (size_t)frames * 4, cudaMemcpyDeviceToHost, st));
        if (out->pe) PBP_CUDA(cudaMemcpyAsync(out->pe, g.pe, (size_t)frames * 8, cudaMemcpyDeviceToHost, st));
        if (out->stop) PBP_CUDA(cudaMemcpyAsync(out->stop, g.stop, (size_t)frames, cudaMemcpyDeviceToHost, st));
        if (out->n_events)
            PBP_CUDA(cudaMemcpyAsync(out->n_events, g.nev, (size_t)frames * 4, cudaMemcpyDeviceToHost, st));
    }
    PBP_CUDA(cudaStreamSynchronize(st));
    return PBP_OK;
}

}  // extern "C"

namespace {
// decode_csfg(..., events) for one frame; fp32 (llrs) or fp64 (llrs64)
int decode_trace_impl(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs, const double* llrs64,
                      double alpha, int32_t max_iter, uint8_t* u_hat, int32_t* iterations, int64_t* pe,
                      int32_t* stop, int32_t* n_events, int32_t* events, int32_t events_cap,
                      uint32_t* events_xhat) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    const int n = ctx->n, nw = (n + 31) / 32;
    const int cap = std::max(events_cap, 1);
    if ((rc = ctx->llr.ensure(n)) || (rc = ctx->ubits.ensure(nw)) || (rc = ctx->iters.ensure(1)) ||
        (rc = ctx->pe.ensure(1)) || (rc = ctx->stop.ensure(1)) || (rc = ctx->nev.ensure(1)) ||
        (rc = ctx->events.ensure((size_t)cap * 5)))
        return rc;
    cudaStream_t st = ctx->stream;
    DecodeReq r;
    if (events_xhat) {
        if ((rc = ctx->evx.ensure((size_t)cap * nw))) return rc;
        PBP_CUDA(cudaMemsetAsync(ctx->evx.p, 0, (size_t)cap * nw * 4, st));
        r.ev_xhat = ctx->evx.p;
    }
    if (llrs64) {
        if ((rc = ctx->llr64.ensure(n))) return rc;
        PBP_CUDA(cudaMemcpyAsync(ctx->llr64.p, llrs64, (size_t)n * 8, cudaMemcpyHostToDevice, st));
        r.llr64 = ctx->llr64.p;
        r.alpha64 = alpha;
    } else {
        PBP_CUDA(cudaMemcpyAsync(ctx->llr.p, llrs, (size_t)n * 4, cudaMemcpyHostToDevice, st));
        r.llr = ctx->llr.p;
        r.alpha = (float)alpha;
    }
    r.kind = decoder;
    r.frames = 1;
    r.max_iter = max_iter;
    r.u_bits = ctx->ubits.p;
    r.iters = ctx->iters.p;
    r.pe = ctx->pe.p;
    r.stop = ctx->stop.p;
    r.nev = ctx->nev.p;
    r.events = ctx->events.p;
    r.ev_cap = cap;
    if ((rc = begin_call(ctx, 1))) return rc;
    if ((rc = run_decode(ctx, r, ctx->slot[0], st))) return rc;
    std::vector<uint32_t> bits(nw);
    int it = 0, sp8 = 0, ne = 0;
    long long act = 0;
    uint8_t s8 = 0;
    PBP_CUDA(cudaMemcpyAsync(bits.data(), ctx->ubits.p, nw * 4, cudaMemcpyDeviceToHost, st));
    PBP_CUDA(cudaMemcpyAsync(&it, ctx->iters.p, 4, cudaMemcpyDeviceToHost, st));
    PBP_CUDA(cudaMemcpyAsync(&act, ctx->pe.p, 8, cudaMemcpyDeviceToHost, st));
    PBP_CUDA(cudaMemcpyAsync(&s8, ctx->stop.p, 1, cudaMemcpyDeviceToHost, st));
    PBP_CUDA(cudaMemcpyAsync(&ne, ctx->nev.p, 4, cudaMemcpyDeviceToHost, st));
    std::vector<int> ev((size_t)cap * 5);
    PBP_CUDA(cudaMemcpyAsync(ev.data(), ctx->events.p, ev.size() * 4, cudaMemcpyDeviceToHost, st));
    if (events_xhat && events_cap > 0)
        PBP_CUDA(cudaMemcpyAsync(events_xhat, ctx->evx.p, (size_t)events_cap * nw * 4, cudaMemcpyDeviceToHost, st));
    PBP_CUDA(cudaStreamSynchronize(st));
    sp8 = s8;
    if (u_hat)
        for (int r2 = 0; r2 < n; ++r2) u_hat[r2] = (bits[r2 >> 5] >> (r2 & 31)) & 1u;
    if (iterations) *iterations = it;
    if (pe) *pe = act;
    if (stop) *stop = sp8;
    if (n_events) *n_events = ne;
    if (events && events_cap > 0)
        std::memcpy(events, ev.data(), (size_t)std::min(ne, events_cap) * 5 * 4);
    return PBP_OK;
}
}  // namespace

extern "C" {

int pbp_decode_trace(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs, float alpha,
                     int32_t max_iter, uint8_t* u_hat, int32_t* iterations, int64_t* pe, int32_t* stop,
                     int32_t* n_events, int32_t* events, int32_t events_cap) {
    return decode_trace_impl(ctx, code, decoder, llrs, nullptr, alpha, max_iter, u_hat, iterations, pe, stop,
                             n_events, events, events_cap, nullptr);
}

int pbp_decode_trace_x(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs, float alpha,
                       int32_t max_iter, uint8_t* u_hat, int32_t* iterations, int64_t* pe, int32_t* stop,
                       int32_t* n_events, int32_t* events, int32_t events_cap, uint32_t* events_xhat) {
    return decode_trace_impl(ctx, code, decoder, llrs, nullptr, alpha, max_iter, u_hat, iterations, pe, stop,
                             n_events, events, events_cap, events_xhat);
}

int pbp_decode_trace_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs, double alpha,
                         int32_t max_iter, uint8_t* u_hat, int32_t* iterations, int64_t* pe, int32_t* stop,
                         int32_t* n_events, int32_t* events, int32_t events_cap) {
    if (!llrs) return fail(PBP_EINVAL, "null llrs");
    return decode_trace_impl(ctx, code, decoder, nullptr, llrs, alpha, max_iter, u_hat, iterations, pe, stop,
                             n_events, events, events_cap, nullptr);
}

int pbp_decode_trace_f64_x(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs, double alpha,
                           int32_t max_iter, uint8_t* u_hat, int32_t* iterations, int64_t* pe, int32_t* stop,
                           int32_t* n_events, int32_t* events, int32_t events_cap, uint32_t* events_xhat) {
    if (!llrs) return fail(PBP_EINVAL, "null llrs");
    return decode_trace_impl(ctx, code, decoder, nullptr, llrs, alpha, max_iter, u_hat, iterations, pe, stop,
                             n_events, events, events_cap, events_xhat);
}

int pbp_decode_batch_f64_device(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs_dev,
                                int64_t frames, double alpha, int32_t max_iter, pbp_frame_out* out_dev,
                                void* stream) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    DecodeReq r;
    r.kind = decoder;
    r.llr64 = llrs_dev;
    r.alpha64 = alpha;
    r.frames = frames;
    r.max_iter = max_iter;
    if (out_dev) {
        r.u_bits = out_dev->u_hat_bits;
        r.iters = out_dev->iterations;
        r.pe = reinterpret_cast<long long*>(out_dev->pe);
        r.stop = out_dev->stop;
        r.nev = out_dev->n_events;
    }
    if ((rc = begin_call(ctx, 1))) return rc;
    return run_decode(ctx, r, next_slot(ctx), pick(ctx, stream));
}

int pbp_decode_batch_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, const double* llrs, int64_t frames,
                         double alpha, int32_t max_iter, pbp_frame_out* out) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (frames < 0) return fail(PBP_EINVAL, "frames < 0");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    const int n = ctx->n, nw = (n + 31) / 32;
    if ((rc = ctx->llr64.ensure((size_t)frames * n)) || (rc = ctx->ubits.ensure((size_t)frames * nw)) ||
        (rc = ctx->iters.ensure(frames)) || (rc = ctx->pe.ensure(frames)) ||
        (rc = ctx->stop.ensure(frames)) || (rc = ctx->nev.ensure(frames)))
        return rc;
    cudaStream_t st = ctx->stream;
    if (frames > 0)
        PBP_CUDA(cudaMemcpyAsync(ctx->llr64.p, llrs, (size_t)frames * n * 8, cudaMemcpyHostToDevice, st));
    DecodeReq r;
    r.kind = decoder;
    r.llr64 = ctx->llr64.p;
    r.alpha64 = alpha;
    r.frames = frames;
    r.max_iter = max_iter;
    r.u_bits = ctx->ubits.p;
    r.iters = ctx->iters.p;
    r.pe = ctx->pe.p;
    r.stop = ctx->stop.p;
    r.nev = ctx->nev.p;
    if ((rc = begin_call(ctx, 1))) return rc;
    if ((rc = run_decode(ctx, r, ctx->slot[0], st))) return rc;
    if (out && frames > 0) {
        if (out->u_hat_bits)
            PBP_CUDA(cudaMemcpyAsync(out->u_hat_bits, r.u_bits, (size_t)frames * nw * 4, cudaMemcpyDeviceToHost, st));
        if (out->iterations)
            PBP_CUDA(cudaMemcpyAsync(out->iterations, r.iters, (size_t)frames * 4, cudaMemcpyDeviceToHost, st));
        if (out->pe) PBP_CUDA(cudaMemcpyAsync(out->pe, r.pe, (size_t)frames * 8, cudaMemcpyDeviceToHost, st));
        if (out->stop) PBP_CUDA(cudaMemcpyAsync(out->stop, r.stop, (size_t)frames, cudaMemcpyDeviceToHost, st));
        if (out->n_events)
            PBP_CUDA(cudaMemcpyAsync(out->n_events, r.nev, (size_t)frames * 4, cudaMemcpyDeviceToHost, st));
    }
    PBP_CUDA(cudaStreamSynchronize(st));
    return PBP_OK;
}

// ---- channel -----------------------------------------------------------------

int pbp_generate_device(pbp_ctx* ctx, const pbp_code* code, uint64_t seed, int64_t first_trial,
                        int64_t count, double ebn0_db, int noiseless, float* llr_dev, double* llr64_dev,
                        uint32_t* u_dev, void* stream) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    DecodeSlot& sl = next_slot(ctx);
    cudaStream_t st = pick(ctx, stream);
    PBP_CUDA(cudaStreamWaitEvent(st, sl.done, 0));  // the slot's seed scratch
    rc = run_generate(ctx, sl, seed, first_trial, count, ebn0_db, noiseless, llr_dev, llr64_dev, u_dev, st);
    if (rc) return rc;
    PBP_CUDA(cudaEventRecord(sl.done, st));
    return PBP_OK;
}

int pbp_generate(pbp_ctx* ctx, const pbp_code* code, uint64_t seed, int64_t first_trial, int64_t count,
                 double ebn0_db, int noiseless, float* llr, double* llr64, uint32_t* u_bits) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (count < 0) return fail(PBP_EINVAL, "count < 0");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    const int n = ctx->n, nw = (n + 31) / 32;
    float* d_llr = nullptr;
    double* d_llr64 = nullptr;
    uint32_t* d_u = nullptr;
    PBP_CUDA(cudaMalloc(&d_llr, std::max<size_t>(1, (size_t)count * n * 4)));
    if (llr64) PBP_CUDA(cudaMalloc(&d_llr64, std::max<size_t>(1, (size_t)count * n * 8)));
    if (u_bits) PBP_CUDA(cudaMalloc(&d_u, std::max<size_t>(1, (size_t)count * nw * 4)));
    DecodeSlot& sl = next_slot(ctx);
    PBP_CUDA(cudaStreamWaitEvent(ctx->stream, sl.done, 0));
    rc = run_generate(ctx, sl, seed, first_trial, count, ebn0_db, noiseless, d_llr, d_llr64, d_u, ctx->stream);
    if (!rc) {
        cudaError_t e = cudaEventRecord(sl.done, ctx->stream);
        if (e != cudaSuccess) rc = cuda_fail(e, "pbp_generate");
    }
    if (!rc && count > 0) {
        cudaStream_t st = ctx->stream;
        if (llr) cudaMemcpyAsync(llr, d_llr, (size_t)count * n * 4, cudaMemcpyDeviceToHost, st);
        if (llr64) cudaMemcpyAsync(llr64, d_llr64, (size_t)count * n * 8, cudaMemcpyDeviceToHost, st);
        if (u_bits) cudaMemcpyAsync(u_bits, d_u, (size_t)count * nw * 4, cudaMemcpyDeviceToHost, st);
        cudaError_t e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) rc = cuda_fail(e, "pbp_generate");
    }
    cudaFree(d_llr);
    if (d_llr64) cudaFree(d_llr64);
    if (d_u) cudaFree(d_u);
    return rc;
}

// ---- Monte-Carlo counters ------------------------------------------------------

int pbp_decode_count_device(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs_dev,
                            const uint32_t* u_dev, int64_t frames, float alpha, int32_t max_iter,
                            int64_t* counters_dev, void* stream) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    // the kernels read truth_u whenever counters are requested
    if (!counters_dev || !u_dev) return fail(PBP_EINVAL, "pbp_decode_count_device: null counters or u");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    DecodeReq r;
    r.kind = decoder;
    r.llr = llrs_dev;
    r.frames = frames;
    r.alpha = alpha;
    r.max_iter = max_iter;
    r.truth = u_dev;
    r.counters = reinterpret_cast<unsigned long long*>(counters_dev);
    if ((rc = begin_call(ctx, 1))) return rc;
    return run_decode(ctx, r, next_slot(ctx), pick(ctx, stream));
}

int pbp_decode_count_batches_device(pbp_ctx* ctx, const pbp_code* code, int decoder, const float* llrs_dev,
                                    const uint32_t* u_dev, int64_t frames, int64_t batch, float alpha,
                                    int32_t max_iter, int64_t* counters_dev, void* stream) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (!counters_dev || !u_dev) return fail(PBP_EINVAL, "pbp_decode_count_batches_device: null counters or u");
    if (batch < 1 || batch > 0x7fffffff) return fail(PBP_EINVAL, "pbp_decode_count_batches_device: batch out of range");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    DecodeReq r;
    r.kind = decoder;
    r.llr = llrs_dev;
    r.frames = frames;
    r.alpha = alpha;
    r.max_iter = max_iter;
    r.truth = u_dev;
    r.counters = reinterpret_cast<unsigned long long*>(counters_dev);
    r.cnt_batch = (int)batch;
    if ((rc = begin_call(ctx, 1))) return rc;
    return run_decode(ctx, r, next_slot(ctx), pick(ctx, stream));
}

// run_point's trial loop on the device: fp32 LLRs (the fast path) or, with
// f64, the reference's double LLRs decoded in double.
static int simulate_point_impl(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                               int64_t first_trial, int64_t frames, double ebn0_db, int noiseless, double alpha,
                               bool f64, int32_t max_iter, int64_t* counters_dev, void* stream,
                               int batch = 0) {
    if (!ctx) return fail(PBP_EINVAL, "null context");
    if (frames < 0) return fail(PBP_EINVAL, "frames < 0");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc = upload_code(ctx, code);
    if (rc) return rc;
    const int n = ctx->n, nw = (n + 31) / 32;
    // chunk so the staging stays bounded (512 MiB of fp32 LLRs: a config's 10^5-frame
    // point at n = 1024 is one chunk, so one decode tail per point)
    long long chunk = std::max<long long>(1, std::min<long long>(frames, (1ll << 27) / n));
    if (batch > 0 && chunk < frames) chunk = std::max<long long>(batch, chunk / batch * batch);  // whole batches
    // this call's slot: its generation staging and launch resources (an
    // asynchronous call may overlap other calls on other streams)
    DecodeSlot& sl = next_slot(ctx);
    if ((rc = sl.gen_llr.ensure((size_t)chunk * n)) || (rc = sl.gen_truth.ensure((size_t)chunk * nw))) return rc;
    if (f64 && (rc = sl.gen_llr64.ensure((size_t)chunk * n))) return rc;
    cudaStream_t st = pick(ctx, stream);
    if ((rc = begin_call(ctx, (int)((frames + chunk - 1) / chunk)))) return rc;
    for (long long done = 0; done < frames; done += chunk) {
        const long long c = std::min(chunk, frames - done);
        PBP_CUDA(cudaStreamWaitEvent(st, sl.done, 0));  // the slot's previous decode read the staging
        if ((rc = run_generate(ctx, sl, seed, first_trial + done, c, ebn0_db, noiseless, sl.gen_llr.p,
                               f64 ? sl.gen_llr64.p : nullptr, sl.gen_truth.p, st)))
            return rc;
        DecodeReq r;
        r.kind = decoder;
        if (f64) {
            r.llr64 = sl.gen_llr64.p;
            r.alpha64 = alpha;
        } else {
            r.llr = sl.gen_llr.p;
            r.alpha = (float)alpha;
        }
        r.frames = c;
        r.max_iter = max_iter;
        r.truth = sl.gen_truth.p;
        r.counters = reinterpret_cast<unsigned long long*>(counters_dev) +
                     (batch > 0 ? (done / batch) * pbp::kNumCounters : 0);
        r.cnt_batch = batch;
        if ((rc = run_decode(ctx, r, sl, st))) return rc;
    }
    return PBP_OK;
}

int pbp_simulate_point_device(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed,
                              int64_t first_trial, int64_t frames, double ebn0_db, int noiseless,
                              float alpha, int32_t max_iter, int64_t* counters_dev, void* stream) {
    return simulate_point_impl(ctx, code, decoder, seed, first_trial, frames, ebn0_db, noiseless, alpha, false,
                               max_iter, counters_dev, stream);
}

static int simulate_point_host(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed, int64_t first_trial,
                               int64_t frames, double ebn0_db, int noiseless, double alpha, bool f64,
                               int32_t max_iter, pbp_counters* out) {
    if (!ctx || !out) return fail(PBP_EINVAL, "null argument");
    PBP_CUDA(cudaSetDevice(ctx->device));
    int rc;
    if ((rc = ctx->counters.ensure(pbp::kNumCounters))) return rc;
    PBP_CUDA(cudaMemsetAsync(ctx->counters.p, 0, pbp::kNumCounters * 8, ctx->stream));
    rc = simulate_point_impl(ctx, code, decoder, seed, first_trial, frames, ebn0_db, noiseless, alpha, f64,
                             max_iter, reinterpret_cast<int64_t*>(ctx->counters.p), ctx->stream);
    if (rc) return rc;
    unsigned long long c[pbp::kNumCounters];
    PBP_CUDA(cudaMemcpyAsync(c, ctx->counters.p, sizeof(c), cudaMemcpyDeviceToHost, ctx->stream));
    PBP_CUDA(cudaStreamSynchronize(ctx->stream));
    out->frames = (int64_t)c[pbp::kCntFrames];
    out->bit_errors = (int64_t)c[pbp::kCntBitErr];
    out->frame_errors = (int64_t)c[pbp::kCntFrameErr];
    out->sum_iters = (int64_t)c[pbp::kCntIters];
    out->sum_iters_sq = (int64_t)c[pbp::kCntItersSq];
    out->sum_pe = (int64_t)c[pbp::kCntPe];
    out->sum_events = (int64_t)c[pbp::kCntEvents];
    for (int i = 0; i < 3; ++i) out->stop_hist[i] = (int64_t)c[pbp::kCntStop0 + i];
    return PBP_OK;
}

int pbp_simulate_point(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed, int64_t first_trial,
                       int64_t frames, double ebn0_db, int noiseless, float alpha, int32_t max_iter,
                       pbp_counters* out) {
    return simulate_point_host(ctx, code, decoder, seed, first_trial, frames, ebn0_db, noiseless, alpha, false,
                               max_iter, out);
}

int pbp_simulate_point_f64(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed, int64_t first_trial,
                           int64_t frames, double ebn0_db, int noiseless, double alpha, int32_t max_iter,
                           pbp_counters* out) {
    return simulate_point_host(ctx, code, decoder, seed, first_trial, frames, ebn0_db, noiseless, alpha, true,
                               max_iter, out);
}

int pbp_simulate_batches(pbp_ctx* ctx, const pbp_code* code, int decoder, uint64_t seed, int64_t first_trial,
                         int64_t frames, int32_t batch, double ebn0_db, int noiseless, double alpha,
                         int32_t max_iter, int fp64, int64_t* counters_out) {
    if (!ctx || !counters_out) return fail(PBP_EINVAL, "null argument");
    if (batch < 1) return fail(PBP_EINVAL, "pbp_simulate_batches: batch < 1");
    if (frames < 0) return fail(PBP_EINVAL, "frames < 0");
    if (decoder < 0 || decoder > 2) return fail(PBP_EINVAL, "unknown decoder kind");
    PBP_CUDA(cudaSetDevice(ctx->device));
    const long long nb = (frames + batch - 1) / batch;
    int rc;
    if ((rc = ctx->counters.ensure((size_t)std::max<long long>(nb, 1) * pbp::kNumCounters))) return rc;
    PBP_CUDA(cudaMemsetAsync(ctx->counters.p, 0, (size_t)nb * pbp::kNumCounters * 8, ctx->stream));
    rc = simulate_point_impl(ctx, code, decoder, seed, first_trial, frames, ebn0_db, noiseless, alpha, fp64 != 0,
                             max_iter, reinterpret_cast<int64_t*>(ctx->counters.p), ctx->stream, batch);
    if (rc) return rc;
    PBP_CUDA(cudaMemcpyAsync(counters_out, ctx->counters.p, (size_t)nb * pbp::kNumCounters * 8,
                             cudaMemcpyDeviceToHost, ctx->stream));
    PBP_CUDA(cudaStreamSynchronize(ctx->stream));
    return PBP_OK;
}

}  // extern "C"
