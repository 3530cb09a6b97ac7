// Multi-GPU Monte-Carlo sweep of one process (include/pbp.h
// pbp_simulate_sweep_multi): one host thread and one pbp_ctx per device, each
// generating and decoding its contiguous trial range of every Eb/N0 point
// (the reference splits trials over worker threads,
// src/sim_harness.cpp:144-161), then ONE in-place ncclAllReduce(int64, sum)
// of the npoints x 10 counters over NVLink / NVSwitch. The counters are
// integer sums, so the result is the single-GPU / CPU aggregate exactly.
//
// NCCL is resolved with dlopen("libnccl.so.2") at first use, so libpbp.so has
// no link-time NCCL dependency (a process that already loaded torch's NCCL
// shares that copy: same soname).
#include <dlfcn.h>
#include <nccl.h>

#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "pbp.h"

namespace {

struct Nccl {
    decltype(&ncclCommInitAll) comm_init_all = nullptr;
    decltype(&ncclAllReduce) all_reduce = nullptr;
    decltype(&ncclCommDestroy) comm_destroy = nullptr;
    decltype(&ncclGetErrorString) error_string = nullptr;
    std::string err;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        // an NCCL the process already loaded (torch's) first, then PBP_NCCL_LIB, then
        // the loader's search path. A copy loaded here owns the soname libnccl.so.2
        // for the rest of the process: a later `import torch` would bind to it, so
        // the Python wrapper imports torch before the first call.
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
        if (!h) {
            const char* env = std::getenv("PBP_NCCL_LIB");
            if (env && *env) h = dlopen(env, RTLD_NOW | RTLD_LOCAL);
        }
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_LOCAL);
        if (!h) {
            const char* e = dlerror();
            n.err = std::string("libnccl.so.2 not loadable: ") + (e ? e : "?");
            return;
        }
        n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(dlsym(h, "ncclCommInitAll"));
        n.all_reduce = reinterpret_cast<decltype(n.all_reduce)>(dlsym(h, "ncclAllReduce"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(dlsym(h, "ncclGetErrorString"));
        if (!n.comm_init_all || !n.all_reduce || !n.comm_destroy || !n.error_string)
            n.err = "libnccl.so.2 lacks ncclCommInitAll/ncclAllReduce/ncclCommDestroy";
    });
    return n;
}

}  // namespace

// pbp_capi.cu: records pbp_last_error() for this thread, returns status
int pbp_set_error(int status, const char* msg);

namespace {
int set_error(int status, const std::string& msg) { return pbp_set_error(status, msg.c_str()); }
}  // namespace

extern "C" int pbp_simulate_sweep_multi(const int* devices, int ndev, const pbp_code* code, int decoder,
                                        uint64_t seed, int64_t frames_per_point, const double* ebn0_db,
                                        int npoints, int noiseless, float alpha, int32_t max_iter,
                                        pbp_counters* out) {
    if (!devices || ndev < 1 || !code || !ebn0_db || !out || npoints < 1)
        return set_error(PBP_EINVAL, "pbp_simulate_sweep_multi: bad arguments");
    if (frames_per_point < 0) return set_error(PBP_EINVAL, "frames < 0");
    if (pbp_device_count() < 1) return set_error(PBP_ENODEV, "no CUDA device");
    const Nccl& nc = nccl();
    if (!nc.err.empty()) return set_error(PBP_ERUNTIME, nc.err);

    constexpr int kC = 10;  // counters per point (pbp_counters field order)
    const size_t nval = (size_t)npoints * kC;
    std::vector<ncclComm_t> comms(ndev);
    ncclResult_t nr = nc.comm_init_all(comms.data(), ndev, devices);
    if (nr != ncclSuccess) return set_error(PBP_ERUNTIME, std::string("ncclCommInitAll: ") + nc.error_string(nr));

    std::vector<int> status(ndev, PBP_OK);
    std::vector<std::string> errs(ndev);
    std::vector<std::vector<long long>> host(ndev, std::vector<long long>(nval, 0));
    std::vector<pbp_ctx*> ctxs(ndev, nullptr);
    std::vector<long long*> dcs(ndev, nullptr);
    auto run_all = [&](auto&& fn) {
        std::vector<std::thread> pool;
        for (int g = 0; g < ndev; ++g) pool.emplace_back(fn, g);
        for (auto& t : pool) t.join();
    };
    auto cleanup = [&]() {
        for (int g = 0; g < ndev; ++g) {
            if (dcs[g]) {
                cudaSetDevice(devices[g]);
                cudaFree(dcs[g]);
            }
            if (ctxs[g]) pbp_ctx_destroy(ctxs[g]);
            nc.comm_destroy(comms[g]);
        }
    };
    // phase 1: every device's context and counters, so no rank can fail after the
    // others entered the collective
    run_all([&](int g) {
        int rc = pbp_ctx_create(devices[g], &ctxs[g]);
        if (rc) {
            status[g] = rc;
            errs[g] = pbp_last_error();
            return;
        }
        if (cudaSetDevice(devices[g]) != cudaSuccess || cudaMalloc(&dcs[g], nval * sizeof(long long)) != cudaSuccess ||
            cudaMemsetAsync(dcs[g], 0, nval * sizeof(long long), (cudaStream_t)pbp_ctx_stream(ctxs[g])) !=
                cudaSuccess) {
            status[g] = PBP_ENOMEM;
            errs[g] = "device counters";
        }
    });
    for (int g = 0; g < ndev; ++g)
        if (status[g]) {
            cleanup();
            return set_error(status[g], "device " + std::to_string(devices[g]) + ": " + errs[g]);
        }
    // phase 2: this device's contiguous share of every point's trials, then the
    // all-reduce (every rank joins it; a rank whose decode failed contributes what
    // it has and the call reports the failure)
    run_all([&](int g) {
        pbp_ctx* ctx = ctxs[g];
        cudaStream_t st = (cudaStream_t)pbp_ctx_stream(ctx);
        const long long first = frames_per_point * g / ndev;
        const long long count = frames_per_point * (g + 1) / ndev - first;
        for (int p = 0; p < npoints && !status[g]; ++p) {
            const int rc = pbp_simulate_point_device(ctx, code, decoder, seed, first, count, ebn0_db[p], noiseless,
                                                     alpha, max_iter, reinterpret_cast<int64_t*>(dcs[g]) + (size_t)p * kC,
                                                     nullptr);
            if (rc) {
                status[g] = rc;
                errs[g] = pbp_last_error();
            }
        }
        cudaSetDevice(devices[g]);
        const ncclResult_t r = nc.all_reduce(dcs[g], dcs[g], nval, ncclInt64, ncclSum, comms[g], st);
        if (r != ncclSuccess && !status[g]) {
            status[g] = PBP_ERUNTIME;
            errs[g] = std::string("ncclAllReduce: ") + nc.error_string(r);
        }
        if ((cudaMemcpyAsync(host[g].data(), dcs[g], nval * sizeof(long long), cudaMemcpyDeviceToHost, st) !=
                 cudaSuccess ||
             cudaStreamSynchronize(st) != cudaSuccess) &&
            !status[g]) {
            status[g] = PBP_ECUDA;
            errs[g] = "counter copy";
        }
    });
    cleanup();
    for (int g = 0; g < ndev; ++g)
        if (status[g]) return set_error(status[g], "device " + std::to_string(devices[g]) + ": " + errs[g]);
    for (int g = 1; g < ndev; ++g)
        if (host[g] != host[0]) return set_error(PBP_ERUNTIME, "ncclAllReduce: ranks disagree");
    for (int p = 0; p < npoints; ++p) {
        const long long* c = host[0].data() + (size_t)p * kC;
        pbp_counters& o = out[p];
        o.frames = c[0];
        o.bit_errors = c[1];
        o.frame_errors = c[2];
        o.sum_iters = c[3];
        o.sum_iters_sq = c[4];
        o.sum_pe = c[5];
        o.sum_events = c[6];
        for (int i = 0; i < 3; ++i) o.stop_hist[i] = c[7 + i];
    }
    return PBP_OK;
}
