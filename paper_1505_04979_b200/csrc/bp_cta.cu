// CTA-per-frame BP decoder for n = 2048 .. 16384 (configs 3 and 4).
//
// The reference schedule literally (src/bp_core.cpp:58-86, csfg_freeze.cpp:
// 99-152): every stage's PEs, the PE mask of is_pe_active (inactive PEs are
// skipped, so frozen boundaries keep their saturation without protection),
// the candidate check/commit right after each stage and the pinned G-check
// after each sweep. What changes is where the messages live: T = 512 (1024
// from n = 8192) threads own P = n/T rows each, and for the K = log2 P stages of a pass a thread's rows
// stay fixed, so R(s) is carried in registers from stage to stage and only
// crosses shared memory at the pass boundaries. Each PE then moves 16 bytes of
// messages (L(s+1) in, L(s) out; per-CTA global scratch, L2-resident at
// n = 4096) instead of 32. Arithmetic as in the warp-resident kernel (one
// min.xorsign.abs per min-with-sign, every product and sum rounded on its own,
// r_top = fma(alpha, m, +0)); frames with |LLR| beyond the clamp-free bound or
// non-finite are re-routed to the generic kernel, which keeps every clamp.
#include "pbp_common.cuh"

namespace pbp {
namespace cta {

constexpr unsigned kFull = 0xffffffffu;

// threads per frame: 512 up to n = 4096 (two frames per SM at <= 64
// registers), 1024 beyond (one frame per SM, 32 warps, scratch in HBM)
template <int M>
constexpr int kLogT = M <= 12 ? 9 : 10;

template <int M_>
struct CPlan {
    static constexpr int M = M_;
    static constexpr int N = 1 << M;
    static constexpr int T = 1 << kLogT<M>;
    static constexpr int K = M - kLogT<M>;  // log2 of the rows per thread
    static constexpr int P = 1 << K;
    static constexpr int Q = (M + K - 1) / K;  // passes
    static constexpr int NW = N / 32;
    // pass q: registers j hold row bits [b, b+K); thread bits fill the rest
    static constexpr int base(int q) { return (M - K * (q + 1)) > 0 ? (M - K * (q + 1)) : 0; }
    static constexpr int first(int q) { return q * K; }
    static constexpr int last(int q) { return ((q + 1) * K < M ? (q + 1) * K : M) - 1; }
    static constexpr int pass_of(int s) { return s / K; }
    static constexpr int pad(int row) { return row + (row >> 5); }  // bank spread of the transpose buffer
    static constexpr int NX = N + N / 32;
};

__device__ __forceinline__ float xsmin(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// Polar transform (polar_code.cpp:13-20) of nbits bits in words[] by one warp.
__device__ void warp_transform(uint32_t* words, int nbits, int lane) {
    const int nw = (nbits + 31) >> 5;
    for (int q = lane; q < nw; q += 32) words[q] = word_transform(words[q], nbits);
    __syncwarp();
    for (int h = 1; h < nw; h <<= 1) {
        for (int p = lane; p < nw / 2; p += 32) {
            const int q = ((p / h) * 2 * h) + (p % h);
            words[q] ^= words[q + h];
        }
        __syncwarp();
    }
}

template <int M>
struct CtaSmem {
    using PL = CPlan<M>;
    float Rx[PL::NX];           // R at pass boundaries, row-indexed (padded)
    uint8_t sgn[PL::N];         // sign of R(s+1) per row, for the candidate check
    uint8_t fst[PL::N];         // freeze_stage per row
    uint32_t xh[PL::NW];        // x_hat = (R(0) + L(0) < 0) of the last sweep
    uint32_t dec_u[PL::NW];     // decided_u
    uint32_t wb0[PL::NW];       // block / u_hat words
    uint32_t frz[PL::NW];       // frozen rows
    long long frame;
    unsigned long long act;
    int frontier, nev, conv, accept, bad, bit_err;
};

template <int M, int KIND>
struct Dec {
    using PL = CPlan<M>;
    static constexpr int N = PL::N, P = PL::P, K = PL::K, Q = PL::Q, NW = PL::NW, kT = PL::T;
    static constexpr bool csfg = KIND == 2;

    CtaSmem<M>* sm;
    const DecodeArgs* a;
    float* L;  // L(s) at L + (s-1) N, s = 1..M
    int tid, lane;
    float alpha;
    float R[P];
    long long act;  // this thread's PE activations

    template <int q>
    __device__ __forceinline__ int row(int j) const {
        constexpr int b = PL::base(q);
        return (tid & ((1 << b) - 1)) | (j << b) | ((tid >> b) << (b + K));
    }

    // stage S: PEs (j, j + dj) of this thread's registers; returns false when
    // the csfg frontier covered n (the reference leaves the stage loop)
    template <int S>
    __device__ __forceinline__ bool stage() {
        constexpr int q = PL::pass_of(S);
        constexpr int b = PL::base(q);
        constexpr int g = M - 1 - S;
        constexpr int dj = 1 << (g - b);
        if constexpr (csfg) {
            if (sm->frontier >= N) return false;
        }
        const float* Lin = L + (size_t)S * N;             // L(S+1)
        float* Lout = L + (size_t)(S > 0 ? S - 1 : 0) * N;  // L(S)
        // loads first (all PEs of the stage), then the math
        float lt[P / 2], lb[P / 2];
        bool on[P / 2];
#pragma unroll
        for (int j = 0, k = 0; j < P; ++j) {
            if (j & dj) continue;
            const int rt = row<q>(j);
            on[k] = !csfg || (int)sm->fst[rt] >= S;  // is_pe_active (csfg_freeze.cpp:95-97)
            lt[k] = on[k] ? Lin[rt] : 0.f;
            lb[k] = on[k] ? Lin[rt + (1 << g)] : 0.f;
            ++k;
        }
#pragma unroll
        for (int j = 0, k = 0; j < P; ++j) {
            if (j & dj) continue;
            const int rt = row<q>(j), rb = rt + (1 << g);
            bool xt = false, xb = false;
            if (on[k]) {
                const float r_t = R[j], r_b = R[j + dj];
                const float cross = __fmul_rn(alpha, xsmin(lt[k], r_t));
                const float sum_bot = __fadd_rn(lb[k], r_b);
                const float l_top = __fmul_rn(alpha, xsmin(lt[k], sum_bot));
                const float l_bot = __fadd_rn(lb[k], cross);
                if constexpr (S > 0) {
                    Lout[rt] = l_top;
                    Lout[rb] = l_bot;
                } else {  // L(0) only feeds the G-check's x_hat (bp_core.cpp:99)
                    xt = __fadd_rn(r_t, l_top) < 0.f;
                    xb = __fadd_rn(r_b, l_bot) < 0.f;
                }
                R[j] = __fmaf_rn(alpha, xsmin(r_t, sum_bot), 0.0f);
                R[j + dj] = __fadd_rn(r_b, cross);
                ++act;
            }
            if constexpr (S == 0 && KIND != 0) {
                // pass 0 keeps row bits [0, 9) in the thread index: a warp's
                // lanes hold 32 consecutive rows of every register
                static_assert(PL::base(0) >= 5, "pass 0 layout");
                const uint32_t wt = __ballot_sync(kFull, xt), wb = __ballot_sync(kFull, xb);
                if (lane == 0) {
                    sm->xh[rt >> 5] = wt;
                    sm->xh[rb >> 5] = wb;
                }
            }
            ++k;
        }
        if constexpr (csfg) return check<S>();
        return true;
    }

    // candidate_block / check_csfg / apply_freeze (csfg_freeze.cpp:8-39,
    // 82-93, 116-118) after stage S
    template <int S>
    __device__ __forceinline__ bool check() {
        constexpr int q = PL::pass_of(S);
#pragma unroll
        for (int j = 0; j < P; ++j) sm->sgn[row<q>(j)] = __float_as_int(R[j]) < 0;
        __syncthreads();
        constexpr int g = M - 1 - S;
        constexpr int sz = 1 << g;
        constexpr int nw = (sz + 31) >> 5;
        const int frontier = sm->frontier;
        const int index = frontier >> g;
        const int start = index << g;
        if constexpr (sz > 32) {  // block bits by the CTA, one word per warp step
            for (int i = tid; i < nw * 32; i += PL::T) {
                const uint32_t w = __ballot_sync(kFull, sm->sgn[start + i] != 0);
                if (lane == 0) sm->wb0[i >> 5] = w;
            }
            __syncthreads();
        }
        if (tid < 32) {
            if constexpr (sz <= 32) {
                const uint32_t w = __ballot_sync(kFull, lane < sz && sm->sgn[start + lane] != 0);
                if (lane == 0) sm->wb0[0] = w;
                __syncwarp();
            }
            warp_transform(sm->wb0, sz, lane);
            bool viol = false;
            if constexpr (sz >= 32) {
                for (int w = lane; w < nw; w += 32) viol |= (sm->wb0[w] & sm->frz[(start >> 5) + w]) != 0u;
            } else {
                if (lane == 0) viol = (sm->wb0[0] & (sm->frz[start >> 5] >> (start & 31)) & low_mask(sz)) != 0u;
            }
            const bool acc = !__any_sync(kFull, viol);
            if (lane == 0) sm->accept = acc ? 1 : 0;
        }
        __syncthreads();
        if (!sm->accept) return true;
        // apply_freeze: L(S+1) = +-CAP over the block, freeze_stage, decided_u, event
        float* Lsat = L + (size_t)S * N;
        for (int i = tid; i < sz; i += PL::T) {
            const int r = start + i;
            Lsat[r] = sm->sgn[r] ? -kCap : kCap;
            if ((int)sm->fst[r] > S) sm->fst[r] = (uint8_t)S;
        }
        if constexpr (sz >= 32) {
            for (int w = tid; w < nw; w += PL::T) sm->dec_u[(start >> 5) + w] = sm->wb0[w];
        } else if (tid == 0) {
            const int off = start & 31;
            const uint32_t msk = low_mask(sz) << off;
            sm->dec_u[start >> 5] = (sm->dec_u[start >> 5] & ~msk) | ((sm->wb0[0] << off) & msk);
        }
        __syncthreads();  // every thread read frontier/accept above
        if (tid == 0) {
            if (a->events && sm->nev < a->ev_cap) {
                int* e = a->events + ((long long)sm->frame * a->ev_cap + sm->nev) * 5;
                e[0] = it;
                e[1] = S;
                e[2] = index;
                e[3] = start;
                e[4] = sz;
            }
            sm->nev += 1;
            sm->frontier = start + sz;
        }
        __syncthreads();
        return true;
    }

    int it = 0;

    // pass boundaries move R through shared memory into the next layout
    template <int S>
    __device__ __forceinline__ bool sweep_from() {
        constexpr int q = PL::pass_of(S);
        if constexpr (S == PL::first(q) && q > 0) {
            __syncthreads();
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = sm->Rx[PL::pad(row<q>(j))];
        }
        if (!stage<S>()) return false;
        if constexpr (S == PL::last(q) && q + 1 < Q) {
            __syncthreads();  // the previous boundary's readers are done
#pragma unroll
            for (int j = 0; j < P; ++j) sm->Rx[PL::pad(row<q>(j))] = R[j];
        }
        if constexpr (S + 1 < M) return sweep_from<S + 1>();
        return true;
    }

    // u_hat of the last sweep (frozen rows 0, rows < pin from decided_u) into
    // wb0; R is in the last pass's layout (rows P*tid + j)
    __device__ __forceinline__ void u_words(int pin) {
        for (int w = tid; w < NW; w += PL::T) sm->wb0[w] = 0u;
        __syncthreads();
        if constexpr (P >= 32) {
#pragma unroll
            for (int c = 0; c < P / 32; ++c) {
                uint32_t w = 0u;
#pragma unroll
                for (int i = 0; i < 32; ++i) w |= (uint32_t)(__float_as_int(R[32 * c + i]) < 0) << i;
                const int wi = (P * tid) / 32 + c;
                w &= ~sm->frz[wi];
                const int r0 = 32 * wi;
                if (pin > r0) {
                    const uint32_t pm = pin - r0 >= 32 ? kFull : low_mask(pin - r0);
                    w = (w & ~pm) | (sm->dec_u[wi] & pm);
                }
                sm->wb0[wi] = w;
            }
        } else {
            uint32_t w = 0u;
#pragma unroll
            for (int i = 0; i < P; ++i) w |= (uint32_t)(__float_as_int(R[i]) < 0) << i;
            const int r0 = P * tid, wi = r0 >> 5, sh = r0 & 31;
            const uint32_t m = low_mask(P);
            w &= ~(sm->frz[wi] >> sh) & m;
            if (pin > r0) {
                const uint32_t pm = pin - r0 >= P ? m : low_mask(pin - r0);
                w = (w & ~pm) | ((sm->dec_u[wi] >> sh) & pm);
            }
            atomicOr(&sm->wb0[wi], w << sh);
        }
        __syncthreads();
    }

    // gmatrix_converged (bp_core.cpp:95-102) with the pinned prefix
    // (csfg_freeze.cpp:120-135)
    __device__ __forceinline__ bool gcheck(int pin) {
        u_words(pin);
        if (tid < 32) {
            warp_transform(sm->wb0, N, lane);
            bool diff = false;
            for (int w = lane; w < NW; w += 32) diff |= sm->wb0[w] != sm->xh[w];
            const bool c = !__any_sync(kFull, diff);
            if (lane == 0) sm->conv = c ? 1 : 0;
        }
        __syncthreads();
        return sm->conv != 0;
    }

    __device__ void run(const DecodeArgs& args, CtaSmem<M>* s) {
        a = &args;
        sm = s;
        tid = threadIdx.x;
        lane = tid & 31;
        alpha = args.alpha;
        L = args.scratch + (long long)blockIdx.x * args.scratch_stride;
        for (int w = tid; w < NW; w += PL::T) sm->frz[w] = args.frozen_bits[w];
        for (;;) {
            __syncthreads();
            if (tid == 0) {
                const unsigned long long idx = atomicAdd(args.queue, 1ull);
                sm->frame = (long long)idx < args.frames ? (long long)idx : -1;
                sm->frontier = 0;
                sm->nev = 0;
                sm->act = 0ull;
                sm->bit_err = 0;
            }
            __syncthreads();
            const long long f = sm->frame;
            if (f < 0) break;
            // channel LLRs (R(0), -0 -> +0) in pass 0's layout; frames beyond the
            // clamp-free bound go to the generic kernel
            const float* llr = args.llr + f * (long long)N;
            bool bad = false;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const float v = llr[row<0>(j)];
                bad |= !(fabsf(v) <= kClampFreeBound);
            }
            if (__syncthreads_or(bad)) {
                if (tid == 0) {
                    const unsigned long long slot = atomicAdd(args.list_len, 1ull);
                    args.list[slot] = f + args.frame_base;
                }
                continue;
            }
            // init_state (bp_core.cpp:43-56)
            for (int r = tid; r < N; r += PL::T) {
                for (int l = 1; l < M; ++l) L[(size_t)(l - 1) * N + r] = 0.f;
                L[(size_t)(M - 1) * N + r] = args.frozen_rows[r] ? kCap : 0.f;
                sm->fst[r] = kNotFrozen;
            }
            for (int w = tid; w < NW; w += PL::T) sm->dec_u[w] = 0u;
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = 0.f;
            act = 0;
            __syncthreads();
            int iters = (KIND == 0) ? args.max_iter : 0;
            int stop = 0;
            bool converged = false;
            for (int t = 1; t <= args.max_iter; ++t) {
                if constexpr (csfg) {
                    if (sm->frontier >= N || converged) break;
                    iters = t;
                }
                it = t;
#pragma unroll
                for (int j = 0; j < P; ++j) R[j] = __fadd_rn(llr[row<0>(j)], 0.0f);
                sweep_from<0>();
                __syncthreads();
                if constexpr (KIND == 1) {
                    if (gcheck(0)) {
                        iters = t;
                        stop = 1;
                        break;
                    }
                } else if constexpr (csfg) {
                    const int pin = sm->frontier;
                    if (pin < N) converged = gcheck(pin);
                }
            }
            if constexpr (KIND == 1) {
                if (stop == 0) iters = args.max_iter;
            }
            const int frontier = sm->frontier;
            if constexpr (csfg) stop = (frontier >= N) ? 2 : (converged ? 1 : 0);
            const int pin = csfg ? (frontier >= N ? N : frontier) : 0;
            // DecodeOutcome (bp_core.cpp:106-115, csfg_freeze.cpp:137-151)
            if (csfg && frontier >= N) {
                __syncthreads();
                for (int w = tid; w < NW; w += PL::T) sm->wb0[w] = sm->dec_u[w];
                __syncthreads();
            } else {
                u_words(pin);
            }
            int berr = 0;
            for (int w = tid; w < NW; w += PL::T) {
                const uint32_t uw = sm->wb0[w];
                if (args.u_bits) args.u_bits[f * NW + w] = uw;
                if (args.truth_u) berr += __popc((uw ^ args.truth_u[f * NW + w]) & ~sm->frz[w]);
            }
            berr = __reduce_add_sync(kFull, berr);
            const long long wact = __reduce_add_sync(kFull, (unsigned)act);  // < 2^32 per thread
            if (lane == 0) {
                if (berr) atomicAdd(&sm->bit_err, berr);
                atomicAdd(&sm->act, (unsigned long long)wact);
            }
            __syncthreads();
            if (tid == 0) {
                const long long pe = (long long)sm->act;
                if (args.iters) args.iters[f] = iters;
                if (args.pe) args.pe[f] = pe;
                if (args.stop) args.stop[f] = (uint8_t)stop;
                if (args.nev) args.nev[f] = sm->nev;
                if (args.counters) {
                    atomicAdd(&args.counters[kCntFrames], 1ull);
                    atomicAdd(&args.counters[kCntBitErr], (unsigned long long)sm->bit_err);
                    atomicAdd(&args.counters[kCntFrameErr], sm->bit_err > 0 ? 1ull : 0ull);
                    atomicAdd(&args.counters[kCntIters], (unsigned long long)iters);
                    atomicAdd(&args.counters[kCntItersSq], (unsigned long long)iters * iters);
                    atomicAdd(&args.counters[kCntPe], (unsigned long long)pe);
                    atomicAdd(&args.counters[kCntEvents], (unsigned long long)sm->nev);
                    atomicAdd(&args.counters[kCntStop0 + stop], 1ull);
                }
            }
        }
    }
};

// 64 registers: two 512-thread frames per SM up to n = 4096, one 1024-thread
// frame beyond
template <int M>
constexpr int kMinCtas = M <= 12 ? 2 : 1;

template <int M, int KIND>
__global__ void __launch_bounds__(CPlan<M>::T, kMinCtas<M>) bp_cta_kernel(DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char csm[];
    Dec<M, KIND> dec;
    dec.run(a, reinterpret_cast<CtaSmem<M>*>(csm));
}

template <int M, int KIND>
static cudaError_t launch_t(const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(CtaSmem<M>);
    cudaError_t e = cudaFuncSetAttribute(bp_cta_kernel<M, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    bp_cta_kernel<M, KIND><<<grid, CPlan<M>::T, smem, st>>>(a);
    return cudaGetLastError();
}

template <int M>
static cudaError_t launch_m(const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (a.kind) {
        case 0: return launch_t<M, 0>(a, grid, st);
        case 1: return launch_t<M, 1>(a, grid, st);
        default: return launch_t<M, 2>(a, grid, st);
    }
}

template <int M, int KIND>
static int occ_t() {
    int nb = 0;
    const size_t smem = sizeof(CtaSmem<M>);
    cudaFuncSetAttribute(bp_cta_kernel<M, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bp_cta_kernel<M, KIND>, CPlan<M>::T, smem) != cudaSuccess)
        return 0;
    return nb;
}

template <int M>
static int occ_m(int kind) {
    return kind == 0 ? occ_t<M, 0>() : kind == 1 ? occ_t<M, 1>() : occ_t<M, 2>();
}

}  // namespace cta

int cta_kernel_supported(int m) { return m >= 11 && m <= 14; }

long long cta_scratch_floats(int m) { return (long long)m << m; }  // L(1..m)

cudaError_t launch_cta(const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (a.m) {
        case 11: return cta::launch_m<11>(a, grid, st);
        case 12: return cta::launch_m<12>(a, grid, st);
        case 13: return cta::launch_m<13>(a, grid, st);
        case 14: return cta::launch_m<14>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

int cta_blocks_per_sm(int m, int kind) {
    switch (m) {
        case 11: return cta::occ_m<11>(kind);
        case 12: return cta::occ_m<12>(kind);
        case 13: return cta::occ_m<13>(kind);
        case 14: return cta::occ_m<14>(kind);
    }
    return 0;
}

}  // namespace pbp
