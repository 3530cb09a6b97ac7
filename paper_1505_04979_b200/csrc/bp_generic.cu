// Generic CTA-per-frame BP decoder (any n = 2^m, m <= 24).
//
// A literal restatement of the reference schedule on the device: one CTA
// owns one frame, runs stage_pass (src/bp_core.cpp:58-80) stage by stage
// with a barrier in between, the csfg candidate check/commit right after
// each stage (src/csfg_freeze.cpp:107-119) and the G-check after each
// sweep (src/bp_core.cpp:95-102, src/csfg_freeze.cpp:120-135). Every clamp,
// sgn(0)=+1 and std::min tie rule of pe_update (src/bp_core.cpp:13-32) is
// kept, so it is exact for any finite or non-finite LLR. Messages L(1..m)
// and the current R level live in shared memory when they fit (n <= 4096 in
// fp32: 13 x 16 KB, one 512-thread CTA per SM), else in a per-CTA global
// scratch region; R(0) is read from the LLR input (clamped) and L(0) is only
// kept as the G-check's hard-decision bits, formed at stage 0.
//
// Roles: (1) the decode path for n outside the warp-resident kernel's range
// (n < 128 and n >= 2048), (2) the path for frames the fast kernel
// re-routes (|LLR| > kClampFreeBound or non-finite), (3) instantiated on
// double, the reference as shipped (its fp64 operation order; DecodeArgs
// llr64 / alpha64).
#include "pbp_common.cuh"

namespace pbp {

namespace {

// The reference's arithmetic (src/bp_core.cpp:13-32) for T = float (its
// fp32 operation order) and T = double (as shipped); every product and sum
// rounded on its own (-fmad=false and explicit _rn intrinsics).
template <typename T> struct RealOps;
template <> struct RealOps<float> {
    static __device__ __forceinline__ float mul(float a, float b) { return __fmul_rn(a, b); }
    static __device__ __forceinline__ float add(float a, float b) { return __fadd_rn(a, b); }
    static __device__ __forceinline__ float abs(float a) { return fabsf(a); }
    static constexpr float cap = kCap;
};
template <> struct RealOps<double> {
    static __device__ __forceinline__ double mul(double a, double b) { return __dmul_rn(a, b); }
    static __device__ __forceinline__ double add(double a, double b) { return __dadd_rn(a, b); }
    static __device__ __forceinline__ double abs(double a) { return fabs(a); }
    static constexpr double cap = 1e30;  // LLR_CAP (include/polarbp/bp_core.hpp:21)
};
template <typename T> __device__ __forceinline__ T ref_sgn(T v) { return v < T(0) ? T(-1) : T(1); }
template <typename T> __device__ __forceinline__ T ref_min(T a, T b) { return b < a ? b : a; }
template <typename T> __device__ __forceinline__ T ref_clamp(T v) {
    const T c = RealOps<T>::cap;
    return v < -c ? -c : (c < v ? c : v);
}
// alpha * sgn(a) * sgn(b) * min(|a|, |b|), left to right, no contraction
template <typename T> __device__ __forceinline__ T ref_f(T alpha, T a, T b) {
    using O = RealOps<T>;
    return O::mul(O::mul(O::mul(alpha, ref_sgn(a)), ref_sgn(b)), ref_min(O::abs(a), O::abs(b)));
}

// Polar transform (polar_code.cpp:13-20) of `nbits` bits held in words[0..ceil(nbits/32))
// of shared memory, by one warp (no CTA barrier between the butterfly levels).
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

}  // namespace

// shared words ahead of the message arrays: decided_u, two scratch bit
// vectors, stage-0 hard decisions, freeze_stage bytes
__host__ __device__ inline size_t generic_bits_bytes(int n) {
    const size_t nw = (size_t)(n + 31) / 32;
    return (4 * nw * 4 + (size_t)n + 15) / 16 * 16;
}

template <int BLOCK, typename T, bool SM>
__global__ void __launch_bounds__(BLOCK) bp_generic_kernel(DecodeArgs a) {
    using O = RealOps<T>;
    const T cap = O::cap;
    extern __shared__ __align__(16) uint32_t smem[];
    const int n = a.n, m = a.m;
    const int nw_all = (n + 31) >> 5;
    uint32_t* dec_u = smem;               // decided_u bits
    uint32_t* wb0 = smem + nw_all;        // scratch words
    uint32_t* wb1 = smem + 2 * nw_all;    // scratch words
    uint32_t* xh = smem + 3 * nw_all;     // x_hat = (R(0) + L(0) < 0) of the last sweep
    uint8_t* fst = reinterpret_cast<uint8_t*>(smem + 4 * nw_all);  // freeze_stage per row

    __shared__ long long s_frame;
    __shared__ int s_frontier, s_nev, s_conv;
    __shared__ unsigned long long s_act;
    __shared__ int s_bit_err;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    // L(s) for s = 1..m at L + (s-1) n, then the current R level
    T* L = SM ? reinterpret_cast<T*>(reinterpret_cast<unsigned char*>(smem) + generic_bits_bytes(n))
              : reinterpret_cast<T*>(a.scratch) + (long long)blockIdx.x * a.scratch_stride;
    T* R = L + (size_t)m * n;
    const T alpha = sizeof(T) == 8 ? T(a.alpha64) : T(a.alpha);
    const bool csfg = a.kind == 2;

    for (;;) {
        if (tid == 0) {
            long long f = -1;
            const unsigned long long idx = atomicAdd(a.queue, 1ull);
            if (a.list_mode) {
                if (idx < *a.list_len) f = a.list[idx];
            } else if ((long long)idx < a.frames) {
                f = (long long)idx;
            }
            s_frame = f;
            s_frontier = 0;
            s_nev = 0;
            s_act = 0;
            s_bit_err = 0;
        }
        __syncthreads();
        const long long frame = s_frame;
        if (frame < 0) break;

        // init_state (src/bp_core.cpp:43-56)
        // R(0) = clamp(LLR), read where needed (src/bp_core.cpp:47)
        const float* llr32 = a.llr + frame * (long long)n;
        const double* llr64 = sizeof(T) == 8 ? a.llr64 + frame * (long long)n : nullptr;
        auto R0 = [&](int r) -> T { return ref_clamp(sizeof(T) == 8 ? T(llr64[r]) : T(llr32[r])); };
        for (int r = tid; r < n; r += BLOCK) {
            for (int s = 1; s < m; ++s) L[(size_t)(s - 1) * n + r] = T(0);
            if (m > 0) L[(size_t)(m - 1) * n + r] = a.frozen_rows[r] ? cap : T(0);
            R[r] = T(0);
            fst[r] = kNotFrozen;
        }
        for (int q = tid; q < nw_all; q += BLOCK) dec_u[q] = 0u;
        __syncthreads();

        unsigned long long act = 0;
        int iters = (a.kind == 0) ? a.max_iter : 0;
        int stop = 0;
        bool converged = false;

        for (int t = 1; t <= a.max_iter; ++t) {
            if (csfg && (s_frontier >= n || converged)) break;
            if (csfg) iters = t;
            for (int s = 0; s < m; ++s) {
                if (csfg && s_frontier >= n) break;
                // ---- stage_pass (src/bp_core.cpp:58-80) ----
                const int ld = m - 1 - s;
                const int d = 1 << ld;
                T* Ls = (s > 0) ? L + (size_t)(s - 1) * n : nullptr;
                const T* Ls1 = L + (size_t)s * n;
                if (s == 0 && n < 64)
                    for (int q = tid; q < nw_all; q += BLOCK) xh[q] = 0u;
                if (s == 0) __syncthreads();
                // two PEs per thread per step, all eight loads issued before the math
                // (the messages sit in L2: one PE at a time leaves the loads' latency bare)
                for (int p0 = 0; p0 < n / 2; p0 += 2 * BLOCK) {
                    int r[2];
                    bool on[2];
                    T lt[2], lb[2], rt[2], rb[2];
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int p = p0 + h * BLOCK + tid;
                        r[h] = ((p >> ld) << (ld + 1)) | (p & (d - 1));
                        // is_pe_active (csfg_freeze.cpp:95-97); stage 0 is always active
                        on[h] = p < n / 2 && !(csfg && (int)fst[r[h]] < s);
                        if (on[h]) {
                            lt[h] = Ls1[r[h]];
                            lb[h] = Ls1[r[h] + d];
                            rt[h] = (s == 0) ? R0(r[h]) : R[r[h]];
                            rb[h] = (s == 0) ? R0(r[h] + d) : R[r[h] + d];
                        }
                    }
#pragma unroll
                    for (int h = 0; h < 2; ++h) {
                        const int p = p0 + h * BLOCK + tid;
                        bool xt = false, xbot = false;
                        if (on[h]) {
                            const T cross = ref_f(alpha, lt[h], rt[h]);
                            const T sum_bot = O::add(lb[h], rb[h]);
                            const T l_top = ref_clamp(ref_f(alpha, lt[h], sum_bot));
                            const T l_bot = ref_clamp(O::add(lb[h], cross));
                            if (s > 0) {
                                Ls[r[h]] = l_top;
                                Ls[r[h] + d] = l_bot;
                            } else {  // L(0) only feeds the G-check's x_hat (bp_core.cpp:99)
                                xt = O::add(rt[h], l_top) < T(0);
                                xbot = O::add(rb[h], l_bot) < T(0);
                            }
                            R[r[h]] = ref_clamp(ref_f(alpha, rt[h], sum_bot));
                            R[r[h] + d] = ref_clamp(O::add(rb[h], cross));
                            ++act;
                        }
                        if (s == 0) {
                            if (n >= 64) {  // rows r = p and r + n/2: whole warps of consecutive rows
                                const uint32_t wt = __ballot_sync(0xffffffffu, xt);
                                const uint32_t wbt = __ballot_sync(0xffffffffu, xbot);
                                if (lane == 0 && p < n / 2) {
                                    xh[r[h] >> 5] = wt;
                                    xh[(r[h] + d) >> 5] = wbt;
                                }
                            } else if (p < n / 2) {
                                if (xt) atomicOr(&xh[r[h] >> 5], 1u << (r[h] & 31));
                                if (xbot) atomicOr(&xh[(r[h] + d) >> 5], 1u << ((r[h] + d) & 31));
                            }
                        }
                    }
                }
                __syncthreads();
                if (!csfg) continue;

                // ---- candidate_block / check_csfg / apply_freeze
                //      (src/csfg_freeze.cpp:8-39,82-93,116-118) ----
                // x_hat of the block gathered by the CTA, its transform and the
                // frozen-row verdict by one warp, the commit by the CTA
                const int frontier = s_frontier;
                const int sz = n >> (s + 1);
                const int index = frontier / sz;
                const int start = index * sz;
                const int nw = (sz + 31) >> 5;
                for (int i = tid; i < nw * 32; i += BLOCK) {
                    const bool b = (i < sz) && (R[start + i] < T(0));
                    const uint32_t w = __ballot_sync(0xffffffffu, b);
                    if (lane == 0) wb0[i >> 5] = w;
                }
                __syncthreads();
                if (tid < 32) {
                    warp_transform(wb0, sz, lane);
                    bool viol = false;
                    if (sz >= 32) {
                        for (int q = lane; q < nw; q += 32)
                            viol |= (wb0[q] & a.frozen_bits[(start >> 5) + q]) != 0u;
                    } else if (lane == 0) {
                        const uint32_t fz = (a.frozen_bits[start >> 5] >> (start & 31)) & low_mask(sz);
                        viol = (wb0[0] & fz) != 0u;
                    }
                    const bool acc = !__any_sync(0xffffffffu, viol);
                    if (lane == 0) s_conv = acc ? 1 : 0;
                }
                __syncthreads();
                if (s_conv) {
                    for (int i = tid; i < sz; i += BLOCK) {
                        const int r = start + i;
                        L[(size_t)s * n + r] = (R[r] < T(0)) ? -cap : cap;  // L(s+1)
                        if ((int)fst[r] > s) fst[r] = (uint8_t)s;
                        if (a.ev_xhat && s_nev < a.ev_cap && R[r] < T(0))
                            atomicOr(&a.ev_xhat[((size_t)frame * a.ev_cap + s_nev) * nw_all + (r >> 5)], 1u << (r & 31));
                    }
                    if (sz >= 32) {
                        for (int q = tid; q < nw; q += BLOCK) dec_u[(start >> 5) + q] = wb0[q];
                    } else if (tid == 0) {
                        const int off = start & 31;
                        const uint32_t msk = low_mask(sz) << off;
                        dec_u[start >> 5] = (dec_u[start >> 5] & ~msk) | ((wb0[0] << off) & msk);
                    }
                    __syncthreads();  // s_frontier / s_conv read above by every thread
                    if (tid == 0) {
                        if (a.events && s_nev < a.ev_cap) {
                            int* e = a.events + ((size_t)frame * a.ev_cap + s_nev) * 5;
                            e[0] = t;
                            e[1] = s;
                            e[2] = index;
                            e[3] = start;
                            e[4] = sz;
                        }
                        s_nev += 1;
                        s_frontier = start + sz;
                    }
                }
                __syncthreads();
            }

            if (a.kind == 0) continue;
            if (m == 0) {  // no stage ran: L(0) = L(m) (bp_core.cpp:53), x_hat = R(0) + L(0) < 0
                if (tid == 0) xh[0] = O::add(R0(0), a.frozen_rows[0] ? cap : T(0)) < T(0) ? 1u : 0u;
                __syncthreads();
            }
            const int pin = csfg ? s_frontier : 0;
            if (csfg && pin >= n) continue;
            // ---- gmatrix_converged (src/bp_core.cpp:95-102), pinned prefix
            //      for csfg (src/csfg_freeze.cpp:120-135) ----
            for (int i = tid; i < nw_all * 32; i += BLOCK) {
                bool ub = false;
                if (i < n)
                    ub = (i < pin) ? ((dec_u[i >> 5] >> (i & 31)) & 1u)
                                   : (!a.frozen_rows[i] && (m == 0 ? R0(i) : R[i]) < T(0));  // m = 0: R(m) = R(0)
                const uint32_t wu = __ballot_sync(0xffffffffu, ub);
                if (lane == 0) {
                    wb0[i >> 5] = wu;
                    wb1[i >> 5] = xh[i >> 5] & low_mask(n - (i & ~31));
                }
            }
            __syncthreads();
            if (tid < 32) {  // transform and compare by one warp
                warp_transform(wb0, n, lane);
                bool diff = false;
                for (int q = lane; q < nw_all; q += 32) diff |= (wb0[q] != wb1[q]);
                const bool c = !__any_sync(0xffffffffu, diff);
                if (lane == 0) s_conv = c ? 1 : 0;
            }
            __syncthreads();
            const bool conv = s_conv != 0;
            if (a.kind == 1 && conv) {
                iters = t;
                stop = 1;
                break;
            }
            if (csfg) converged = conv;
        }

        // ---- DecodeOutcome (src/bp_core.cpp:106-115, csfg_freeze.cpp:137-151) ----
        const int frontier = s_frontier;
        if (a.kind == 1 && stop == 0) iters = a.max_iter;
        if (csfg) stop = (frontier >= n) ? 2 : (converged ? 1 : 0);
        const int pin = csfg ? (frontier >= n ? n : frontier) : 0;
        int berr = 0;
        for (int i = tid; i < nw_all * 32; i += BLOCK) {
            bool ub = false;
            if (i < n)
                ub = (i < pin) ? ((dec_u[i >> 5] >> (i & 31)) & 1u)
                               : (!a.frozen_rows[i] && (m == 0 ? R0(i) : R[i]) < T(0));
            const uint32_t w = __ballot_sync(0xffffffffu, ub);
            if (lane == 0) {
                if (a.u_bits) a.u_bits[frame * nw_all + (i >> 5)] = w;
                if (a.truth_u)
                    berr += __popc((w ^ a.truth_u[frame * nw_all + (i >> 5)]) &
                                   ~a.frozen_bits[i >> 5]);
            }
        }
        if (berr) atomicAdd(&s_bit_err, berr);
        if (act) atomicAdd(&s_act, act);
        __syncthreads();
        if (tid == 0) {
            const long long pe = (long long)s_act;
            if (a.iters) a.iters[frame] = iters;
            if (a.pe) a.pe[frame] = pe;
            if (a.stop) a.stop[frame] = (uint8_t)stop;
            if (a.nev) a.nev[frame] = s_nev;
            if (a.counters) {
                unsigned long long* cs = counter_set(a, frame);
                atomicAdd(&cs[kCntFrames], 1ull);
                atomicAdd(&cs[kCntBitErr], (unsigned long long)s_bit_err);
                atomicAdd(&cs[kCntFrameErr], s_bit_err > 0 ? 1ull : 0ull);
                atomicAdd(&cs[kCntIters], (unsigned long long)iters);
                atomicAdd(&cs[kCntItersSq], (unsigned long long)iters * iters);
                atomicAdd(&cs[kCntPe], (unsigned long long)pe);
                atomicAdd(&cs[kCntEvents], (unsigned long long)s_nev);
                atomicAdd(&cs[kCntStop0 + stop], 1ull);
            }
        }
        __syncthreads();
    }
}

// Host-side launch helpers (called from pbp_capi.cu)
constexpr int kGenericBlock = 256;     // messages in global scratch
constexpr int kGenericBlockSM = 512;   // messages in shared memory
constexpr size_t kMaxSmem = 227 * 1024;

static size_t smem_state_bytes(int n, int m, size_t esz) {
    return generic_bits_bytes(n) + (size_t)(m + 1) * n * esz;
}

// Messages in shared memory when at least four frames fit per SM: the kernel
// is bound by its per-stage barriers, so frames per SM matter more than the
// memory level (n = 4096 in shared memory, one frame per SM, measured 18 %
// slower than L2-resident scratch with eight frames per SM).
bool generic_in_smem(int n, int m, bool f64) {
    return smem_state_bytes(n, m, f64 ? 8 : 4) <= kMaxSmem / 4;
}

size_t generic_smem_bytes(int n) { return generic_bits_bytes(n); }

// per-CTA message scratch (global variant) in elements of the decode
// precision: L(1..m) and the current R level
long long generic_scratch_elems(int n, int m) {
    long long f = (long long)(m + 1) * n;
    return (f + 63) / 64 * 64;
}

template <int BLOCK, typename T, bool SM>
static cudaError_t launch_t(const DecodeArgs& a, int grid, cudaStream_t stream) {
    const size_t smem = SM ? smem_state_bytes(a.n, a.m, sizeof(T)) : generic_bits_bytes(a.n);
    // always opt in: the kernel's static shared variables come on top of smem
    // (n = 32768 needs exactly 48 KB dynamic)
    cudaError_t e = cudaFuncSetAttribute(bp_generic_kernel<BLOCK, T, SM>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    bp_generic_kernel<BLOCK, T, SM><<<grid, BLOCK, smem, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_generic(const DecodeArgs& a, int grid, cudaStream_t stream) {
    const bool f64 = a.llr64 != nullptr;
    if (generic_in_smem(a.n, a.m, f64))
        return f64 ? launch_t<kGenericBlockSM, double, true>(a, grid, stream)
                   : launch_t<kGenericBlockSM, float, true>(a, grid, stream);
    return f64 ? launch_t<kGenericBlock, double, false>(a, grid, stream)
               : launch_t<kGenericBlock, float, false>(a, grid, stream);
}

}  // namespace pbp
