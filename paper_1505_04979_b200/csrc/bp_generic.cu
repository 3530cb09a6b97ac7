// Generic CTA-per-frame BP decoder (any n = 2^m, m <= 24).
//
// A literal restatement of the reference schedule on the device: one CTA
// owns one frame, runs stage_pass (src/bp_core.cpp:58-80) stage by stage
// with a barrier in between, the csfg candidate check/commit right after
// each stage (src/csfg_freeze.cpp:107-119) and the G-check after each
// sweep (src/bp_core.cpp:95-102, src/csfg_freeze.cpp:120-135). Every clamp,
// sgn(0)=+1 and std::min tie rule of pe_update (src/bp_core.cpp:13-32) is
// kept, so it is exact for any finite or non-finite LLR. Messages live in a
// per-CTA global scratch region (L2 resident for the configs), bit-level
// state in shared memory.
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

// Polar transform of `nbits` bits held in words[0..ceil(nbits/32)) of
// shared memory, by the whole CTA (polar_code.cpp:13-20 on packed words).
template <int BLOCK>
__device__ void cta_transform(uint32_t* words, int nbits) {
    const int nw = (nbits + 31) >> 5;
    for (int q = threadIdx.x; q < nw; q += BLOCK) words[q] = word_transform(words[q], nbits);
    __syncthreads();
    for (int h = 1; h < nw; h <<= 1) {
        for (int p = threadIdx.x; p < nw / 2; p += BLOCK) {
            const int q = ((p / h) * 2 * h) + (p % h);
            words[q] ^= words[q + h];
        }
        __syncthreads();
    }
}

}  // namespace

template <int BLOCK, typename T>
__global__ void __launch_bounds__(BLOCK) bp_generic_kernel(DecodeArgs a) {
    using O = RealOps<T>;
    const T cap = O::cap;
    extern __shared__ uint32_t smem[];
    const int n = a.n, m = a.m;
    const int nw_all = (n + 31) >> 5;
    uint32_t* dec_u = smem;               // decided_u bits
    uint32_t* wb0 = smem + nw_all;        // scratch words
    uint32_t* wb1 = smem + 2 * nw_all;    // scratch words
    uint8_t* fst = reinterpret_cast<uint8_t*>(smem + 3 * nw_all);  // freeze_stage per row

    __shared__ long long s_frame;
    __shared__ int s_frontier, s_nev;
    __shared__ unsigned long long s_act;
    __shared__ int s_bit_err;

    const int tid = threadIdx.x;
    const int lane = tid & 31;
    T* L = reinterpret_cast<T*>(a.scratch) + (long long)blockIdx.x * a.scratch_stride;  // (m+1) x n
    T* R0 = L + (size_t)(m + 1) * n;
    T* R = R0 + n;
    const T* Rm = (m == 0) ? R0 : R;
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
        for (int r = tid; r < n; r += BLOCK) {
            const T v = sizeof(T) == 8 ? T(a.llr64[frame * (long long)n + r]) : T(a.llr[frame * (long long)n + r]);
            R0[r] = ref_clamp(v);
            for (int s = 0; s < m; ++s) L[(size_t)s * n + r] = T(0);
            L[(size_t)m * n + r] = a.frozen_rows[r] ? cap : T(0);
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
                const T* Rin = (s == 0) ? R0 : R;
                T* Ls = L + (size_t)s * n;
                const T* Ls1 = L + (size_t)(s + 1) * n;
                for (int p = tid; p < n / 2; p += BLOCK) {
                    const int r = ((p >> ld) << (ld + 1)) | (p & (d - 1));
                    if (csfg && (int)fst[r] < s) continue;  // is_pe_active (csfg_freeze.cpp:95-97)
                    const T lt = Ls1[r], lb = Ls1[r + d], rt = Rin[r], rb = Rin[r + d];
                    const T cross = ref_f(alpha, lt, rt);
                    const T sum_bot = O::add(lb, rb);
                    Ls[r] = ref_clamp(ref_f(alpha, lt, sum_bot));
                    Ls[r + d] = ref_clamp(O::add(lb, cross));
                    R[r] = ref_clamp(ref_f(alpha, rt, sum_bot));
                    R[r + d] = ref_clamp(O::add(rb, cross));
                    ++act;
                }
                __syncthreads();
                if (!csfg) continue;

                // ---- candidate_block / check_csfg / apply_freeze
                //      (src/csfg_freeze.cpp:8-39,82-93,116-118) ----
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
                cta_transform<BLOCK>(wb0, sz);
                int viol = 0;
                if (sz >= 32) {
                    for (int q = tid; q < nw; q += BLOCK)
                        viol |= (wb0[q] & a.frozen_bits[(start >> 5) + q]) != 0u;
                } else if (tid == 0) {
                    const uint32_t fz = (a.frozen_bits[start >> 5] >> (start & 31)) & low_mask(sz);
                    viol = (wb0[0] & fz) != 0u;
                }
                const bool accept = !__syncthreads_or(viol);
                if (accept) {
                    for (int i = tid; i < sz; i += BLOCK) {
                        const int r = start + i;
                        L[(size_t)(s + 1) * n + r] = (R[r] < T(0)) ? -cap : cap;
                        if ((int)fst[r] > s) fst[r] = (uint8_t)s;
                    }
                    if (sz >= 32) {
                        for (int q = tid; q < nw; q += BLOCK) dec_u[(start >> 5) + q] = wb0[q];
                    } else if (tid == 0) {
                        const int off = start & 31;
                        const uint32_t msk = low_mask(sz) << off;
                        dec_u[start >> 5] = (dec_u[start >> 5] & ~msk) | ((wb0[0] << off) & msk);
                    }
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
            const int pin = csfg ? s_frontier : 0;
            if (csfg && pin >= n) continue;
            // ---- gmatrix_converged (src/bp_core.cpp:95-102), pinned prefix
            //      for csfg (src/csfg_freeze.cpp:120-135) ----
            for (int i = tid; i < nw_all * 32; i += BLOCK) {
                bool ub = false, xb = false;
                if (i < n) {
                    ub = (i < pin) ? ((dec_u[i >> 5] >> (i & 31)) & 1u)
                                   : (!a.frozen_rows[i] && Rm[i] < T(0));
                    xb = O::add(R0[i], L[i]) < T(0);
                }
                const uint32_t wu = __ballot_sync(0xffffffffu, ub);
                const uint32_t wx = __ballot_sync(0xffffffffu, xb);
                if (lane == 0) {
                    wb0[i >> 5] = wu;
                    wb1[i >> 5] = wx;
                }
            }
            __syncthreads();
            cta_transform<BLOCK>(wb0, n);
            int diff = 0;
            for (int q = tid; q < nw_all; q += BLOCK) diff |= (wb0[q] != wb1[q]);
            const bool conv = !__syncthreads_or(diff);
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
                               : (!a.frozen_rows[i] && Rm[i] < T(0));
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
                atomicAdd(&a.counters[kCntFrames], 1ull);
                atomicAdd(&a.counters[kCntBitErr], (unsigned long long)s_bit_err);
                atomicAdd(&a.counters[kCntFrameErr], s_bit_err > 0 ? 1ull : 0ull);
                atomicAdd(&a.counters[kCntIters], (unsigned long long)iters);
                atomicAdd(&a.counters[kCntItersSq], (unsigned long long)iters * iters);
                atomicAdd(&a.counters[kCntPe], (unsigned long long)pe);
                atomicAdd(&a.counters[kCntEvents], (unsigned long long)s_nev);
                atomicAdd(&a.counters[kCntStop0 + stop], 1ull);
            }
        }
        __syncthreads();
    }
}

// Host-side launch helpers (called from pbp_capi.cu)
constexpr int kGenericBlock = 256;

size_t generic_smem_bytes(int n) {
    const int nw = (n + 31) / 32;
    return (size_t)3 * nw * 4 + (size_t)n + 16;
}

// per-CTA message scratch in elements of the decode precision (float or
// double); scratch_stride is in those elements
long long generic_scratch_elems(int n, int m) {
    long long f = (long long)(m + 3) * n;
    return (f + 63) / 64 * 64;
}

template <typename T>
static cudaError_t launch_t(const DecodeArgs& a, int grid, cudaStream_t stream) {
    const size_t smem = generic_smem_bytes(a.n);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(bp_generic_kernel<kGenericBlock, T>,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    bp_generic_kernel<kGenericBlock, T><<<grid, kGenericBlock, smem, stream>>>(a);
    return cudaGetLastError();
}

cudaError_t launch_generic(const DecodeArgs& a, int grid, cudaStream_t stream) {
    return a.llr64 ? launch_t<double>(a, grid, stream) : launch_t<float>(a, grid, stream);
}

}  // namespace pbp
