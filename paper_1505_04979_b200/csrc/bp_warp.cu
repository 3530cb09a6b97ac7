// Warp-resident BP decoder for n = 128 .. 1024 (the north-star path).
//
// One warp owns one frame for its whole decode; warps pull frames from a
// global atomic queue (persistent grid), so early-stopping frames never
// idle a CTA. Rows are distributed as P = n/32 rows per lane. The m PE
// stages of one sweep (src/bp_core.cpp:82-86) are grouped into passes of
// K = m-5 consecutive stages; within a pass every butterfly partner of a
// lane's row sits in the same lane's registers, so R (src/bp_core.cpp:58-80)
// never leaves the register file inside a pass:
//   pass q register layout: row(lane, j) = lane_lo | j << b_q | lane_hi << (b_q+K)
//   (b_0 = 5: row = lane + 32 j ; last pass b = 0: row = P*lane + j).
// Between passes R(e) goes through a row-indexed, XOR-swizzled shared array
// X that then holds L(e) in place (the two never live at the same time).
// L(s) of stages inside a pass stays in registers (n <= 512, and n = 1024's
// first pass) or in lane-private float4 shared slots (n = 1024's last pass).
//
// Exactness: the PE is Eq. (1) of
// src/bp_core.cpp:18-32 in fp32 with min.xorsign.abs + mul/add rounded
// separately (no FMA contraction); r_top = fma(alpha, m, +0) never yields
// -0, so R's sign bit equals the reference's (v < 0) decision; clamps are
// elided because frames with |LLR| > kClampFreeBound are re-routed to the
// generic kernel, which keeps them.
//
// The csfg schedule (src/csfg_freeze.cpp:99-152) is followed literally:
// after each stage the candidate block containing the frontier is checked
// on the fresh R(s+1) (sign bits packed per lane, XOR butterfly along the
// block's row bits: in-word for register bits, shfl_xor for lane bits),
// committed, and the PE mask takes effect from the next stage on. Inactive
// PEs are computed anyway (their outputs are never read by an active PE);
// only the saturated boundary L(f+1) of a frozen block must survive, which
// is enforced per storage class (read-side override for register arrays,
// predicated stores for shared slots, re-saturation for X). PE activations
// are counted by the reference rule from per-stage inactive-row counts.
#include "pbp_common.cuh"

namespace pbp {
namespace wk {

constexpr unsigned kFull = 0xffffffffu;

template <int M_>
struct Plan {
    static constexpr int M = M_;
    static constexpr int N = 1 << M;
    static constexpr int P = N / 32;
    static constexpr int K = M - 5;
    static constexpr int Q = (M + K - 1) / K;
    static constexpr int NW = N / 32;
    static constexpr int base_bit(int q) { return (M - K - q * K) > 0 ? (M - K - q * K) : 0; }
    static constexpr int pass_of(int s) { return s / K; }
    static constexpr int first(int q) { return q * K; }
    static constexpr int last(int q) { return ((q + 1) * K < M ? (q + 1) * K : M) - 1; }
    static constexpr bool is_boundary(int s) { return s > 0 && s < M && s % K == 0; }
    static constexpr bool is_local(int s) { return s >= 1 && s < M && s % K != 0; }
    static constexpr int n_local() {
        int c = 0;
        for (int s = 1; s < M; ++s) c += is_local(s) ? 1 : 0;
        return c;
    }
    static constexpr bool SMEM_LAST = P * n_local() > 128;
    static constexpr bool local_smem(int s) { return SMEM_LAST && is_local(s) && pass_of(s) == Q - 1; }
    static constexpr bool local_reg(int s) { return is_local(s) && !local_smem(s); }
    static constexpr int reg_slot(int s) {
        int c = 0;
        for (int x = 1; x < s; ++x) c += local_reg(x) ? 1 : 0;
        return c;
    }
    static constexpr int smem_slot(int s) {
        int c = 0;
        for (int x = 1; x < s; ++x) c += local_smem(x) ? 1 : 0;
        return c;
    }
    static constexpr int n_reg() {
        int c = 0;
        for (int s = 1; s < M; ++s) c += local_reg(s) ? 1 : 0;
        return c;
    }
    static constexpr int n_smem() {
        int c = 0;
        for (int s = 1; s < M; ++s) c += local_smem(s) ? 1 : 0;
        return c;
    }
    static constexpr int NLR = n_reg() > 0 ? n_reg() : 1;
    static constexpr int NLS = n_smem() > 0 ? n_smem() : 1;
};

template <int M>
struct WarpSmem {
    using PL = Plan<M>;
    float R0[PL::N];                       // channel LLRs, row order
    float X[PL::Q - 1][PL::N];             // pass boundaries: R(e) then L(e), swizzled rows
    float4 Ls[PL::NLS][PL::P / 4][32];     // lane-private L slots (last pass, n=1024)
    float4 LM[PL::P / 4][32];              // L(m), lane-private, last-pass layout
    uint32_t dec_u[PL::NW];                // decided_u bits (row order)
    uint32_t sat[PL::NW];                  // x_hat of the latest commit per row
    uint32_t xprot[PL::Q - 1][PL::NW];     // per boundary: blocks frozen at stage e-1
    int inact[32];                         // inactive top rows per stage
    int tmp[32];
    unsigned long long cnt[16];            // per-warp counter accumulators
    uint8_t fst[PL::N];                    // freeze_stage per row
};

__device__ __forceinline__ float xsmin(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

__device__ __forceinline__ int xidx(int row) { return row ^ ((row >> 5) & 31); }

__device__ __forceinline__ uint32_t signbit_u(float v) { return __float_as_uint(v) >> 31; }

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
    const uint32_t masks[5] = {0x0000FFFFu, 0x00FF00FFu, 0x0F0F0F0Fu, 0x33333333u, 0x55555555u};
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int s = 16 >> i;
        const uint32_t y = __shfl_xor_sync(kFull, x, s);
        if ((lane & s) == 0)
            x = (x & masks[i]) | ((y & masks[i]) << s);
        else
            x = (x & ~masks[i]) | ((y >> s) & masks[i]);
    }
    return x;
}

template <int M, int KIND>
struct Dec {
    using PL = Plan<M>;
    static constexpr int N = PL::N, P = PL::P, K = PL::K, Q = PL::Q, NW = PL::NW;

    WarpSmem<M>* sm;
    int lane;
    float alpha;
    const DecodeArgs* a;

    float R[P];
    float Lr[PL::NLR][P];
    uint32_t PM[PL::NLR];   // register arrays: rows whose L must read as +-CAP
    uint32_t SS[PL::NLR];   // ... and their signs
    uint32_t PMW[PL::NLS];  // shared slots: rows whose L must not be overwritten
    uint32_t FZ[Q];         // frozen rows per pass layout
    uint32_t FZW;           // frozen word (row order) of this lane (lane < NW)

    int frontier, nev, it;
    long long act;
    uint32_t xq;            // channel-side decisions, pass-0 layout

    template <int q>
    __device__ __forceinline__ int row_of(int j) const {
        constexpr int b = PL::base_bit(q);
        return (lane & ((1 << b) - 1)) | (j << b) | ((lane >> b) << (b + K));
    }

    // ---- L(S) sources / sinks ----------------------------------------
    template <int T>
    __device__ __forceinline__ void load_L(float (&Lt)[P]) {
        // L(T) as read by stage T-1 (layout of pass_of(T-1))
        constexpr int q = PL::pass_of(T - 1);
        if constexpr (T == M) {
#pragma unroll
            for (int c = 0; c < P / 4; ++c) {
                const float4 v = sm->LM[c][lane];
                Lt[4 * c] = v.x;
                Lt[4 * c + 1] = v.y;
                Lt[4 * c + 2] = v.z;
                Lt[4 * c + 3] = v.w;
            }
        } else if constexpr (PL::is_boundary(T)) {
            constexpr int xs = PL::pass_of(T) - 1;
#pragma unroll
            for (int j = 0; j < P; ++j) Lt[j] = sm->X[xs][xidx(row_of<q>(j))];
        } else if constexpr (PL::local_reg(T)) {
            constexpr int sl = PL::reg_slot(T);
#pragma unroll
            for (int j = 0; j < P; ++j) Lt[j] = Lr[sl][j];
            if (__any_sync(kFull, PM[sl] != 0u)) {
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if ((PM[sl] >> j) & 1u) Lt[j] = ((SS[sl] >> j) & 1u) ? -kCap : kCap;
            }
        } else {
            constexpr int sl = PL::smem_slot(T);
#pragma unroll
            for (int c = 0; c < P / 4; ++c) {
                const float4 v = sm->Ls[sl][c][lane];
                Lt[4 * c] = v.x;
                Lt[4 * c + 1] = v.y;
                Lt[4 * c + 2] = v.z;
                Lt[4 * c + 3] = v.w;
            }
        }
    }

    template <int S>
    __device__ __forceinline__ void store_L(const float (&Lt)[P]) {
        constexpr int q = PL::pass_of(S);
        if constexpr (S == 0) {
            // L(0) is only consumed through x_hat (packed in the PE loop)
        } else if constexpr (PL::is_boundary(S)) {
            constexpr int xs = PL::pass_of(S) - 1;
#pragma unroll
            for (int j = 0; j < P; ++j) sm->X[xs][xidx(row_of<q>(j))] = Lt[j];
        } else if constexpr (PL::local_reg(S)) {
            constexpr int sl = PL::reg_slot(S);
#pragma unroll
            for (int j = 0; j < P; ++j) Lr[sl][j] = Lt[j];
        } else {
            constexpr int sl = PL::smem_slot(S);
            constexpr int d = 1 << (M - 1 - S);  // last pass: b = 0
            const uint32_t pm = PMW[sl];
            if (d >= 2) {
#pragma unroll
                for (int c = 0; c < P / 4; ++c)
                    if (!((pm >> (4 * c)) & 1u))
                        sm->Ls[sl][c][lane] = make_float4(Lt[4 * c], Lt[4 * c + 1], Lt[4 * c + 2], Lt[4 * c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < P / 2; ++c)
                    if (!((pm >> (2 * c)) & 1u))
                        reinterpret_cast<float2*>(&sm->Ls[sl][c >> 1][lane])[c & 1] =
                            make_float2(Lt[2 * c], Lt[2 * c + 1]);
            }
        }
    }

    // ---- re-saturation of boundary arrays (protected blocks) ----------
    template <int QB>
    __device__ __forceinline__ void resaturate() {
        // boundary e = first(QB): blocks frozen at stage e-1 keep L(e) = +-CAP
        constexpr int e = PL::first(QB);
        constexpr int g = M - e;  // log2 block size
        constexpr int nblk_words = ((1 << e) + 31) / 32;
        bool touched = false;
        for (int w = 0; w < nblk_words; ++w) {
            uint32_t bits = sm->xprot[QB - 1][w];
            while (bits) {
                const int bi = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1;
                touched = true;
                for (int i = lane; i < (1 << g); i += 32) {
                    const int row = (bi << g) + i;
                    const bool neg = (sm->sat[row >> 5] >> (row & 31)) & 1u;
                    sm->X[QB - 1][xidx(row)] = neg ? -kCap : kCap;
                }
            }
        }
        (void)touched;
        __syncwarp();  // X holds other lanes' L(e) writes of the previous iteration
    }

    // ---- one PE stage ---------------------------------------------------
    template <int S>
    __device__ __forceinline__ void pe_stage(float (&Lt)[P]) {
        constexpr int q = PL::pass_of(S);
        constexpr int t = (M - 1 - S) - PL::base_bit(q);
        constexpr int d = 1 << t;
#pragma unroll
        for (int j = 0; j < P; ++j) {
            if (j & d) continue;
            const float lt = Lt[j], lb = Lt[j + d], rt = R[j], rb = R[j + d];
            const float cross = __fmul_rn(alpha, xsmin(lt, rt));
            const float sum_bot = __fadd_rn(lb, rb);
            const float l_top = __fmul_rn(alpha, xsmin(lt, sum_bot));
            const float r_top = __fmaf_rn(alpha, xsmin(rt, sum_bot), 0.0f);
            const float l_bot = __fadd_rn(lb, cross);
            const float r_bot = __fadd_rn(rb, cross);
            if constexpr (S == 0 && KIND != 0) {
                xq |= signbit_u(__fadd_rn(rt, l_top)) << j;
                xq |= signbit_u(__fadd_rn(rb, l_bot)) << (j + d);
            }
            Lt[j] = l_top;
            Lt[j + d] = l_bot;
            R[j] = r_top;
            R[j + d] = r_bot;
        }
    }

    // ---- csfg: candidate check + commit after stage S -------------------
    template <int S>
    __device__ __forceinline__ void check_commit() {
        constexpr int q = PL::pass_of(S);
        constexpr int b = PL::base_bit(q);
        constexpr int g = M - 1 - S;       // log2 block size
        constexpr int W = 1 << (g - b);    // registers per lane in a block
        constexpr int hs = b + K - g;      // block-index bits above the register field
        const int sz = 1 << g;
        const int bi = frontier >> g;
        const int start = bi << g;
        // block membership of this lane's registers
        const int lane_hi = lane >> b;
        uint32_t msk = 0u;
        if (lane_hi == (bi >> hs)) {
            const uint32_t wmask = (W >= 32) ? 0xffffffffu : ((1u << W) - 1u);
            msk = wmask << ((bi & ((1 << hs) - 1)) * W);
        }
        if constexpr (b < 5) {
            // lanes whose low bits do not match the block are outside it
            // only when g < b (never: g >= b); nothing to do
        }
        // x_hat bits of R(S+1)
        uint32_t xb = 0u;
#pragma unroll
        for (int j = P - 1; j >= 0; --j) xb = __funnelshift_l(__float_as_uint(R[j]), xb, 1);
        uint32_t u = xb;
        // butterfly along row bits 0 .. g-1
#pragma unroll
        for (int gp = 0; gp < g; ++gp) {
            if (gp >= b) {
                const int tp = gp - b;
                const uint32_t jm = tp == 0 ? 0x55555555u : tp == 1 ? 0x33333333u
                                  : tp == 2 ? 0x0F0F0F0Fu : tp == 3 ? 0x00FF00FFu : 0x0000FFFFu;
                u ^= (u >> (1 << tp)) & jm;
            } else {
                const uint32_t o = __shfl_xor_sync(kFull, u, 1 << gp);
                if (!((lane >> gp) & 1)) u ^= o;
            }
        }
        const uint32_t viol = u & msk & FZ[q];
        if (__any_sync(kFull, viol != 0u)) return;
        commit<S>(bi, start, sz, msk, xb & msk, u & msk);
    }

    template <int S>
    __device__ __forceinline__ void commit(int bi, int start, int sz, uint32_t msk, uint32_t xbits,
                                       uint32_t ubits) {
        constexpr int q = PL::pass_of(S);
        constexpr int b = PL::base_bit(q);
        constexpr int T = S + 1;
        // 1. saturate / protect L(S+1) (csfg_freeze.cpp:84-86)
        if constexpr (T == M) {
            uint32_t bits = msk;
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1;
                reinterpret_cast<float*>(&sm->LM[j >> 2][lane])[j & 3] = ((xbits >> j) & 1u) ? -kCap : kCap;
            }
        } else if constexpr (PL::is_boundary(T)) {
            constexpr int qb = PL::pass_of(T);
            if (lane == 0) sm->xprot[qb - 1][bi >> 5] |= 1u << (bi & 31);
            scatter<q>(sm->sat, xbits, msk, start, sz);
        } else if constexpr (PL::local_reg(T)) {
            constexpr int sl = PL::reg_slot(T);
            PM[sl] |= msk;
            SS[sl] = (SS[sl] & ~msk) | xbits;
        } else {
            constexpr int sl = PL::smem_slot(T);
            PMW[sl] |= msk;
            uint32_t bits = msk;
            while (bits) {
                const int j = __ffs(bits) - 1;
                bits &= bits - 1;
                reinterpret_cast<float*>(&sm->Ls[sl][j >> 2][lane])[j & 3] = ((xbits >> j) & 1u) ? -kCap : kCap;
            }
        }
        // 2. decided_u (csfg_freeze.cpp:87)
        scatter<q>(sm->dec_u, ubits, msk, start, sz);
        // 3. inactive-PE bookkeeping for stages after S (reference count rule)
        if (start < frontier) {
            if (lane < 32) sm->tmp[lane] = 0;
            __syncwarp();
            for (int r = start + lane; r < frontier; r += 32) {
                const int fo = sm->fst[r];
                for (int s2 = S + 1; s2 < M; ++s2)
                    if (fo < s2 && !((r >> (M - 1 - s2)) & 1)) atomicAdd(&sm->tmp[s2], 1);
            }
            __syncwarp();
            if (lane > S && lane < M) sm->inact[lane] += (sz >> 1) - sm->tmp[lane];
        } else {
            if (lane > S && lane < M) sm->inact[lane] += (sz >> 1);
        }
        for (int i = lane; i < sz; i += 32) sm->fst[start + i] = (uint8_t)S;
        // 4. event log + frontier (csfg_freeze.cpp:88-92)
        if (lane == 0 && a->events && nev < a->ev_cap) {
            int* e = a->events + ((long long)frame_ * a->ev_cap + nev) * 5;
            e[0] = it;
            e[1] = S;
            e[2] = bi;
            e[3] = start;
            e[4] = sz;
        }
        ++nev;
        frontier = start + sz;
        __syncwarp();
    }

    long long frame_;

    // write `bits` (pass-q layout, rows selected by msk) into row-order words
    template <int q>
    __device__ __forceinline__ void scatter(uint32_t* words, uint32_t bits, uint32_t msk, int start,
                                            int sz) {
        constexpr int b = PL::base_bit(q);
        if constexpr (b == 5) {
            // row = lane + 32 j : word j collects bit j of every lane
            const int j0 = start >> 5, j1 = (start + sz + 31) >> 5;
            for (int j = j0; j < j1; ++j) {
                const uint32_t w = __ballot_sync(kFull, (bits >> j) & 1u);
                if (lane == 0) words[j] = w;
            }
        } else if constexpr (b == 0) {
            // row = P*lane + j : the block lives in one lane
            if (msk) {
                const int row0 = P * lane + (__ffs(msk) - 1);
                const int off = row0 & 31;
                const uint32_t bm = (sz >= 32) ? 0xffffffffu : ((1u << sz) - 1u);
                const uint32_t v = (bits >> (__ffs(msk) - 1)) & bm;
                words[row0 >> 5] = (words[row0 >> 5] & ~(bm << off)) | (v << off);
            }
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) {
                if ((msk >> j) & 1u) {
                    const int row = row_of<q>(j);
                    if ((bits >> j) & 1u)
                        atomicOr(&words[row >> 5], 1u << (row & 31));
                    else
                        atomicAnd(&words[row >> 5], ~(1u << (row & 31)));
                }
            }
        }
        __syncwarp();
    }

    // ---- stage S with everything around it; returns false when csfg is done
    template <int S>
    __device__ __forceinline__ bool stage() {
        constexpr int q = PL::pass_of(S);
        constexpr bool first_of_pass = (S == PL::first(q));
        constexpr bool last_of_pass = (S == PL::last(q));
        if constexpr (S == 0) {
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = sm->R0[row_of<0>(j)];
            if constexpr (KIND != 0) xq = 0u;
        } else if constexpr (first_of_pass) {
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = sm->X[q - 1][xidx(row_of<q>(j))];
        }
        if constexpr (PL::is_boundary(S + 1)) {
            if constexpr (KIND == 2)
                resaturate<PL::pass_of(S + 1)>();
            else
                __syncwarp();  // X holds other lanes' L(e) writes of the previous iteration
        }
        float Lt[P];
        load_L<S + 1>(Lt);
        pe_stage<S>(Lt);
        store_L<S>(Lt);
        if constexpr (last_of_pass && S + 1 < M) {
#pragma unroll
            for (int j = 0; j < P; ++j) sm->X[q][xidx(row_of<q>(j))] = R[j];
        }
        if constexpr (first_of_pass || (last_of_pass && S + 1 < M)) __syncwarp();
        if constexpr (KIND == 2) {
            act += (N >> 1) - sm->inact[S];
            check_commit<S>();
            if (frontier >= N) return false;
        } else {
            act += (N >> 1);
        }
        return true;
    }

    template <int S>
    __device__ __forceinline__ bool sweep_from() {
        if (!stage<S>()) return false;
        if constexpr (S + 1 < M)
            return sweep_from<S + 1>();
        else
            return true;
    }

    // û in the last-pass layout (rows P*lane + j), frozen rows forced to 0,
    // the decided prefix [0, pin) taken from decided_u; returned as the
    // row-order word of this lane (lane < NW).
    __device__ __forceinline__ uint32_t u_words(int pin) {
        uint32_t uq = 0u;
#pragma unroll
        for (int j = P - 1; j >= 0; --j) uq = __funnelshift_l(__float_as_uint(R[j]), uq, 1);
        uq &= ~FZ[Q - 1];
        if (pin > 0) {
            const int r0 = P * lane;
            int cnt = pin - r0;
            cnt = cnt < 0 ? 0 : (cnt > P ? P : cnt);
            const uint32_t pm = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
            const uint32_t pmask = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
            const uint32_t db = (sm->dec_u[r0 >> 5] >> (r0 & 31)) & pmask;
            uq = (uq & ~pm) | (db & pm);
        }
        if constexpr (P == 32) {
            return uq;
        } else {
            constexpr int per = 32 / P;
            uint32_t w = 0u;
#pragma unroll
            for (int c = 0; c < per; ++c) {
                const uint32_t v = __shfl_sync(kFull, uq, (lane * per + c) & 31);
                w |= v << (P * c);
            }
            return lane < NW ? w : 0u;
        }
    }

    __device__ __forceinline__ bool gcheck(int pin) {
        uint32_t uw = u_words(pin);
        uw = word_transform(uw, 32);
#pragma unroll
        for (int h = 1; h < NW; h <<= 1) {
            const uint32_t o = __shfl_xor_sync(kFull, uw, h);
            if (!(lane & h)) uw ^= o;
        }
        const uint32_t xw = transpose32(xq, lane);
        return !__any_sync(kFull, (uw ^ xw) != 0u);
    }

    __device__ __forceinline__ void run(const DecodeArgs& args, WarpSmem<M>* s, int ln) {
        a = &args;
        sm = s;
        lane = ln;
        alpha = args.alpha;
        // frozen rows per pass layout (fixed for the launch)
#pragma unroll
        for (int q = 0; q < Q; ++q) FZ[q] = 0u;
        fz_init<0>();
        FZW = lane < NW ? args.frozen_bits[lane] : 0u;

        if (lane < kNumCounters) sm->cnt[lane] = 0ull;
        __syncwarp();

        for (;;) {
            long long f = 0;
            if (lane == 0) f = (long long)atomicAdd(args.queue, 1ull);
            f = __shfl_sync(kFull, f, 0);
            if (f >= args.frames) break;
            frame_ = f;
            // ---- load LLRs (coalesced float4), bound check ----
            const float4* src = reinterpret_cast<const float4*>(args.llr + f * (long long)N);
            bool bad = false;
#pragma unroll
            for (int i = 0; i < P / 4; ++i) {
                float4 v = __ldcs(src + lane + 32 * i);
                bad |= !(fabsf(v.x) <= kClampFreeBound) | !(fabsf(v.y) <= kClampFreeBound) |
                       !(fabsf(v.z) <= kClampFreeBound) | !(fabsf(v.w) <= kClampFreeBound);
                v.x = __fadd_rn(v.x, 0.0f);
                v.y = __fadd_rn(v.y, 0.0f);
                v.z = __fadd_rn(v.z, 0.0f);
                v.w = __fadd_rn(v.w, 0.0f);
                reinterpret_cast<float4*>(sm->R0)[lane + 32 * i] = v;
            }
            if (__any_sync(kFull, bad)) {
                if (lane == 0) {
                    const unsigned long long slot = atomicAdd(args.list_len, 1ull);
                    args.list[slot] = f;
                }
                continue;
            }
            init_frame();
            int iters = (KIND == 0) ? args.max_iter : 0;
            int stop = 0;
            bool converged = false;
            for (int t = 1; t <= args.max_iter; ++t) {
                if constexpr (KIND == 2) {
                    if (frontier >= N || converged) break;
                    iters = t;
                }
                it = t;
                const bool full = sweep_from<0>();
                if constexpr (KIND == 1) {
                    if (gcheck(0)) {
                        iters = t;
                        stop = 1;
                        break;
                    }
                } else if constexpr (KIND == 2) {
                    if (full && frontier < N) converged = gcheck(frontier);
                }
            }
            if constexpr (KIND == 1) {
                if (stop == 0) iters = args.max_iter;
            }
            uint32_t uw;
            if constexpr (KIND == 2) {
                stop = frontier >= N ? 2 : (converged ? 1 : 0);
                if (frontier >= N)
                    uw = lane < NW ? sm->dec_u[lane] : 0u;
                else
                    uw = u_words(frontier);
            } else {
                uw = u_words(0);
            }
            // ---- outputs ----
            if (args.u_bits && lane < NW) args.u_bits[f * NW + lane] = uw;
            if (lane == 0) {
                if (args.iters) args.iters[f] = iters;
                if (args.pe) args.pe[f] = act;
                if (args.stop) args.stop[f] = (uint8_t)stop;
                if (args.nev) args.nev[f] = nev;
            }
            if (args.counters) {
                int be = 0;
                if (lane < NW) be = __popc((uw ^ args.truth_u[f * NW + lane]) & ~FZW);
                be = __reduce_add_sync(kFull, be);
                unsigned long long v = 0ull;
                switch (lane) {
                    case kCntFrames: v = 1; break;
                    case kCntBitErr: v = (unsigned long long)be; break;
                    case kCntFrameErr: v = be > 0; break;
                    case kCntIters: v = (unsigned long long)iters; break;
                    case kCntItersSq: v = (unsigned long long)iters * iters; break;
                    case kCntPe: v = (unsigned long long)act; break;
                    case kCntEvents: v = (unsigned long long)nev; break;
                    case kCntStop0: v = stop == 0; break;
                    case kCntStop1: v = stop == 1; break;
                    case kCntStop2: v = stop == 2; break;
                    default: break;
                }
                if (lane < kNumCounters) sm->cnt[lane] += v;
            }
        }
        if (args.counters && lane < kNumCounters && sm->cnt[lane])
            atomicAdd(&args.counters[lane], sm->cnt[lane]);
    }

    template <int q>
    __device__ __forceinline__ void fz_init() {
        uint32_t w = 0u;
#pragma unroll
        for (int j = 0; j < P; ++j) w |= (uint32_t)(a->frozen_rows[row_of<q>(j)] != 0) << j;
        FZ[q] = w;
        if constexpr (q + 1 < Q) fz_init<q + 1>();
    }

    __device__ __forceinline__ void init_frame() {
#pragma unroll
        for (int j = 0; j < P; ++j) R[j] = 0.f;
#pragma unroll
        for (int sl = 0; sl < PL::NLR; ++sl) {
            PM[sl] = 0u;
            SS[sl] = 0u;
#pragma unroll
            for (int j = 0; j < P; ++j) Lr[sl][j] = 0.f;
        }
#pragma unroll
        for (int sl = 0; sl < PL::NLS; ++sl) {
            PMW[sl] = 0u;
#pragma unroll
            for (int c = 0; c < P / 4; ++c) sm->Ls[sl][c][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int x = 0; x < Q - 1; ++x)
#pragma unroll
            for (int i = 0; i < P / 4; ++i)
                reinterpret_cast<float4*>(sm->X[x])[lane + 32 * i] = make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t fl = FZ[Q - 1];
#pragma unroll
        for (int c = 0; c < P / 4; ++c)
            sm->LM[c][lane] = make_float4(((fl >> (4 * c)) & 1u) ? kCap : 0.f, ((fl >> (4 * c + 1)) & 1u) ? kCap : 0.f,
                                          ((fl >> (4 * c + 2)) & 1u) ? kCap : 0.f, ((fl >> (4 * c + 3)) & 1u) ? kCap : 0.f);
        if (lane < NW) sm->dec_u[lane] = 0u;
#pragma unroll
        for (int x = 0; x < Q - 1; ++x)
            if (lane < NW) sm->xprot[x][lane] = 0u;
        sm->inact[lane] = 0;
#pragma unroll
        for (int i = 0; i < N / 128; ++i) reinterpret_cast<uint32_t*>(sm->fst)[lane + 32 * i] = 0x7f7f7f7fu;
        frontier = 0;
        nev = 0;
        act = 0;
        xq = 0u;
        __syncwarp();
    }
};

template <int M, int KIND>
__global__ void __launch_bounds__(32) bp_warp_kernel(DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char wsm[];
    Dec<M, KIND> dec;
    dec.run(a, reinterpret_cast<WarpSmem<M>*>(wsm), threadIdx.x & 31);
}

}  // namespace wk

int warp_kernel_supported(int m) { return m >= 7 && m <= 10; }

size_t warp_smem_bytes(int m) {
    switch (m) {
        case 7: return sizeof(wk::WarpSmem<7>);
        case 8: return sizeof(wk::WarpSmem<8>);
        case 9: return sizeof(wk::WarpSmem<9>);
        case 10: return sizeof(wk::WarpSmem<10>);
    }
    return 0;
}

template <int M, int KIND>
static cudaError_t launch_w(const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(wk::WarpSmem<M>);
    cudaError_t e = cudaFuncSetAttribute(wk::bp_warp_kernel<M, KIND>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    wk::bp_warp_kernel<M, KIND><<<grid, 32, smem, st>>>(a);
    return cudaGetLastError();
}

template <int M>
static cudaError_t launch_wk(const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (a.kind) {
        case 0: return launch_w<M, 0>(a, grid, st);
        case 1: return launch_w<M, 1>(a, grid, st);
        default: return launch_w<M, 2>(a, grid, st);
    }
}

cudaError_t launch_warp(const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (a.m) {
        case 7: return launch_wk<7>(a, grid, st);
        case 8: return launch_wk<8>(a, grid, st);
        case 9: return launch_wk<9>(a, grid, st);
        case 10: return launch_wk<10>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

int warp_blocks_per_sm(int m, int kind) {
    int nb = 0;
    const size_t smem = warp_smem_bytes(m);
    cudaError_t e = cudaErrorInvalidValue;
#define PBP_OCC(MM)                                                                               \
    case MM:                                                                                      \
        if (kind == 0) {                                                                          \
            cudaFuncSetAttribute(wk::bp_warp_kernel<MM, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wk::bp_warp_kernel<MM, 0>, 32, smem); \
        } else if (kind == 1) {                                                                   \
            cudaFuncSetAttribute(wk::bp_warp_kernel<MM, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wk::bp_warp_kernel<MM, 1>, 32, smem); \
        } else {                                                                                  \
            cudaFuncSetAttribute(wk::bp_warp_kernel<MM, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem); \
            e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wk::bp_warp_kernel<MM, 2>, 32, smem); \
        }                                                                                         \
        break;
    switch (m) {
        PBP_OCC(7)
        PBP_OCC(8)
        PBP_OCC(9)
        PBP_OCC(10)
    }
#undef PBP_OCC
    return e == cudaSuccess ? nb : 0;
}

}  // namespace pbp
