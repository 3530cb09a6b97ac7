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
// Between passes R(e) goes through a padded row-indexed shared array X
// (index = row + 4*(row/32): conflict-free scalar stores from pass 0 and
// conflict-free 128-bit loads in the last pass, no address arithmetic) that
// then holds L(e) in place. L(s) inside a pass stays in registers (n <= 512,
// and n = 1024's first pass) or in lane-private float4 shared slots
// (n = 1024's last pass).
//
// Arithmetic: Eq. (1) of src/bp_core.cpp:18-32 in fp32, two PEs at a time
// with the packed FADD2 / FMUL2 / FFMA2 (add/mul/fma.rn.f32x2) and
// min.xorsign.abs (FMNMX.XORSIGN): 6 issue slots per PE, every product and
// sum rounded separately as in the reference (no contraction).
// r_top = fma(alpha, m, +0) never yields -0, so R's sign bit equals the
// reference's (v < 0) decision; clamps are elided
// because frames with |LLR| > kClampFreeBound are re-routed to the generic
// kernel, which keeps them.
//
// The csfg schedule (src/csfg_freeze.cpp:99-152) is followed literally:
// after each stage the candidate block containing the frontier is checked
// on the fresh R(s+1) (sign bits of only the block's registers packed with
// funnel shifts, XOR butterfly along the block's row bits: in-word for
// register bits, shfl_xor for lane bits), committed, and the PE mask takes
// effect from the next stage on. Inactive PEs are computed anyway (their
// outputs are never read by an active PE); only the saturated boundary
// L(f+1) of a frozen block must survive, enforced per storage class
// (read-side override for register arrays, predicated stores for shared
// slots, re-saturation for X). PE activations are counted by the reference
// rule from per-stage inactive-row counts.
#include <type_traits>

#include "pbp_common.cuh"
#include "tmem.cuh"

namespace pbp {
namespace wk {

constexpr unsigned kFull = 0xffffffffu;
#ifndef PBP_TMEM_G
#define PBP_TMEM_G 32
#endif
constexpr int kTG = PBP_TMEM_G;  // TMEM columns per tcgen05.ld/st of a 32-value row
__constant__ uint32_t c_jmask[5] = {0x55555555u, 0x33333333u, 0x0F0F0F0Fu, 0x00FF00FFu, 0x0000FFFFu};

template <int M_>
struct Plan {
    static constexpr int M = M_;
    static constexpr int N = 1 << M;
    static constexpr int P = N / 32;
    static constexpr int K = M - 5;
    static constexpr int Q = (M + K - 1) / K;
    static constexpr int NW = N / 32;
    static constexpr int NX = N + N / 8;  // padded boundary array
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
    // protection-mask slot of array L(s): register arrays first, then shared ones
    static constexpr int prot_slot(int s) { return local_reg(s) ? reg_slot(s) : NLR + smem_slot(s); }
    // csfg: stages of the last pass (base bit 0) keep every candidate block
    // inside one lane; those checks read raw R rows of two lanes (see snap_rows)
    static constexpr int SL = (Q - 1) * K;  // first stage of the last pass
    static constexpr int NL = M - SL;       // stages in the last pass
    // n = 1024: eight frames (warps) per CTA and per SM, each warp with 256
    // TMEM columns of its lane quarter: R(0) [C_R0, +32), L(m) [C_LM, +32)
    // and the csfg snapshots of R(1..5) [C_S + 32 s, +32), pass-0 layout
    // (lane l, column j <-> row l + 32 j; L(m) in the last-pass layout)
    static constexpr bool TM = (M == 10);
    static constexpr int WARPS = TM ? 8 : 1;
    static constexpr uint32_t C_R0 = 0, C_LM = 32, C_S = 64, C_LM0 = 224;  // C_LM0: L(m) at frame start
};

// LMB: L(m) as bit masks (csfg: frees 3.8 KB for an 8th warp per SM at n =
// 1024); float4 slots otherwise (measured faster for the other decoders)
template <int M, bool LMB = false>
struct alignas(16) WarpSmem {
    using PL = Plan<M>;
    float X[PL::Q - 1][PL::NX];            // pass boundaries: R(e) then L(e), padded rows
    float4 Ls[PL::NLS][PL::P / 4][32];     // lane-private L slots (last pass, n=1024)
    float4 LM[(LMB || PL::TM) ? 1 : PL::P / 4][32];  // L(m), lane-private, last-pass layout (float slots; TMEM at n=1024)
    uint32_t lmz[32], lmn[32];             // L(m) in {0, +-CAP}: nonzero / negative bits per lane (LMB)
    uint32_t pm[PL::NLR + PL::NLS][32];    // per lane: rows whose L(s) is a frozen boundary
    uint32_t ss[PL::NLR][32];              // ... and their signs (register arrays)
    uint32_t dec_u[PL::NW];                // decided_u bits (row order)
    uint32_t sat[PL::NW];                  // x_hat of the latest commit per row
    uint32_t xprot[PL::Q - 1][PL::NW];     // per boundary: blocks frozen at stage e-1
    int tmp[32];
    unsigned long long cnt[16];            // per-warp counter accumulators
    uint32_t su[PL::SL][32];               // per stage < SL: block-transformed sign bits of R(s+1)
                                           // (TM: per early commit k, u_hat of its block)
    uint32_t sv[PL::TM ? 1 : PL::SL][32];  // ... and violated groups, OR over a block's lanes
    float rs[PL::NL][2][PL::P];            // per stage >= SL: R(s+1) of the two candidate lanes
    int cS[PL::M], cbi[PL::M];             // commits recorded by the walks of one iteration
    uint32_t frz[PL::NW];                  // frozen rows, row-order words
    uint32_t fz[PL::Q][32];                // frozen rows per pass layout
    uint8_t fst[PL::N];                    // freeze_stage per row
    uint32_t skipm[PL::TM ? 5 : 1];        // PBP_SKIP_FROZEN: pass-0 register columns inactive at stage s
};

__device__ __forceinline__ float xsmin(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// packed fp32x2 arithmetic (FADD2 / FMUL2 / FFMA2), round-to-nearest per lane half
__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{ .reg .b64 a, b, d; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; add.rn.f32x2 d, a, b; mov.b64 {%0, %1}, d; }"
        : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
__device__ __forceinline__ void mul2s(float& d0, float& d1, float s, float a0, float a1) {
    asm("{ .reg .b64 a, b, d; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %4}; mul.rn.f32x2 d, a, b; mov.b64 {%0, %1}, d; }"
        : "=f"(d0), "=f"(d1) : "f"(s), "f"(a0), "f"(a1));
}
__device__ __forceinline__ void fma2s0(float& d0, float& d1, float s, float a0, float a1) {
    // s * a + (+0): never -0
    asm("{ .reg .b64 a, b, c, d; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %4}; mov.b64 c, 0; "
        "fma.rn.f32x2 d, a, b, c; mov.b64 {%0, %1}, d; }"
        : "=f"(d0), "=f"(d1) : "f"(s), "f"(a0), "f"(a1));
}

__device__ __forceinline__ uint32_t transpose32(uint32_t x, int lane) {
#pragma unroll
    for (int i = 0; i < 5; ++i) {
        const int s = 16 >> i;
        const uint32_t m = i == 0 ? 0x0000FFFFu : i == 1 ? 0x00FF00FFu : i == 2 ? 0x0F0F0F0Fu
                         : i == 3 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(kFull, x, s);
        x = (lane & s) ? ((x & ~m) | ((y >> s) & m)) : ((x & m) | ((y & m) << s));
    }
    return x;
}

__device__ __forceinline__ uint32_t jmask(int tp) {
    return tp == 0 ? 0x55555555u : tp == 1 ? 0x33333333u : tp == 2 ? 0x0F0F0F0Fu
         : tp == 3 ? 0x00FF00FFu : 0x0000FFFFu;
}

#ifdef PBP_DEBUG_PROGRESS
// hang debugging only: per-warp progress words in mapped host memory
__device__ unsigned long long* g_dbg;
extern "C" int pbp_debug_set(void* p) { return cudaMemcpyToSymbol(g_dbg, &p, sizeof(p)) != cudaSuccess; }
#define PBP_DBG(loc)                                                                                           \
    do {                                                                                                       \
        if (lane == 0 && g_dbg)                                                                                \
            *(volatile unsigned long long*)&g_dbg[blockIdx.x * 8 + (threadIdx.x >> 5)] =                       \
                ((unsigned long long)frame_ << 32) | ((unsigned long long)it << 8) | (unsigned long long)(loc); \
    } while (0)
#else
#define PBP_DBG(loc)
#endif
#ifdef PBP_PROF_SECTIONS
// timing experiments only: per-warp clock64 time per code section
__device__ unsigned long long g_prof[8];
extern "C" int pbp_prof_read(unsigned long long* out, int reset) {
    if (cudaMemcpyFromSymbol(out, g_prof, sizeof(g_prof)) != cudaSuccess) return 1;
    if (reset) {
        unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        cudaMemcpyToSymbol(g_prof, z, sizeof(z));
    }
    return 0;
}
#ifndef PBP_SLOT_APPLY_TM
#define PBP_SLOT_APPLY_TM 4
#endif
#define PBP_T0(v) const long long v = clock64()
#define PBP_T1(v, k) do { if (lane == 0) prof[k] += clock64() - (v); } while (0)
#else
#define PBP_T0(v)
#define PBP_T1(v, k)
#endif

// XH: also record each freeze event's x_hat (trace calls; a separate
// instantiation keeps the decode kernel's code unchanged)
template <int M, int KIND, bool XH = false>
struct Dec {
#ifdef PBP_PROF_SECTIONS
    unsigned long long prof[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#endif
    using PL = Plan<M>;
    static constexpr int N = PL::N, P = PL::P, K = PL::K, Q = PL::Q, NW = PL::NW;

    using Smem = WarpSmem<M, KIND == 2>;
    static constexpr bool TM = PL::TM;
    Smem* sm;
    float4* r0g;  // this warp's channel LLRs in global scratch, lane-private pass-0 layout (n < 1024)
    uint32_t tb;  // this warp's TMEM columns (n = 1024)
    const uint32_t* fzt;  // n = 1024: walk0's frozen-row field words, [F/32][lane] (shared by the CTA)
    const DecodeArgs* a;
    int lane;
    float alpha;

    float R[P];
    float Lr[PL::NLR][P];
    uint32_t FZ[Q];  // frozen rows per pass layout (bit j = row_of<q>(j))

    int frontier, nev, it;
    int inact;     // lane s < M: inactive top rows of stage s
    // csfg walk state of the current iteration
    int L1;        // lane of the frontier when the last pass starts (candidate rows: L1, L1+1)
    int nce_;      // commits of the early walk (stages < SL)
    int s_last_, fr_start_;
    bool done_;    // the frontier reached n
    uint32_t prot;   // bit per protection slot: some lane holds a frozen-boundary row
    long long act, frame_;
    long long cset_;  // counter set sm->cnt accumulates (cnt_batch > 0)
    uint32_t xq;     // channel-side decisions of stage 0, permuted pass-0 layout
    int xperm;       // lane holding row-order word `lane` of x_hat after transpose

    template <int q>
    __device__ __forceinline__ int row_of(int j) const {
        constexpr int b = PL::base_bit(q);
        return (lane & ((1 << b) - 1)) | (j << b) | ((lane >> b) << (b + K));
    }
    __device__ __forceinline__ static int xpad(int row) { return row + 4 * (row >> 5); }

    // ---- boundary array access (R out of pass q / L into pass q) ----------
    template <int q>
    __device__ __forceinline__ void x_load(const float* X, float (&v)[P]) const {
        if constexpr (PL::base_bit(q) == 0) {
            const float4* p = reinterpret_cast<const float4*>(X + xpad(P * lane));
#pragma unroll
            for (int c = 0; c < P / 4; ++c) {
                const float4 t = p[c];
                v[4 * c] = t.x;
                v[4 * c + 1] = t.y;
                v[4 * c + 2] = t.z;
                v[4 * c + 3] = t.w;
            }
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) v[j] = X[xpad(row_of<q>(j))];
        }
    }
    template <int q>
    __device__ __forceinline__ void x_store(float* X, const float (&v)[P]) const {
        if constexpr (PL::base_bit(q) == 0) {
            float4* p = reinterpret_cast<float4*>(X + xpad(P * lane));
#pragma unroll
            for (int c = 0; c < P / 4; ++c) p[c] = make_float4(v[4 * c], v[4 * c + 1], v[4 * c + 2], v[4 * c + 3]);
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) X[xpad(row_of<q>(j))] = v[j];
        }
    }

    // ---- L(T) as read by stage T-1 -----------------------------------------
    template <int T>
    __device__ __forceinline__ void load_L(float (&Lt)[P]) {
        constexpr int q = PL::pass_of(T - 1);
        if constexpr (T == M && TM) {
            tm::wait_st();  // a stage m-1 commit's column update (apply_tm)
            tm::ld_row<kTG>(tb + PL::C_LM, Lt);
            tm::wait_ld();
        } else if constexpr (T == M && KIND == 2) {
            const uint32_t z = sm->lmz[lane], ng = sm->lmn[lane];
#pragma unroll
            for (int j = 0; j < P; ++j) Lt[j] = ((z >> j) & 1u) ? (((ng >> j) & 1u) ? -kCap : kCap) : 0.f;
        } else if constexpr (T == M) {
#pragma unroll
            for (int c = 0; c < P / 4; ++c) {
                const float4 v = sm->LM[c][lane];
                Lt[4 * c] = v.x;
                Lt[4 * c + 1] = v.y;
                Lt[4 * c + 2] = v.z;
                Lt[4 * c + 3] = v.w;
            }
        } else if constexpr (PL::is_boundary(T)) {
            x_load<q>(sm->X[PL::pass_of(T) - 1], Lt);
        } else if constexpr (PL::local_reg(T)) {
            constexpr int sl = PL::reg_slot(T);
#pragma unroll
            for (int j = 0; j < P; ++j) Lt[j] = Lr[sl][j];
            // TM: fixed up once after each sweep (fixup_regs), off the stages' code path
            if (!TM && (prot & (1u << sl))) {  // uniform, rare: boundary rows read as +-CAP
                const uint32_t pm = sm->pm[sl][lane], ss = sm->ss[sl][lane];
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if ((pm >> j) & 1u) Lt[j] = ((ss >> j) & 1u) ? -kCap : kCap;
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
        if constexpr (S == 0) {
            // L(0) is only consumed through x_hat (packed in the PE loop)
        } else if constexpr (PL::is_boundary(S)) {
            x_store<PL::pass_of(S)>(sm->X[PL::pass_of(S) - 1], Lt);
        } else if constexpr (PL::local_reg(S)) {
            constexpr int sl = PL::reg_slot(S);
#pragma unroll
            for (int j = 0; j < P; ++j) Lr[sl][j] = Lt[j];
        } else {
            constexpr int sl = PL::smem_slot(S);
            constexpr int ps = PL::prot_slot(S);
            constexpr int d = 1 << (M - 1 - S);  // last pass: b = 0
            if (!TM && !(prot & (1u << ps))) {  // TM: one (predicated) version, smaller hot code
#pragma unroll
                for (int c = 0; c < P / 4; ++c)
                    sm->Ls[sl][c][lane] = make_float4(Lt[4 * c], Lt[4 * c + 1], Lt[4 * c + 2], Lt[4 * c + 3]);
            } else {
                // frozen-boundary rows (blocks of >= 2 rows) keep their saturation
                const uint32_t pm = sm->pm[ps][lane];
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
    }

    // ---- re-saturation of a boundary array (blocks frozen at stage e-1) ---
    template <int QB>
    __device__ __forceinline__ void resaturate() {
        constexpr int e = PL::first(QB);
        constexpr int g = M - e;  // log2 block size
        constexpr int nblk_words = ((1 << e) + 31) / 32;
#pragma unroll 1
        for (int w = 0; w < nblk_words; ++w) {
            uint32_t bits = sm->xprot[QB - 1][w];
#pragma unroll 1
            while (bits) {
                const int bi = 32 * w + __ffs(bits) - 1;
                bits &= bits - 1;
#pragma unroll 1
                for (int i = lane; i < (1 << g); i += 32) {
                    const int row = (bi << g) + i;
                    const bool neg = (sm->sat[row >> 5] >> (row & 31)) & 1u;
                    sm->X[QB - 1][xpad(row)] = neg ? -kCap : kCap;
                }
            }
        }
        __syncwarp();  // X holds other lanes' L(e) writes of the previous iteration
    }

    // ---- the PEs of stage S: two at a time with packed math --------------
    template <int S>
    __device__ __forceinline__ void pe_stage(float (&Lt)[P]) {
        constexpr int q = PL::pass_of(S);
        constexpr int t = (M - 1 - S) - PL::base_bit(q);
        constexpr int d = 1 << t;
#ifdef PBP_SCALAR_PE
        constexpr bool packed = false;
#else
        constexpr bool packed = true;
#endif
#ifdef PBP_SKIP_FROZEN
        // experiment (DESIGN.md §5 "Skipping frozen PEs"): at n = 1024 a block frozen at
        // stage f <= 3 covers whole register columns of the pass-0 layout (all 32
        // lanes), so its PEs of stages f+1..4 are skipped by a warp-uniform branch per
        // packed pair; the skipped rows keep stale R / L, which only inactive PEs and
        // pinned rows read (the boundary L(f+1) is restored by fixup_regs as before)
        constexpr bool kSkip = TM && KIND == 2 && q == 0 && S > 0;
        const uint32_t skc = kSkip ? sm->skipm[S] : 0u;
#else
        constexpr bool kSkip = false;
        const uint32_t skc = 0u;
#endif
        if constexpr (d >= 2 && packed) {
            // stage 0: x_hat bits pushed into four independent 8-bit chains
            // (pushes 8c..8c+7 in chain c), concatenated below into the same bit
            // positions a single chain would give (push p at bit P-1-p)
            uint32_t xqc[4] = {0u, 0u, 0u, 0u};
#pragma unroll
            for (int j = 0; j < P; j += 2) {
                if (j & d) continue;
                if (kSkip && ((skc >> j) & 3u) == 3u) continue;  // warp-uniform
                const float lt0 = Lt[j], lt1 = Lt[j + 1], lb0 = Lt[j + d], lb1 = Lt[j + d + 1];
                const float rt0 = R[j], rt1 = R[j + 1], rb0 = R[j + d], rb1 = R[j + d + 1];
                float c0, c1, s0, s1, lt0o, lt1o, rt0o, rt1o, lb0o, lb1o, rb0o, rb1o;
                // products as fma(alpha, m, +0): ptxas fuses a bare mul.rn.f32x2 into a
                // following add.rn.f32x2 (FFMA2, one rounding) even under -fmad=false;
                // an FFMA2 with the zero register is the single-rounded product (it only
                // turns a -0 product into +0, which changes no decision).
                fma2s0(c0, c1, alpha, xsmin(lt0, rt0), xsmin(lt1, rt1));
                add2(s0, s1, lb0, lb1, rb0, rb1);
                fma2s0(lt0o, lt1o, alpha, xsmin(lt0, s0), xsmin(lt1, s1));
                fma2s0(rt0o, rt1o, alpha, xsmin(rt0, s0), xsmin(rt1, s1));
                add2(lb0o, lb1o, lb0, lb1, c0, c1);
                add2(rb0o, rb1o, rb0, rb1, c0, c1);
                if constexpr (S == 0 && KIND != 0) {
                    // channel-side decisions (R(0) + L(0) < 0), pushed in a fixed order
                    float x0, x1, x2, x3;
                    add2(x0, x1, rt0, rt1, lt0o, lt1o);
                    add2(x2, x3, rb0, rb1, lb0o, lb1o);
                    uint32_t& c = xqc[j >> 2];
                    c = __funnelshift_l(__float_as_uint(x0), c, 1);
                    c = __funnelshift_l(__float_as_uint(x1), c, 1);
                    c = __funnelshift_l(__float_as_uint(x2), c, 1);
                    c = __funnelshift_l(__float_as_uint(x3), c, 1);
                }
                Lt[j] = lt0o;
                Lt[j + 1] = lt1o;
                Lt[j + d] = lb0o;
                Lt[j + d + 1] = lb1o;
                R[j] = rt0o;
                R[j + 1] = rt1o;
                R[j + d] = rb0o;
                R[j + d + 1] = rb1o;
            }
            if constexpr (S == 0 && KIND != 0) {
                uint32_t x = 0u;
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int n = (P - 8 * c) < 8 ? (P - 8 * c) : 8;  // pushes in chain c
                    if (n > 0) x |= xqc[c] << (P - 8 * c - n);
                }
                xq = x;
            }
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) {
                if (j & d) continue;
                if (kSkip && ((skc >> j) & 1u)) continue;  // warp-uniform
                const float lt = Lt[j], lb = Lt[j + d], rt = R[j], rb = R[j + d];
                const float cross = __fmul_rn(alpha, xsmin(lt, rt));
                const float sum_bot = __fadd_rn(lb, rb);
                const float l_top = __fmul_rn(alpha, xsmin(lt, sum_bot));
                const float l_bot = __fadd_rn(lb, cross);
                if constexpr (S == 0 && KIND != 0) {
                    xq |= (__float_as_uint(__fadd_rn(rt, l_top)) >> 31) << (P - 1 - xpush(j));
                    xq |= (__float_as_uint(__fadd_rn(rb, l_bot)) >> 31) << (P - 1 - xpush(j + d));
                }
                Lt[j] = l_top;
                R[j] = __fmaf_rn(alpha, xsmin(rt, sum_bot), 0.0f);
                Lt[j + d] = l_bot;
                R[j + d] = __fadd_rn(rb, cross);
            }
        }
    }

    // push index of stage-0 row-bit j in the packed x_hat order (see run())
    __device__ __forceinline__ static constexpr int xpush(int j) {
        return (j >= P / 2) ? 4 * ((j - P / 2) >> 1) + 2 + ((j - P / 2) & 1) : 4 * (j >> 1) + (j & 1);
    }

    // sign bits of R[J0 .. J0+W) packed at bits 0..W-1
    template <int J0, int W>
    __device__ __forceinline__ uint32_t pack_range() const {
        uint32_t v = 0u;
#pragma unroll
        for (int i = W - 1; i >= 0; --i) v = __funnelshift_l(__float_as_uint(R[J0 + i]), v, 1);
        return v;
    }

    // sign bits of all P registers (bit j = R[j] < 0), four independent
    // funnel-shift chains combined with PRMT (short dependency chain)
    __device__ __forceinline__ uint32_t pack_all() const {
        if constexpr (P >= 32) {
            const uint32_t a0 = pack_range<0, 8>(), a1 = pack_range<8, 8>();
            const uint32_t a2 = pack_range<16, 8>(), a3 = pack_range<24, 8>();
            return __byte_perm(__byte_perm(a0, a1, 0x0040), __byte_perm(a2, a3, 0x0040), 0x5410);
        } else if constexpr (P == 16) {
            return __byte_perm(pack_range<0, 8>(), pack_range<8, 8>(), 0x0040) & 0xffffu;
        } else {
            return pack_range<0, P>();
        }
    }

    // ---- csfg: the candidate chain of one iteration -------------------------
    // csfg_freeze.cpp:109-119 with the verified restructuring of SURVEY.md 0.9:
    // the sweep computed every stage and snapshotted the sign bits of each
    // R(s+1) (sm->snap); here the reference's stage loop is replayed in order -
    // stop once the frontier covers n, count stage s's active PEs, check the
    // block containing the frontier, commit - with the stage as a runtime value,
    // so this code exists once. Exact because a stage-s commit only changes
    // what later stages of the same sweep compute inside the frozen block
    // (never read by an active PE or a later candidate) and L(s+1), which is
    // next read in the following iteration.
    static constexpr uint32_t mask_of(int which) {
        uint32_t m = 0;
        for (int x = 1; x <= M; ++x)
            if ((which == 0 && PL::local_reg(x)) || (which == 1 && PL::local_smem(x))) m |= 1u << x;
        return m;
    }

    // Sweep side of the check for stage S < SL: the sign bits of R(S+1) of
    // this lane's rows (bit j = row_of(j)); the rest happens in verdicts().
    template <int S>
    __device__ __forceinline__ void snapshot() {
        if constexpr (S < PL::SL - 1) sm->su[S][lane] = pack_all();
    }

    // For every stage S < SL: x_hat's polar transform inside every block (all
    // candidate positions at once): in-word for the register bits, shfl_xor
    // for the lane bits; then the frozen-row violations OR-ed over the lanes a
    // block spans (its lane_lo bits). sv[S][l] tells, for the lane group of l,
    // which register groups would be rejected; su[S] keeps u_hat. Run once per
    // iteration off the sweep's straight line, the stages' independent
    // shuffle chains interleaved.
    template <int S>
    __device__ __forceinline__ void verdict_of(uint32_t& u, uint32_t& v) {
        constexpr int q = PL::pass_of(S);
        constexpr int b = PL::base_bit(q);
        constexpr int g = M - 1 - S;  // >= b before the last pass
#pragma unroll
        for (int tp = 0; tp < g - b; ++tp) u ^= (u >> (1 << tp)) & jmask(tp);
#pragma unroll
        for (int gp = 0; gp < b; ++gp) {
            const uint32_t o = __shfl_xor_sync(kFull, u, 1 << gp);
            if (!((lane >> gp) & 1)) u ^= o;
        }
        v = u & FZ[q];
        if constexpr (b == 5) {
            v = __reduce_or_sync(kFull, v);
        } else {
#pragma unroll
            for (int gp = 0; gp < b; ++gp) v |= __shfl_xor_sync(kFull, v, 1 << gp);
        }
    }
    // stages 0 .. SL-2; stage SL-1's block is one row-order word of R(SL),
    // which is in X when the walk runs (walk_early)
    static constexpr int NV = PL::SL - 1;
    template <int S>
    __device__ __forceinline__ void verdicts_from(uint32_t (&u)[NV], uint32_t (&v)[NV]) {
        verdict_of<S>(u[S], v[S]);
        if constexpr (S + 1 < NV) verdicts_from<S + 1>(u, v);
    }
    __device__ __forceinline__ void verdicts() {
        uint32_t u[NV], v[NV];
#pragma unroll
        for (int S = 0; S < NV; ++S) u[S] = sm->su[S][lane];
        verdicts_from<0>(u, v);
#pragma unroll
        for (int S = 0; S < NV; ++S) {
            sm->sv[S][lane] = v[S];
            sm->su[S][lane] = u[S];
        }
    }

    // The reference's stage loop (csfg_freeze.cpp:109-119), replayed in two
    // walks. Between two commits the frontier is fixed, so lane s evaluates
    // stage s's candidate for the current frontier and one ballot finds the
    // first accepting stage; stages before it reject, it commits, the frontier
    // moves, the rest are evaluated again. The early walk (stages < SL, from
    // the snapshots' verdicts) runs when the sweep reaches the last pass; it
    // fixes the lane whose rows can still hold candidates (L1, L1+1), whose
    // R(s+1) the last pass then stores raw. The late walk checks the last-pass
    // stages on those rows. Side effects (apply_freeze) follow after the sweep.
    __device__ __forceinline__ void walk_early() {
        verdicts();
        __syncwarp();  // verdicts of the whole warp
        constexpr int SL = PL::SL;
        fr_start_ = frontier;
        int nc = 0;
        s_last_ = M - 1;
        done_ = false;
        int s_next = 0;
        constexpr int g4 = M - SL;  // stage SL-1: blocks of 2^g4 <= 32 rows
        uint32_t u4 = 0u;
#pragma unroll 1
        while (s_next < SL) {
            // stage SL-1's candidate: its rows' sign bits straight from R(SL) in X
            const int A4 = (frontier >> g4) << g4;
            {
                const float xv = sm->X[Q - 2][xpad((A4 & ~31) + lane)];
                const uint32_t w4 = __ballot_sync(kFull, __float_as_int(xv) < 0);
                u4 = (w4 >> (A4 & 31)) & low_mask(1 << g4);
#pragma unroll
                for (int tp = 0; tp < g4; ++tp) u4 ^= (u4 >> (1 << tp)) & jmask(tp);
            }
            bool acc = false;
            if (lane == SL - 1 && lane >= s_next) {
                acc = (u4 & (sm->frz[A4 >> 5] >> (A4 & 31)) & low_mask(1 << g4)) == 0u;
            } else if (lane >= s_next && lane < SL - 1) {
                const int st = lane;
                const int q = st / K;
                const int b = (M - K - q * K) > 0 ? (M - K - q * K) : 0;
                const int g = M - 1 - st;
                const int W = 1 << (g - b);
                const int hs = b + K - g;
                const int bi = frontier >> g;
                const int j0 = (bi & ((1 << hs) - 1)) * W;
                const uint32_t wm = W >= 32 ? 0xffffffffu : ((1u << W) - 1u);
                acc = ((sm->sv[st][(bi >> hs) << b] >> j0) & wm) == 0u;
            }
            const uint32_t am = __ballot_sync(kFull, acc);
            if (!am) break;
            const int st = __ffs(am) - 1;
            const int g = M - 1 - st;
            if (lane == 0) {
                sm->cS[nc] = st;
                sm->cbi[nc] = frontier >> g;
            }
            if (st == SL - 1) {
                // u_hat of the block in the pass layout, for apply_commits:
                // lane bit j0 = u of the row this lane holds at register j0
                constexpr int qq = Q - 2, b = PL::base_bit(qq);
                const int j0 = (A4 >> b) & (P - 1);
                const int r = row_of<qq>(j0);
                const bool in = r >= A4 && r < A4 + (1 << g4);
                sm->su[SL - 1][lane] = in ? (((u4 >> (r - A4)) & 1u) << j0) : 0u;
            }
            ++nc;
            frontier = ((frontier >> g) + 1) << g;
            if (frontier >= N) {
                s_last_ = st;
                done_ = true;
                break;
            }
            s_next = st + 1;
        }
        nce_ = nc;
        L1 = done_ ? -4 : frontier / P;
    }

    // n = 1024 (TM): the reference's stage loop over the first pass
    // (csfg_freeze.cpp:109-119) from the sweep's TMEM snapshots of R(1..5).
    // At a fixed frontier F the candidate blocks of stages 0..4 (512 >> s
    // rows: words j0_s = F/32 rounded down to 16 >> s, every lane) are
    // checked together: their sign bits go to disjoint fields of one word per
    // lane (16, 8, 4, 2 and 1 bits at offsets 0, 16, 24, 28, 30), so one
    // in-word pass transforms the register bits of all five blocks, one
    // 5-level butterfly across lanes their lane bits, and one OR-reduction of
    // the frozen-row violations gives all five verdicts. The first accepting
    // stage commits; the frontier moves and the later stages are evaluated
    // again at the new frontier (rare: ~1 first-pass commit per frame at
    // 3 dB). Commit side effects follow after the sweep (apply_commits).
    __device__ __forceinline__ void walk0() {
        static_assert(M == 10 && PL::SL == 5 && P == 32, "walk0: n = 1024 layout");
        PBP_DBG(10);
        tm::wait_st();  // this sweep's snapshots
        PBP_DBG(11);
        fr_start_ = frontier;
        int nc = 0;
        s_last_ = M - 1;
        done_ = false;
        uint32_t skip = 0u;  // stages already past (one decision per stage)
#pragma unroll 1
        while (true) {
            const int jf = frontier >> 5;
            const int j00 = jf & ~15, j01 = jf & ~7, j02 = jf & ~3, j03 = jf & ~1, j04 = jf;
            // two load phases keep the peak at 16 extra registers (R(5) and
            // the register L levels are live here)
            float v0[16], v1[8], v2[4], v3[2], v4[1];
            tm::ld16(tb + PL::C_S + j00, v0);
            tm::wait_ld();
            // sign bits, independent chains: bit i of a chain = element i
            uint32_t c0 = 0u, c1 = 0u, c2 = 0u, c3 = 0u;
#pragma unroll
            for (int i = 7; i >= 0; --i) {
                c0 = __funnelshift_l(__float_as_uint(v0[i]), c0, 1);
                c1 = __funnelshift_l(__float_as_uint(v0[8 + i]), c1, 1);
            }
            tm::ld8(tb + PL::C_S + 32 + j01, v1);
            tm::ld4(tb + PL::C_S + 64 + j02, v2);
            tm::ld2(tb + PL::C_S + 96 + j03, v3);
            tm::ld1(tb + PL::C_S + 128 + j04, v4);
            tm::wait_ld();
#pragma unroll
            for (int i = 7; i >= 0; --i) c2 = __funnelshift_l(__float_as_uint(v1[i]), c2, 1);
#pragma unroll
            for (int i = 3; i >= 0; --i) c3 = __funnelshift_l(__float_as_uint(v2[i]), c3, 1);
            c3 = __funnelshift_l(__float_as_uint(v3[1]), c3, 1);  // bits: v3[1] v2[3..0] -> shifted below
            uint32_t u = __byte_perm(c0, c1, 0x7740) | (c2 << 16);  // c1 < 256: bytes 2, 3 zero
            // c3 holds v2[3..0] at bits 4..1 and v3[1] at bit 0: rebuild fields 2..4
            const uint32_t f2 = (c3 >> 1) & 0xFu;
            const uint32_t f3 = ((__float_as_uint(v3[0]) >> 31) | ((c3 & 1u) << 1));
            const uint32_t f4 = __float_as_uint(v4[0]) >> 31;
            u |= (f2 << 24) | (f3 << 28) | (f4 << 30);
            // polar transform inside every field (register bits), then across lanes
            u ^= (u >> 1) & 0x55555555u;
            u ^= (u >> 2) & 0x03333333u;
            u ^= (u >> 4) & 0x000F0F0Fu;
            u ^= (u >> 8) & 0x000000FFu;
#pragma unroll
            for (int gp = 0; gp < 5; ++gp) {
                const uint32_t o = __shfl_xor_sync(kFull, u, 1 << gp);
                if (!((lane >> gp) & 1)) u ^= o;
            }
            const uint32_t fzw = fzt[jf * 32 + lane];  // frozen rows of the five blocks, same fields
            PBP_DBG(12);
            const uint32_t V = __reduce_or_sync(kFull, u & fzw);
            uint32_t acc = (uint32_t)((V & 0xFFFFu) == 0u) | ((uint32_t)(((V >> 16) & 0xFFu) == 0u) << 1) |
                           ((uint32_t)(((V >> 24) & 0xFu) == 0u) << 2) | ((uint32_t)(((V >> 28) & 3u) == 0u) << 3) |
                           ((uint32_t)(((V >> 30) & 1u) == 0u) << 4);
            acc &= ~skip;
            if (!acc) break;
            const int st = __ffs(acc) - 1;
            const int g = M - 1 - st;  // the block has 2^g rows
            const int bi = frontier >> g;
            if (lane == 0) {
                sm->cS[nc] = st;
                sm->cbi[nc] = bi;
            }
            // u_hat of the block in the pass-0 layout (bit j = row lane + 32 j), for apply_commits
            const int W = 16 >> st, off = st == 0 ? 0 : (st == 1 ? 16 : (st == 2 ? 24 : (st == 3 ? 28 : 30)));
            sm->su[nc][lane] = ((u >> off) & low_mask(W)) << (jf & ~(W - 1));
            ++nc;
            frontier = (bi + 1) << g;
            if (frontier >= N) {
                s_last_ = st;
                done_ = true;
                break;
            }
            skip = (2u << st) - 1u;
            if (st == PL::SL - 1) break;
        }
        nce_ = nc;
        L1 = done_ ? -4 : frontier / P;
        PBP_DBG(13);
    }

    // last-pass stage S: lanes L1 and L1+1 keep R(S+1) (rows P*lane + j)
    template <int S>
    __device__ __forceinline__ void snap_rows() {
        const unsigned c = (unsigned)(lane - L1);
        if (c < 2u) {
            float4* d = reinterpret_cast<float4*>(&sm->rs[S - PL::SL][c][0]);
#pragma unroll
            for (int i = 0; i < P / 4; ++i) d[i] = make_float4(R[4 * i], R[4 * i + 1], R[4 * i + 2], R[4 * i + 3]);
        }
    }

    // Late walk over the last-pass stages. Every candidate block lies in the
    // window of 2*W1 <= 32 rows from A5 = frontier rounded down to the first
    // last-pass block size W1 (after a commit the blocks shrink). x_t = sign
    // bits of the window after stage SL + t (one ballot); lane t transforms x_t
    // inside its 2^g-row blocks and marks the rejected ones (bit at the block's
    // first row); every lane then runs the stage loop as a straight scan.
    struct LastWalk {
        int A5;               // window start
        uint32_t x[PL::NL];   // window sign bits per last-pass stage (uniform)
        int E[PL::NL];        // block end of stage SL + t's commit (blocks tile [A0, frontier))
        int A0;               // start of the first commit's block
        uint32_t xl, ul;      // lane t: x_hat / u_hat bits of the window at stage SL + t
        int Al;               // lane t: A[t]
        uint32_t cmask;       // bit t: stage SL + t committed
    };
    __device__ __forceinline__ void walk_late(LastWalk& w) {
        constexpr int SL = PL::SL, NL = PL::NL;
        constexpr int W1 = 1 << (M - 1 - SL);
        __syncwarp();  // rs rows
        w.cmask = 0u;
        if (done_) return;
        w.A5 = frontier & ~(W1 - 1);
        const int off = w.A5 - P * L1;  // window offset in the two stored lanes' rows
        uint32_t xl = 0u;
#pragma unroll
        for (int t = 0; t < NL; ++t) {
            const float v = lane < 2 * W1 ? (&sm->rs[t][0][0])[off + lane] : 0.f;
            const uint32_t xt = __ballot_sync(kFull, lane < 2 * W1 && __float_as_int(v) < 0);
            w.x[t] = xt;
            if (lane == t) xl = xt;
        }
        uint32_t viol;
        {
            const int w0 = w.A5 >> 5;
            const unsigned long long f2 =
                (unsigned long long)sm->frz[w0] | ((unsigned long long)(w0 + 1 < NW ? sm->frz[w0 + 1] : 0u) << 32);
            viol = (uint32_t)(f2 >> (w.A5 & 31));
        }
        const int g = M - 1 - (SL + lane);  // lane t < NL: its stage's block bits
        uint32_t u = xl;
#pragma unroll
        for (int tp = 0; tp < K - 1; ++tp)
            if (tp < g) u ^= (u >> (1 << tp)) & jmask(tp);
        w.xl = xl;
        w.ul = u;
        viol &= u;
#pragma unroll
        for (int tp = 0; tp < K - 1; ++tp)
            if (tp < g) viol |= viol >> (1 << tp);
        // the reference's stage loop over the last pass
        int F = frontier, slast = s_last_, A0 = N;
        uint32_t cm = 0u;
        bool done = false;
#pragma unroll
        for (int t = 0; t < NL; ++t) {
            const uint32_t vt = __shfl_sync(kFull, viol, t);
            const int gt = M - 1 - (SL + t);
            const int A = (F >> gt) << gt;
            if (lane == t) w.Al = A;
            const bool acc = !done && !((vt >> (A - w.A5)) & 1u);
            cm |= (uint32_t)acc << t;
            A0 = (acc && cm == (1u << t)) ? A : A0;  // first commit's block start
            F = acc ? A + (1 << gt) : F;
            w.E[t] = F;                              // end of stage t's block when it commits
            const bool fin = acc && F >= N;
            slast = fin ? SL + t : slast;
            done = done || fin;
        }
        w.cmask = cm;
        w.A0 = A0;
        s_last_ = slast;
        frontier = F;
        done_ = done;
    }

    // n = 1024 (TM): the reference's stage loop over the last pass
    // (csfg_freeze.cpp:109-119). As walk_late, specialised: the window is the
    // 32 rows from A5 = frontier rounded down to 16 (lanes L1, L1+1 stored
    // them, rs[t] = R(6 + t)); lane t transforms stage 5 + t's window bits
    // inside its blocks of 16 >> t rows and marks rejected blocks; the stage
    // loop is a uniform scan.
    struct LateTM {
        int A5;
        uint32_t x[PL::NL];  // window sign bits of R(6 + t) (uniform)
        int At[PL::NL];      // block start of stage 5 + t at its check (uniform)
        uint32_t u, xl;      // lane t: u_hat / x_hat bits of the window at stage 5 + t
        int Al;              // lane t: At[t]
        uint32_t cm;         // bit t: stage 5 + t committed
    };
    __device__ __forceinline__ void walk_tm(LateTM& w) {
        static_assert(M == 10 && PL::SL == 5 && PL::NL == 5, "walk_tm: n = 1024 layout");
        __syncwarp();  // rs rows
        w.cm = 0u;
        if (done_) return;
        const int A5 = frontier & ~15;
        w.A5 = A5;
        const float* rsf = &sm->rs[0][0][0] + (A5 - P * L1);  // rs[t][c][j], t stride 2 P
        uint32_t xl = 0u;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const uint32_t xt = __ballot_sync(kFull, __float_as_int(rsf[2 * P * t + lane]) < 0);
            w.x[t] = xt;
            xl = lane == t ? xt : xl;
        }
        const int w0 = A5 >> 5;
        const uint32_t fw = (uint32_t)(((unsigned long long)sm->frz[w0] |
                                        ((unsigned long long)(w0 + 1 < NW ? sm->frz[w0 + 1] : 0u) << 32)) >>
                                       (A5 & 31));
        const int g = 4 - lane;  // lane t < 5: log2 of its block size
        uint32_t u = xl;
#pragma unroll
        for (int tp = 0; tp < 4; ++tp)
            if (tp < g) u ^= (u >> (1 << tp)) & jmask(tp);
        w.u = u;
        w.xl = xl;
        uint32_t viol = u & fw;
#pragma unroll
        for (int tp = 0; tp < 4; ++tp)
            if (tp < g) viol |= viol >> (1 << tp);
        // the scan on window offsets (f = frontier - A5 < 16); rows from offset lim
        // on do not exist, and a commit reaching them completes the frame
        uint32_t vt[5];
#pragma unroll
        for (int t = 0; t < 5; ++t) vt[t] = __shfl_sync(kFull, viol, t);  // off the scan's chain
        const int lim = N - A5;
        int f = frontier - A5, Al = 0;
        uint32_t cm = 0u;
#pragma unroll
        for (int t = 0; t < 5; ++t) {
            const int B = 16 >> t;
            const int o = f & ~(B - 1);
            w.At[t] = A5 + o;
            Al = lane == t ? o : Al;
            const bool acc = f < lim && !((vt[t] >> o) & 1u);
            cm |= (uint32_t)acc << t;
            f = acc ? o + B : f;
        }
        w.Al = A5 + Al;
        w.cm = cm;
        done_ = f >= lim;
        if (done_) s_last_ = 5 + (31 - __clz(cm));  // the commit that reached n is the iteration's last
        frontier = A5 + f;
    }

    // Re-covered rows [start, fr_start) of a commit at stage S (only the first
    // commit of an iteration can re-cover rows decided before): the top rows
    // already inactive at a stage s2 > S under their old freeze_stage (fo < s2)
    // must not be counted twice. Per-lane counts in 16-bit fields of five words
    // (stages (1,2) .. (9)), one warp sum per word; returns this lane's count
    // (lane = stage s2).
    __device__ __forceinline__ int recovered_inactive(int S, int start, int fr_start) const {
        static_assert(M <= 10, "stages 1..9 in five packed words");
        uint32_t c[5] = {0u, 0u, 0u, 0u, 0u};
#pragma unroll 1
        for (int r = start + lane; r < fr_start; r += 32) {
            const int fo = sm->fst[r];
            const int lo = fo > S ? fo : S;
            const uint32_t top = __brev(~(uint32_t)r) >> (32 - M);  // bit s2: row r is a top row at s2
            const uint32_t msk = top & ~((2u << lo) - 1u);            // s2 in (max(fo, S), m)
#pragma unroll
            for (int q = 0; q < 5; ++q) c[q] += ((msk >> (2 * q + 1)) & 1u) | (((msk >> (2 * q + 2)) & 1u) << 16);
        }
        int mine = 0;
#pragma unroll
        for (int q = 0; q < 5; ++q) {
            const uint32_t t = __reduce_add_sync(kFull, c[q]);
            if (lane == 2 * q + 1) mine = (int)(t & 0xffffu);
            if (lane == 2 * q + 2) mine = (int)(t >> 16);
        }
        return lane < M ? mine : 0;
    }

    // TM: the saturated boundary L(S+1) of blocks frozen at a first-pass stage S
    // whose level lives in registers: after each sweep (and each commit) the
    // protected rows are set back to +-CAP, so the next sweep's stage S reads
    // them as the reference does (its inactive stage S+1 PEs never write them).
    // One place after the sweep instead of a select in every read keeps the
    // stages' straight-line code free of these rarely taken blocks.
    template <int SL_ = 0>
    __device__ __forceinline__ void fixup_regs_from() {
        if constexpr (SL_ < PL::NLR) {
            if (__any_sync(kFull, prot & (1u << SL_))) {  // warp-uniform: no reconvergence stack
                const uint32_t pm = sm->pm[SL_][lane], ss = sm->ss[SL_][lane];
#pragma unroll
                for (int j = 0; j < P; ++j) {  // selects, not branches
                    const float sat = __uint_as_float(__float_as_uint(kCap) | (((ss >> j) & 1u) << 31));
                    Lr[SL_][j] = ((pm >> j) & 1u) ? sat : Lr[SL_][j];
                }
            }
            fixup_regs_from<SL_ + 1>();
        }
    }
    __device__ __forceinline__ void fixup_regs() { fixup_regs_from<0>(); }

    // apply_freeze (csfg_freeze.cpp:82-93) for the first-pass commits of one
    // iteration (TM, rare: ~1 per frame at 3 dB), kept compact so that it costs
    // little instruction cache when it runs. Commit k (stage S <= 4) covers the
    // 16 >> S registers j0.. of every lane (pass-0 layout, row = lane + 32 j).
    // Returns this lane's newly inactive top rows (lane = a later stage).
    __device__ __forceinline__ int apply_early_tm() {
        static_assert(M == 10 && PL::SL == 5, "apply_early_tm: n = 1024 layout");
        const int nce = nce_, fr_start = fr_start_;
        __syncwarp();
        int dinact = 0;
#pragma unroll 1
        for (int k = 0; k < nce; ++k) {
            const int S = sm->cS[k], bi = sm->cbi[k];
            const int g = M - 1 - S, W = 16 >> S;
            const int start = bi << g, sz = 1 << g;
            const int j0 = (start >> 5) & 31;
            const uint32_t wm = (W >= 32) ? 0xffffffffu : ((1u << W) - 1u);
            // u_hat of the block (walk0); x_hat = T(u_hat): the transform is an involution
            const uint32_t uu = sm->su[k][lane];
            uint32_t xx = uu;
#pragma unroll 1
            for (int tp = 0; tp < 4 - S; ++tp) xx ^= (xx >> (1 << tp)) & c_jmask[tp];
#pragma unroll
            for (int gp = 0; gp < 5; ++gp) {
                const uint32_t o = __shfl_xor_sync(kFull, xx, 1 << gp);
                if (!((lane >> gp) & 1)) xx ^= o;
            }
            const uint32_t xbits = (xx >> j0) & wm, ubits = (uu >> j0) & wm;
            // 1. saturate L(S+1) (csfg_freeze.cpp:84-86): register level, or the
            //    pass boundary L(5) (re-saturated before each of its reads)
            if (S < 4) {
                sm->pm[S][lane] |= wm << j0;
                sm->ss[S][lane] = (sm->ss[S][lane] & ~(wm << j0)) | (xbits << j0);
                prot |= 1u << S;
            } else {
                if (lane == 0) sm->xprot[0][bi >> 5] |= 1u << (bi & 31);
                const uint32_t xw = __ballot_sync(kFull, xbits & 1u);  // one register: row word j0
                if (lane == 0) sm->sat[start >> 5] = xw;
            }
            // 2. decided_u (:87): row-order word j0 + i collects bit i of every lane
            uint32_t dw = 0u;
#pragma unroll 1
            for (int i = 0; i < W; ++i) {
                const uint32_t b = __ballot_sync(kFull, (ubits >> i) & 1u);
                dw = lane == i ? b : dw;
            }
            if (lane < W) sm->dec_u[(start >> 5) + lane] = dw;
            // 3. inactive top rows of the stages after S; only the first commit can
            //    re-cover rows decided before (freeze_stage still holds their stages):
            //    those already inactive at s2 are counted once (packed warp sums)
            if (lane > S && lane < M) dinact += sz >> 1;
            if (k == 0 && start < fr_start) dinact -= recovered_inactive(S, start, fr_start);
#ifdef PBP_SKIP_FROZEN
            if (S <= 3 && lane == 0) {  // register columns start/32 .. (start+sz)/32 - 1
                const uint32_t cols = low_mask(sz >> 5) << ((start >> 5) & 31);
                for (int s2 = S + 1; s2 <= 4; ++s2) sm->skipm[s2] |= cols;
            }
#endif
            //    freeze_stage over the block (:86), 16 bytes per lane and step
            {
                const uint32_t w4 = 0x01010101u * (uint32_t)S;
#pragma unroll 1
                for (int i = 16 * lane; i < sz; i += 512)
                    *reinterpret_cast<uint4*>(&sm->fst[start + i]) = make_uint4(w4, w4, w4, w4);
            }
            // 4. event log (:91-92)
            if (lane == 0 && a->events && nev < a->ev_cap) {
                int* e = a->events + ((long long)frame_ * a->ev_cap + nev) * 5;
                e[0] = it;
                e[1] = S;
                e[2] = bi;
                e[3] = start;
                e[4] = sz;
            }
            if (XH && a->ev_xhat && nev < a->ev_cap) {  // FreezeEvent::x_hat (trace calls only)
                uint32_t xw = 0u;
#pragma unroll 1
                for (int i = 0; i < W; ++i) {
                    const uint32_t b = __ballot_sync(kFull, (xbits >> i) & 1u);
                    xw = lane == i ? b : xw;
                }
                if (lane < W) a->ev_xhat[((long long)frame_ * a->ev_cap + nev) * NW + (start >> 5) + lane] = xw;
            }
            ++nev;
            __syncwarp();
        }
        return dinact;
    }

    // apply_freeze (csfg_freeze.cpp:82-93) for the last-pass commits of one
    // iteration (TM): lane i takes window row A5 + i (saturation of L(S+1),
    // freeze_stage, decided_u by ballot), lane t takes stage 5 + t's commit
    // (protection mask, event). The first commit of an iteration may re-cover
    // rows decided before: their top rows already inactive at a stage s2 > S
    // under their old freeze_stage are counted once (one packed warp sum).
    __device__ __forceinline__ void apply_tm(const LateTM& w, int& dinact) {
        const uint32_t cm = w.cm;
        const int A5 = w.A5, r = A5 + lane;
        // stage m-1 commit: its L(m) column, loaded first (the rest hides the latency)
        const bool c9 = (cm >> 4) & 1u;
        float v9 = 0.f;
        if (c9) tm::ld1(tb + PL::C_LM + (w.At[4] & 31), &v9);
        int Sr = -1;
        uint32_t xb = 0u;
        int tr = 0;
#pragma unroll
        for (int t = 0; t < 5; ++t) {  // selects: the committed blocks are disjoint
            const bool in = ((cm >> t) & 1u) && (unsigned)(r - w.At[t]) < (16u >> t);
            Sr = in ? 5 + t : Sr;
            tr = in ? t : tr;
            xb = in ? (w.x[t] >> lane) & 1u : xb;
        }
        const uint32_t ub = (__shfl_sync(kFull, w.u, tr) >> lane) & 1u;
        const bool cov = Sr >= 0;
        if (nce_ == 0) {
            const bool rc = cov && r < fr_start_;
            if (__any_sync(kFull, rc)) {
                uint32_t pk = 0u;
                if (rc) {
                    const int fo = sm->fst[r];
                    const int S0 = 5 + (__ffs(cm) - 1);
                    const int lo = fo > S0 ? fo : S0;
                    const uint32_t top = __brev(~(uint32_t)r) >> (32 - M);  // bit s2: top row at s2
                    const uint32_t was = top & ~((2u << lo) - 1u);          // s2 in (lo, m)
                    pk = ((was >> 6) & 1u) | (((was >> 7) & 1u) << 8) | (((was >> 8) & 1u) << 16) |
                         (((was >> 9) & 1u) << 24);
                }
                const uint32_t c = __reduce_add_sync(kFull, pk);
                if (lane >= 6 && lane < M) dinact -= (int)((c >> (8 * (lane - 6))) & 0xffu);
            }
        }
        {  // predicated stores (no divergent branch): L(S+1) saturation and freeze_stage of row r
            const int owner = r >> 5, j = r & 31;
            float* base = reinterpret_cast<float*>(&sm->Ls[(Sr > 5 ? Sr : 5) - 5][0][0]);
            const float sv = __uint_as_float(__float_as_uint(kCap) | (xb << 31));
            if (cov && Sr < M - 1) base[((j >> 2) * 32 + owner) * 4 + (j & 3)] = sv;
            if (cov) sm->fst[r] = (uint8_t)Sr;
        }
        if (c9) {  // stage m-1: L(m) of one row, TMEM column j of lane owner
            const int r9 = w.At[4];
            const uint32_t x9 = (w.x[4] >> (r9 - A5)) & 1u;
            tm::wait_ld();
            if (lane == (r9 >> 5)) v9 = x9 ? -kCap : kCap;
            tm::st1(tb + PL::C_LM + (r9 & 31), v9);  // completed before the next L(m) load (wait_st there)
        }
        // decided_u over the window (two row-order words; shared atomics: no round trip)
        const uint32_t cvw = __ballot_sync(kFull, cov), uw = __ballot_sync(kFull, cov && ub);
        {  // lanes 0 and 1 own the window's two words: plain read-modify-write
            const int wd = (A5 >> 5) + lane, sh = A5 & 31;
            const uint32_t mk = lane == 0 ? cvw << sh : (sh ? cvw >> (32 - sh) : 0u);
            const uint32_t vv = lane == 0 ? uw << sh : (sh ? uw >> (32 - sh) : 0u);
            if (lane < 2 && mk) sm->dec_u[wd] = (sm->dec_u[wd] & ~mk) | vv;
        }
        // inactive top rows: a stage-S block of B rows has B/2 top rows at every later stage
        if (lane < M) dinact += (int)((__brev((cm << 5) & ((1u << lane) - 1u)) >> (32 - M)) >> 1);
        const bool mine = (cm >> lane) & 1u;
        const int B = 16 >> lane, A = w.Al;
        const uint32_t wm = (1u << B) - 1u;
        if (mine && lane < 4) atomicOr(&sm->pm[PL::NLR + lane][A >> 5], wm << (A & 31));  // L(S+1): shared slot S - 5
        if (a->events) {  // trace calls only (uniform)
            const int e_ix = nev + __popc(cm & ((1u << lane) - 1u));
            if (mine && e_ix < a->ev_cap) {
                int* e = a->events + ((long long)frame_ * a->ev_cap + e_ix) * 5;
                e[0] = it;
                e[1] = 5 + lane;
                e[2] = A >> (4 - lane);
                e[3] = A;
                e[4] = B;
            }
            if (XH && a->ev_xhat && mine && e_ix < a->ev_cap)  // the block is <= 16 aligned rows
                atomicOr(&a->ev_xhat[((long long)frame_ * a->ev_cap + e_ix) * NW + (A >> 5)],
                         ((w.xl >> (A - A5)) & wm) << (A & 31));
        }
        prot |= (cm & 0xFu) << PL::NLR;
        nev += __popc(cm);
    }

    // after the sweep: late walk, side effects, stage_pass counts of stages
    // 0..s_last under the freeze state each ran with (a commit at stage s only
    // changes inact[s' > s]). Returns frontier < n (the reference then runs the
    // pinned G-check).
    __device__ __forceinline__ bool finish_iter() {
        if constexpr (TM) {
            PBP_T0(tw);
            LateTM w;
            walk_tm(w);
            PBP_T1(tw, 3);
            PBP_T0(ta);
            int dinact = 0;
            if (__builtin_expect(nce_ != 0, 0)) dinact = apply_early_tm();
            PBP_T1(ta, 4);
            PBP_T0(tb2);
            if (w.cm) apply_tm(w, dinact);
            if (lane < M) inact += dinact;
            if (prot & ((1u << PL::NLR) - 1u)) fixup_regs();
            __syncwarp();
            PBP_T1(tb2, PBP_SLOT_APPLY_TM);
        } else {
            PBP_T0(tw);
            LastWalk w;
            walk_late(w);
            PBP_T1(tw, 3);
            PBP_T0(ta);
            if (nce_ | w.cmask) {
                const int dinact = apply_commits(w);
                if (lane < M) inact += dinact;
                __syncwarp();
            }
            PBP_T1(ta, 4);
        }
        const int v = lane <= s_last_ ? (N >> 1) - inact : 0;
        act += __reduce_add_sync(kFull, v);
        return !done_;
    }

    // apply_freeze (csfg_freeze.cpp:82-93) for the commits of one iteration:
    // saturate/protect L(S+1), decided_u, inactive-PE counts, freeze_stage,
    // event log. Commits of the early walk one after the other with the whole
    // warp (their blocks span lanes); last-pass commits one per lane (blocks
    // are disjoint, their L(S+1) are different arrays).
    template <class Walk>
    __device__ __forceinline__ int apply_commits(const Walk& w) {
        constexpr uint32_t REGM = mask_of(0), SMEMM = mask_of(1);
        const int nce = nce_, fr_start = fr_start_;
        __syncwarp();
        int dinact = 0;  // this lane's stage: newly inactive top rows
#pragma unroll 1
        for (int k = 0; k < nce; ++k) {
            const int S = sm->cS[k], bi = sm->cbi[k];
            const int q = S / K;
            const int b = (M - K - q * K) > 0 ? (M - K - q * K) : 0;
            const int g = M - 1 - S;
            const int W = 1 << (g - b);
            const int hs = b + K - g;
            const int j0 = (bi & ((1 << hs) - 1)) * W;
            const bool in_block = (lane >> b) == (bi >> hs);
            const uint32_t wm = W >= 32 ? 0xffffffffu : ((1u << W) - 1u);
            const uint32_t msk = in_block ? (wm << j0) : 0u;
            const int sz = 1 << g, start = bi << g;
            // u_hat of the block; x_hat = T(u_hat) (the transform is an involution)
            const uint32_t uu = TM ? sm->su[k][lane] : sm->su[S][lane];
            uint32_t xx = uu;
#pragma unroll 1
            for (int tp = 0; tp < g - b; ++tp) xx ^= (xx >> (1 << tp)) & c_jmask[tp];
#pragma unroll 1
            for (int gp = 0; gp < (g < b ? g : b); ++gp) {
                const uint32_t o = __shfl_xor_sync(kFull, xx, 1 << gp);
                if (!((lane >> gp) & 1)) xx ^= o;
            }
            const uint32_t xbits = (xx >> j0) & wm, ubits = (uu >> j0) & wm;
            // 1. saturate / protect L(S+1) (csfg_freeze.cpp:84-86)
            const int T = S + 1;
            if (T == M) {  // stage m-1 commits are last-pass commits (apply_last); kept for completeness
                if (in_block) {
                    sm->lmz[lane] |= wm << j0;
                    sm->lmn[lane] = (sm->lmn[lane] & ~(wm << j0)) | (xbits << j0);
                }
            } else if ((SMEMM >> T) & 1u) {
                float4* base = &sm->Ls[__popc(SMEMM & ((1u << T) - 1u))][0][0];
                if (in_block) {
                    if (W >= 4) {
#pragma unroll 1
                        for (int i = 0; i < W; i += 4)
                            base[((j0 + i) >> 2) * 32 + lane] = make_float4(
                                ((xbits >> i) & 1u) ? -kCap : kCap, ((xbits >> (i + 1)) & 1u) ? -kCap : kCap,
                                ((xbits >> (i + 2)) & 1u) ? -kCap : kCap, ((xbits >> (i + 3)) & 1u) ? -kCap : kCap);
                    } else {
#pragma unroll 1
                        for (int i = 0; i < W; ++i) {
                            const int j = j0 + i;
                            reinterpret_cast<float*>(&base[(j >> 2) * 32 + lane])[j & 3] =
                                ((xbits >> i) & 1u) ? -kCap : kCap;
                        }
                    }
                }
                if (T != M) {
                    const int ps = PL::NLR + __popc(SMEMM & ((1u << T) - 1u));
                    sm->pm[ps][lane] |= msk;
                    if (__any_sync(kFull, msk != 0u)) prot |= 1u << ps;
                }
            } else if ((REGM >> T) & 1u) {
                const int sl = __popc(REGM & ((1u << T) - 1u));
                sm->pm[sl][lane] |= msk;
                sm->ss[sl][lane] = (sm->ss[sl][lane] & ~msk) | ((xbits << j0) & msk);
                if (__any_sync(kFull, msk != 0u)) prot |= 1u << sl;
            } else {  // pass boundary: re-saturated before its next read
                if (lane == 0) sm->xprot[T / K - 1][bi >> 5] |= 1u << (bi & 31);
                scatter(sm->sat, xbits, in_block, b, q, W, j0, start);
            }
            // 2. decided_u (csfg_freeze.cpp:87)
            scatter(sm->dec_u, ubits, in_block, b, q, W, j0, start);
            // 3. inactive top rows of the stages after S. Only the first commit of
            //    an iteration can re-cover rows decided before (later blocks start
            //    at the frontier), so freeze_stage still holds their old stages.
            if (lane > S && lane < M) dinact += sz >> 1;
            if (k == 0 && start < fr_start) dinact -= recovered_inactive(S, start, fr_start);
            //    freeze_stage over the block (csfg_freeze.cpp:86)
            if (sz >= 4) {
                const uint32_t w4 = 0x01010101u * (uint32_t)S;
#pragma unroll 1
                for (int i = 4 * lane; i < sz; i += 128) *reinterpret_cast<uint32_t*>(&sm->fst[start + i]) = w4;
            } else if (lane < sz) {
                sm->fst[start + lane] = (uint8_t)S;
            }
            // 4. event log (csfg_freeze.cpp:91-92)
            if (lane == 0 && a->events && nev < a->ev_cap) {
                int* e = a->events + ((long long)frame_ * a->ev_cap + nev) * 5;
                e[0] = it;
                e[1] = S;
                e[2] = bi;
                e[3] = start;
                e[4] = sz;
            }
            if (XH && a->ev_xhat && nev < a->ev_cap)  // FreezeEvent::x_hat (trace calls only)
                scatter(a->ev_xhat + ((long long)frame_ * a->ev_cap + nev) * NW, xbits, in_block, b, q, W, j0, start);
            ++nev;
        }
        if constexpr (!TM) {
            if (w.cmask) apply_last(w, nce, fr_start, dinact);
        }
        return dinact;
    }

    // Last-pass commits (cmask bit t: stage SL + t), all inside the window:
    // lane i takes row A5 + i (its block's stage and x_hat bit: saturation,
    // freeze_stage); lane t takes stage SL + t's commit (decided_u, protection
    // mask, event).
    __device__ __forceinline__ void apply_last(const LastWalk& w, int nce, int fr_start, int& dinact) {
        constexpr uint32_t REGM = mask_of(0), SMEMM = mask_of(1);
        constexpr int SL = PL::SL, NL = PL::NL;
        const uint32_t cmask = w.cmask;
        // inactive top rows: a stage-S block of sz rows has sz/2 top rows at
        // every later stage (stages are distinct and increasing in one walk)
        const uint32_t cm = cmask << SL;
        if (lane < M) dinact += (int)((__brev(cm & ((1u << lane) - 1u)) >> (32 - M)) >> 1);
        const int r = w.A5 + lane;
        int Sr = -1;
        uint32_t xbit = 0u;
        // row r >= A0 belongs to the earliest committed stage whose block ends after it
#pragma unroll
        for (int t = NL - 1; t >= 0; --t) {
            if (((cmask >> t) & 1u) && r < w.E[t]) {
                Sr = SL + t;
                xbit = (w.x[t] >> lane) & 1u;
            }
        }
        if (r < w.A0) Sr = -1;
        int fo = kNotFrozen;
        if (Sr >= 0) fo = sm->fst[r];
        if (nce == 0) {
            // the first commit of the iteration may re-cover decided rows
            // [A0, fr_start): those already inactive at a stage s2 > S0 under
            // their old freeze_stage are not counted twice
            const int t0 = __ffs(cmask) - 1;
            const int S0 = SL + t0;
            if (__any_sync(kFull, Sr >= 0 && r < fr_start)) {
                uint32_t was = 0u;
                if (Sr >= 0 && r < fr_start) {
                    const int lo = fo > S0 ? fo : S0;  // s2 > max(fo, S0)
                    const uint32_t top = __brev(~(uint32_t)r) >> (32 - M);  // bit s2: row is top at s2
                    was = top & ~((2u << lo) - 1u);
                }
#pragma unroll
                for (int s2 = 1; s2 < M; ++s2) {
                    const int c = __popc(__ballot_sync(kFull, (was >> s2) & 1u));
                    if (lane == s2) dinact -= c;
                }
            }
        }
        // 1. saturate L(S+1) (csfg_freeze.cpp:84-86), 3. freeze_stage (:86)
        if (Sr >= 0) {
            const int T = Sr + 1;
            const int owner = r / P, j = r % P;  // last-pass layout: row = P*lane + j
            if (T == M) {  // one row per iteration: a plain read-modify-write of the owner's bits
                if constexpr (!TM) {
                    sm->lmz[owner] |= 1u << j;
                    sm->lmn[owner] = (sm->lmn[owner] & ~(1u << j)) | (xbit << j);
                }
            } else if ((SMEMM >> T) & 1u) {
                float* base = reinterpret_cast<float*>(&sm->Ls[__popc(SMEMM & ((1u << T) - 1u))][0][0]);
                base[((j >> 2) * 32 + owner) * 4 + (j & 3)] = xbit ? -kCap : kCap;
            }
            sm->fst[r] = (uint8_t)Sr;
        }
        // 2. decided_u (:87), protection masks, event log (:91-92): lane t
        uint32_t myprot = 0u;
        if ((cmask >> lane) & 1u) {
            const int S = SL + lane;
            const int g = M - 1 - S, W = 1 << g;
            const int A = w.Al;
            const uint32_t xt = w.xl;
            const uint32_t wm = (1u << W) - 1u;
            const int o = A - w.A5;
            const uint32_t xb = (xt >> o) & wm, ub = (w.ul >> o) & wm;
            atomicAnd(&sm->dec_u[A >> 5], ~(wm << (A & 31)));
            atomicOr(&sm->dec_u[A >> 5], ub << (A & 31));
            const int owner = A / P, j0 = A % P;
            const int T = S + 1;
            if (T != M) {
                if ((SMEMM >> T) & 1u) {
                    const int ps = PL::NLR + __popc(SMEMM & ((1u << T) - 1u));
                    sm->pm[ps][owner] |= wm << j0;
                    myprot = 1u << ps;
                } else {  // register array in the last-pass layout
                    const int sl = __popc(REGM & ((1u << T) - 1u));
                    sm->pm[sl][owner] |= wm << j0;
                    sm->ss[sl][owner] = (sm->ss[sl][owner] & ~(wm << j0)) | (xb << j0);
                    myprot = 1u << sl;
                }
            }
            const int e_ix = nev + __popc(cmask & ((1u << lane) - 1u));
            if (a->events && e_ix < a->ev_cap) {
                int* e = a->events + ((long long)frame_ * a->ev_cap + e_ix) * 5;
                e[0] = it;
                e[1] = S;
                e[2] = A >> g;
                e[3] = A;
                e[4] = W;
            }
            if (XH && a->ev_xhat && e_ix < a->ev_cap)  // the block is <= 32 aligned rows
                atomicOr(&a->ev_xhat[((long long)frame_ * a->ev_cap + e_ix) * NW + (A >> 5)], xb << (A & 31));
        }
        prot |= __reduce_or_sync(kFull, myprot);
        nev += __popc(cmask);
    }

    // write W block bits of a pass layout (base bit b) into row-order words
    __device__ __forceinline__ void scatter(uint32_t* words, uint32_t bits, bool in_block, int b, int q, int W,
                                            int j0, int start) {
        if (b == 5) {
            // row = lane + 32 j : word j collects bit j of every lane
#pragma unroll 1
            for (int i = 0; i < W; ++i) {
                const uint32_t w = __ballot_sync(kFull, (bits >> i) & 1u);
                if (lane == 0) words[(start >> 5) + i] = w;
            }
        } else if (b == 0) {
            // row = P*lane + j : the block lives in one lane
            if (in_block) {
                const int row0 = P * lane + j0;
                const int off = row0 & 31;
                const uint32_t bm = (W >= 32) ? 0xffffffffu : ((1u << W) - 1u);
                words[row0 >> 5] = (words[row0 >> 5] & ~(bm << off)) | ((bits & bm) << off);
            }
        } else if (in_block) {
#pragma unroll 1
            for (int i = 0; i < W; ++i) {
                const int j = j0 + i;
                const int row = (lane & ((1 << b) - 1)) | (j << b) | ((lane >> b) << (b + K));
                if ((bits >> i) & 1u)
                    atomicOr(&words[row >> 5], 1u << (row & 31));
                else
                    atomicAnd(&words[row >> 5], ~(1u << (row & 31)));
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
            if constexpr (KIND != 0) xq = 0u;
            if constexpr (TM) {
                tm::ld_row<kTG>(tb + PL::C_R0, R);
                tm::wait_ld();
            } else {
#pragma unroll
                for (int c = 0; c < P / 4; ++c) {
                    const float4 v = r0g[c * 32 + lane];
                    R[4 * c] = v.x;
                    R[4 * c + 1] = v.y;
                    R[4 * c + 2] = v.z;
                    R[4 * c + 3] = v.w;
                }
            }
        } else if constexpr (first_of_pass) {
            x_load<q>(sm->X[q - 1], R);
        }
        if constexpr (PL::is_boundary(S + 1)) {
            PBP_T0(tr);
            if constexpr (KIND == 2)
                resaturate<PL::pass_of(S + 1)>();
            else
                __syncwarp();  // X holds other lanes' L(e) writes of the previous iteration
            PBP_T1(tr, 0);
        }
        PBP_T0(tm);
        float Lt[P];
        load_L<S + 1>(Lt);
        pe_stage<S>(Lt);
        store_L<S>(Lt);
        if constexpr (last_of_pass && S + 1 < M) x_store<q>(sm->X[q], R);
        if constexpr (first_of_pass || (last_of_pass && S + 1 < M)) __syncwarp();
        PBP_T1(tm, 0);
        if constexpr (KIND == 2) {
            PBP_T0(ts);
            if constexpr (S < PL::SL && TM) {
                tm::st_row<kTG>(tb + PL::C_S + 32u * S, R);  // R(S+1), pass-0 layout
                if constexpr (S == PL::SL - 1) {
                    PBP_T1(ts, 1);
                    PBP_T0(tw0);
                    walk0();
                    PBP_T1(tw0, 2);
                    return true;
                }
            } else if constexpr (S < PL::SL) {
                snapshot<S>();
                if constexpr (S == PL::SL - 1) walk_early();
            } else {
                snap_rows<S>();
            }
            PBP_T1(ts, 1);
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
    // TM csfg: R(m) of the last finished sweep, kept for the G-check and the
    // outputs while the next sweep's stage 0 runs (stage 4's snapshot columns:
    // walk0 has read them, stage 4 of the next sweep rewrites them)
    static constexpr uint32_t C_SAVE = PL::C_S + 128;
    __device__ __forceinline__ uint32_t signs_saved() const {
        tm::wait_st();  // the sweep's R(m) store
        uint32_t uq = 0u;
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            float v[8];
            tm::ld8(tb + C_SAVE + 8 * c, v);
            tm::wait_ld();
#pragma unroll
            for (int i = 0; i < 8; ++i) uq |= (__float_as_uint(v[i]) >> 31) << (8 * c + i);
        }
        return uq;
    }

    __device__ __forceinline__ uint32_t u_words(int pin, bool saved = false) {
        uint32_t uq;
        if constexpr (TM) uq = saved ? signs_saved() : pack_all();
        else uq = pack_all();
        uq &= ~FZ[Q - 1];
        if (pin > 0) {
            const int r0 = P * lane;
            int cnt = pin - r0;
            cnt = cnt < 0 ? 0 : (cnt > P ? P : cnt);
            const uint32_t pmk = cnt >= 32 ? 0xffffffffu : ((1u << cnt) - 1u);
            const uint32_t pmask = P >= 32 ? 0xffffffffu : ((1u << P) - 1u);
            const uint32_t db = (sm->dec_u[r0 >> 5] >> (r0 & 31)) & pmask;
            uq = (uq & ~pmk) | (db & pmk);
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

    // Pinned G-check (csfg_freeze.cpp:128-140, bp_core.cpp:104-110): x_hat of
    // stage 0 == polar_transform(u_hat'), u_hat' = u_hat with frozen rows 0
    // and rows < pin from decided_u. Exact filter first: the parity of x_hat
    // over each row class mod 32 (one bit per lane of the pass-0 layout) must
    // equal that of G(u_hat'), which is the in-word transform of u_hat' rows
    // 0..31 alone (a row i >= 32 lies above an even number of rows of each
    // class). Those rows are known without the sweep's R when they are all
    // frozen or decided; a mismatch proves x_hat != G(u_hat').
    __device__ __forceinline__ bool gcheck(int pin) {
        const uint32_t free0 = ~sm->frz[0] & ~low_mask(pin < 32 ? pin : 32);
        if (free0 == 0u) {
            const uint32_t cls = __ballot_sync(kFull, __popc(xq) & 1);
            const uint32_t u0 = pin > 0 ? sm->dec_u[0] & low_mask(pin < 32 ? pin : 32) : 0u;
            if (cls != word_transform(u0, 32)) return false;
        }
        return gcheck_full(pin);
    }

    __device__ __forceinline__ bool gcheck_full(int pin, bool saved = false, uint32_t xqv = 0u) {
        uint32_t uw = u_words(pin, saved);
        uw = word_transform(uw, 32);
#pragma unroll
        for (int h = 1; h < NW; h <<= 1) {
            const uint32_t o = __shfl_xor_sync(kFull, uw, h);
            if (!(lane & h)) uw ^= o;
        }
        const uint32_t xw = __shfl_sync(kFull, transpose32(saved ? xqv : xq, lane), xperm);
        return !__any_sync(kFull, lane < NW && uw != xw);
    }

    // gcheck's exact filter without a branch: false proves x_hat != G(u_hat')
    __device__ __forceinline__ bool gfilter(int pin, uint32_t xqv) {
        const uint32_t free0 = ~sm->frz[0] & ~low_mask(pin < 32 ? pin : 32);
        const uint32_t cls = __ballot_sync(kFull, __popc(xqv) & 1);
        const uint32_t u0 = pin > 0 ? sm->dec_u[0] & low_mask(pin < 32 ? pin : 32) : 0u;
        return free0 != 0u || cls == word_transform(u0, 32);
    }

    // the last-pass commits and the PE count of the sweep that ended (a no-op
    // when cm = 0 and !live): run inside the next sweep's stage 0
    __device__ __forceinline__ void book_tail(const LateTM& w, int dinact, bool live) {
        apply_tm(w, dinact);
        if (lane < M) inact += dinact;
        const int v = (live && lane <= s_last_) ? (N >> 1) - inact : 0;
        act += __reduce_add_sync(kFull, v);
    }

    // n = 1024 csfg decode of one frame, software-pipelined: after sweep t the
    // last-pass walk, the first-pass commits and the register fix-up run at
    // once (sweep t+1's stages read their results); apply_freeze of the
    // last-pass commits, the PE count and the G-check filter of sweep t run in
    // the same straight-line block as sweep t+1's stage 0, which reads none of
    // what they write (R(0), L(1) against L(6..10), freeze state, decided_u),
    // so their latency chains hide under its PE math. When the G-check finds
    // sweep t converged, the speculative stage 0 is dropped (R(m) and x_hat of
    // sweep t are kept in TMEM / a register for the check and the outputs).
#ifndef PBP_PIPE
#define PBP_PIPE 1
#endif
    static constexpr int kPipe = PBP_PIPE;  // stages of the next sweep the book-keeping overlaps
    static_assert(kPipe >= 1 && kPipe <= 4, "stages 0..3 only (walk0 runs at stage 4)");
    __device__ __forceinline__ void decode_tm_csfg(int& iters, int& stop, uint32_t& uw) {
        const DecodeArgs& args = *a;
        iters = 0;
        bool converged = false, pend = false;
        // the first book_tail (nothing pending) reads the walk state before any walk0
        // has set it: uniform values, or the warp's collectives would diverge on
        // uninitialised registers
        nce_ = 0;
        fr_start_ = 0;
        s_last_ = -1;
        done_ = false;
        LateTM w;
        w.cm = 0u;
        w.A5 = 0;
        w.u = 0u;
        w.xl = 0u;
        w.Al = 0;
#pragma unroll
        for (int t = 0; t < PL::NL; ++t) {
            w.x[t] = 0u;
            w.At[t] = 0;
        }
        int dpend = 0;
        uint32_t xqp = 0u;
#pragma unroll 1
        for (int t = 1; t <= args.max_iter; ++t) {
            it = t - 1;  // events of the pending commits carry their own iteration
            PBP_DBG(1);
            book_tail(w, dpend, pend);
            const bool full = pend && gfilter(frontier, xqp);
            it = t;
            PBP_DBG(2);
            // stages 0 .. kPipe-1 of sweep t read none of the pending book-keeping's
            // results (only walk0, at stage 4, needs the new frontier)
            stage<0>();
            if constexpr (kPipe > 1) stage<1>();
            if constexpr (kPipe > 2) stage<2>();
            if constexpr (kPipe > 3) stage<3>();
            PBP_DBG(3);
            if (pend) {
                pend = false;
                if (full) converged = gcheck_full(frontier, true, xqp);
                if (converged) break;  // the frame ended with sweep t-1
            }
            iters = t;
            sweep_from<kPipe>();
            PBP_DBG(4);
            tm::st_row<kTG>(tb + C_SAVE, R);  // R(m) of sweep t
            xqp = xq;
            walk_tm(w);
            PBP_DBG(5);
            dpend = nce_ ? apply_early_tm() : 0;
            if (prot & ((1u << PL::NLR) - 1u)) fixup_regs();
            __syncwarp();
            pend = true;
            if (done_) break;  // the frontier reached n: no G-check
            w.cm = w.cm;  // keep w live across the loop edge
        }
        PBP_DBG(6);
        if (pend) {  // the last sweep's commits and count; its G-check when the frontier is < n
            it = iters;
            book_tail(w, dpend, true);
            if (!done_) converged = gfilter(frontier, xqp) && gcheck_full(frontier, true, xqp);
        }
        PBP_DBG(7);
        stop = frontier >= N ? 2 : (converged ? 1 : 0);
        if (frontier >= N) uw = lane < NW ? sm->dec_u[lane] : 0u;
        else uw = u_words(frontier, iters > 0);
        PBP_DBG(8);
    }

    __device__ __forceinline__ void run(const DecodeArgs& args, Smem* s, int ln) {
        a = &args;
        r0g = TM ? nullptr : reinterpret_cast<float4*>(args.r0s) + (long long)blockIdx.x * (N / 4);
        sm = s;
        lane = ln;
        alpha = args.alpha;
        fz_init<0>();
        if (lane < NW) sm->frz[lane] = a->frozen_bits[lane];
        if constexpr (TM) {
            // L(m) at frame start: +CAP at frozen rows (bp_core.cpp:53), last-pass layout
            const uint32_t fl = FZ[Q - 1];
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = ((fl >> j) & 1u) ? kCap : 0.f;
            tm::st_row<kTG>(tb + PL::C_LM0, R);
            tm::wait_st();
        }
        // stage 0 pushes x_hat bits of rows (lane + 32 j) in the order
        // j = j0, j0+1, j0+d, j0+d+1 for j0 = 0, 2, ... (d = P/2); the first push
        // lands in bit 31. xperm = bit position that holds row-order word `lane`.
        {
            const int j = lane;
            constexpr int d = P / 2;
            const int hi = (j >= d) ? 1 : 0;
            const int jj = j - hi * d;
            const int p = 4 * (jj >> 1) + 2 * hi + (jj & 1);  // push index
            xperm = P - 1 - p;
        }
        if (lane < kNumCounters) sm->cnt[lane] = 0ull;
        cset_ = 0;
        __syncwarp();

        for (;;) {
            long long f = 0;
            if (lane == 0) f = (long long)atomicAdd(args.queue, 1ull);
            f = __shfl_sync(kFull, f, 0);
            if (f >= args.frames) break;
            frame_ = f;
            PBP_T0(tf);
            if (!load_frame(f)) {
                if (lane == 0) {
                    const unsigned long long slot = atomicAdd(args.list_len, 1ull);
                    args.list[slot] = f + args.frame_base;
                }
                continue;
            }
            init_frame();
            PBP_T1(tf, 6);
            PBP_T0(tl);
            int iters = (KIND == 0) ? args.max_iter : 0;
            int stop = 0;
            bool converged = false;
#ifndef PBP_NO_PIPELINE
            if constexpr (TM && KIND == 2) {
                uint32_t uwp;
                decode_tm_csfg(iters, stop, uwp);
                PBP_T1(tl, 7);
                write_outputs(f, uwp, iters, stop);
                continue;
            }
#endif
#pragma unroll 1
            for (int t = 1; t <= args.max_iter; ++t) {
                if constexpr (KIND == 2) {
                    if (frontier >= N || converged) break;
                    iters = t;
                }
                it = t;
                sweep_from<0>();
                if constexpr (KIND == 2) {
                    if (finish_iter()) {
                        PBP_T0(tg);
                        converged = gcheck(frontier);
                        PBP_T1(tg, 5);
                    }
                } else {
                    act += (long long)M * (N >> 1);
                }
                if constexpr (KIND == 1) {
                    if (gcheck(0)) {
                        iters = t;
                        stop = 1;
                        break;
                    }
                }
            }
            PBP_T1(tl, 7);
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
            write_outputs(f, uw, iters, stop);
        }
        if (args.counters && lane < kNumCounters && sm->cnt[lane])
            atomicAdd(&args.counters[cset_ * kNumCounters + lane], sm->cnt[lane]);
#ifdef PBP_PROF_SECTIONS
        if (lane == 0)
            for (int i = 0; i < 8; ++i) atomicAdd(&g_prof[i], prof[i]);
#endif
    }

    __device__ __forceinline__ void write_outputs(long long f, uint32_t uw, int iters, int stop) {
        const DecodeArgs& args = *a;
        if (args.u_bits && lane < NW) args.u_bits[f * NW + lane] = uw;
        if (lane == 0) {
            if (args.iters) args.iters[f] = iters;
            if (args.pe) args.pe[f] = act;
            if (args.stop) args.stop[f] = (uint8_t)stop;
            if (args.nev) args.nev[f] = nev;
        }
        if (args.counters) {
            int be = 0;
            if (lane < NW) be = __popc((uw ^ args.truth_u[f * NW + lane]) & ~args.frozen_bits[lane]);
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
            // a warp's frames come from the queue in increasing order: accumulate
            // locally while they stay in one counter set, flush when the set changes
            if (args.cnt_batch > 0) {
                const long long set = f / args.cnt_batch;
                if (set != cset_) {
                    if (lane < kNumCounters && sm->cnt[lane]) {
                        atomicAdd(&args.counters[cset_ * kNumCounters + lane], sm->cnt[lane]);
                        sm->cnt[lane] = 0ull;
                    }
                    cset_ = set;
                }
            }
            if (lane < kNumCounters) sm->cnt[lane] += v;
        }
    }

    // LLRs -> lane-private pass-0 layout; false when the frame needs the
    // generic kernel (|LLR| beyond the clamp-free bound or non-finite)
    __device__ __forceinline__ bool load_frame(long long f) {
        const float4* src = reinterpret_cast<const float4*>(a->llr + f * (long long)N);
        bool bad = false;
        float* r0 = sm->X[0];  // staging (X is re-initialised after the frame load)
#pragma unroll 4
        for (int i = 0; i < P / 4; ++i) {
            const float4 v = __ldcs(src + lane + 32 * i);
            const float e[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                bad |= !(fabsf(e[k]) <= kClampFreeBound);
                const int row = 4 * (lane + 32 * i) + k;  // row -> (lane', j) of pass 0
                const int l2 = row & 31, j = row >> 5;
                r0[((j >> 2) * 32 + l2) * 4 + (j & 3)] = __fadd_rn(e[k], 0.0f);  // -0 -> +0
            }
        }
        __syncwarp();
        // each lane keeps its own slots: it is the only reader (stage 0)
        if constexpr (TM) {
#pragma unroll
            for (int c = 0; c < P / 4; ++c) {
                const float4 t = reinterpret_cast<const float4*>(r0)[c * 32 + lane];
                R[4 * c] = t.x;
                R[4 * c + 1] = t.y;
                R[4 * c + 2] = t.z;
                R[4 * c + 3] = t.w;
            }
            tm::st_row<kTG>(tb + PL::C_R0, R);
            tm::wait_st();
        } else {
#pragma unroll
            for (int c = 0; c < P / 4; ++c) r0g[c * 32 + lane] = reinterpret_cast<const float4*>(r0)[c * 32 + lane];
        }
        __syncwarp();  // X is overwritten next
        return !__any_sync(kFull, bad);
    }

    template <int q>
    __device__ __forceinline__ void fz_init() {
        uint32_t w = 0u;
#pragma unroll 1
        for (int j = 0; j < P; ++j) w |= (uint32_t)(a->frozen_rows[row_of<q>(j)] != 0) << j;
        FZ[q] = w;
        sm->fz[q][lane] = w;
        if constexpr (q + 1 < Q) fz_init<q + 1>();
    }

    __device__ __forceinline__ void init_frame() {
        init_smem();
#pragma unroll
        for (int j = 0; j < P; ++j) R[j] = 0.f;  // R(m) = 0 until the first sweep (max_iter = 0)
#pragma unroll
        for (int sl = 0; sl < PL::NLR; ++sl)
#pragma unroll
            for (int j = 0; j < P; ++j) Lr[sl][j] = 0.f;
        frontier = 0;
        inact = 0;
        nev = 0;
        act = 0;
        prot = 0u;
        xq = 0u;
    }

    __device__ __forceinline__ void init_smem() {
#pragma unroll 1
        for (int sl = 0; sl < PL::NLS; ++sl)
#pragma unroll 1
            for (int c = 0; c < P / 4; ++c) sm->Ls[sl][c][lane] = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll 1
        for (int x = 0; x < Q - 1; ++x)
#pragma unroll 1
            for (int i = lane; i < PL::NX; i += 32) sm->X[x][i] = 0.f;
        // L(m): +CAP at frozen rows (bp_core.cpp:53), last-pass layout
        if constexpr (TM) {
            // copied from the warp's pristine L(m) columns (written once in
            // run(): computing the 32 values here lets the compiler hoist them
            // out of the frame loop, 32 registers live across the decode);
            // R is the staging register set (init_frame zeroes it afterwards)
            tm::ld_row<kTG>(tb + PL::C_LM0, R);
            tm::wait_ld();
            tm::st_row<kTG>(tb + PL::C_LM, R);
            tm::wait_st();
        } else if constexpr (KIND == 2) {
            sm->lmz[lane] = FZ[Q - 1];
            sm->lmn[lane] = 0u;
        } else {
            const uint32_t fl = FZ[Q - 1];
#pragma unroll 1
            for (int c = 0; c < P / 4; ++c)
                sm->LM[c][lane] = make_float4(((fl >> (4 * c)) & 1u) ? kCap : 0.f, ((fl >> (4 * c + 1)) & 1u) ? kCap : 0.f,
                                              ((fl >> (4 * c + 2)) & 1u) ? kCap : 0.f,
                                              ((fl >> (4 * c + 3)) & 1u) ? kCap : 0.f);
        }
        if (lane < NW) sm->dec_u[lane] = 0u;
        if (TM && lane < 5) sm->skipm[lane] = 0u;
#pragma unroll 1
        for (int x = 0; x < Q - 1; ++x)
            if (lane < NW) sm->xprot[x][lane] = 0u;
#pragma unroll 1
        for (int sl = 0; sl < PL::NLR + PL::NLS; ++sl) sm->pm[sl][lane] = 0u;
#pragma unroll 1
        for (int i = lane; i < N / 4; i += 32) reinterpret_cast<uint32_t*>(sm->fst)[i] = 0x7f7f7f7fu;
        __syncwarp();
    }
};

// resident warps per SM the register budget is sized for (per 16K-register
// SM partition: 2 warps at <= 256 registers, 3 at <= 168, 5 at <= 102;
// n = 256 measured +2.6 % for csfg at 20 warps over 16 despite a small spill)
template <int M>
constexpr int kMinWarps = M >= 10 ? 1 : (M == 9 ? 12 : 20);

// CTA-shared shared memory after the warps' own: walk0's frozen-field table (n = 1024 csfg)
template <int M, int KIND>
constexpr size_t extra_smem() { return (Plan<M>::TM && KIND == 2) ? 32 * 32 * sizeof(uint32_t) : 0; }

// n = 1024: eight warps (frames) per CTA, one CTA per SM, so the CTA's TMEM
// allocation (all 512 columns) gives each warp 256 columns of its lane quarter
template <int M, int KIND, bool XH = false>
__global__ void __launch_bounds__(32 * Plan<M>::WARPS, Plan<M>::TM ? 1 : kMinWarps<M>) bp_warp_kernel(DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char wsm[];
    using D = Dec<M, KIND, XH>;
    D dec;
    if constexpr (Plan<M>::TM) {
        __shared__ uint32_t tbase;
        const int warp = threadIdx.x >> 5;
        if (warp == 0) tm::alloc512(&tbase);
        if constexpr (KIND == 2) {
            // walk0's frozen-row fields for every frontier word jf (pass-0 layout, bit j of
            // fz0 = row lane + 32 j): blocks of 16, 8, 4, 2, 1 words at offsets 0, 16, 24, 28, 30
            uint32_t* t = reinterpret_cast<uint32_t*>(reinterpret_cast<typename D::Smem*>(wsm) + Plan<M>::WARPS);
            for (int i = threadIdx.x; i < 32 * 32; i += blockDim.x) {
                const int jf = i >> 5, ln = i & 31;
                uint32_t fz0 = 0u;
                for (int j = 0; j < 32; ++j) fz0 |= (uint32_t)(a.frozen_rows[ln + 32 * j] != 0) << j;
                t[i] = ((fz0 >> (jf & ~15)) & 0xFFFFu) | (((fz0 >> (jf & ~7)) & 0xFFu) << 16) |
                       (((fz0 >> (jf & ~3)) & 0xFu) << 24) | (((fz0 >> (jf & ~1)) & 3u) << 28) |
                       (((fz0 >> jf) & 1u) << 30);
            }
        }
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        dec.tb = tm::warp_base(tbase, warp);
        dec.fzt = reinterpret_cast<const uint32_t*>(reinterpret_cast<typename D::Smem*>(wsm) + Plan<M>::WARPS);
        dec.run(a, reinterpret_cast<typename D::Smem*>(wsm) + warp, threadIdx.x & 31);
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        if (warp == 0) tm::dealloc512(tbase);
    } else {
        dec.run(a, reinterpret_cast<typename D::Smem*>(wsm), threadIdx.x & 31);
    }
}

}  // namespace wk

int warp_kernel_supported(int m) { return m >= 7 && m <= 10; }
// warps (frames) per CTA of the warp kernel: eight at n = 1024 (TMEM), else one
int warp_kernel_warps(int m) { return m == 10 ? wk::Plan<10>::WARPS : 1; }

size_t warp_smem_bytes(int m, int kind) {
    const bool b = kind == 2;
    switch (m) {
        case 7: return b ? sizeof(wk::WarpSmem<7, true>) : sizeof(wk::WarpSmem<7>);
        case 8: return b ? sizeof(wk::WarpSmem<8, true>) : sizeof(wk::WarpSmem<8>);
        case 9: return b ? sizeof(wk::WarpSmem<9, true>) : sizeof(wk::WarpSmem<9>);
        case 10: return b ? sizeof(wk::WarpSmem<10, true>) : sizeof(wk::WarpSmem<10>);
    }
    return 0;
}

template <int M, int KIND, bool XH>
static cudaError_t launch_wx(const DecodeArgs& a, int grid, cudaStream_t st) {
    constexpr int W = wk::Plan<M>::WARPS;
    const size_t smem = W * sizeof(typename wk::Dec<M, KIND, XH>::Smem) + wk::extra_smem<M, KIND>();
    cudaError_t e = cudaFuncSetAttribute(wk::bp_warp_kernel<M, KIND, XH>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    wk::bp_warp_kernel<M, KIND, XH><<<grid, 32 * W, smem, st>>>(a);
    return cudaGetLastError();
}

template <int M, int KIND>
static cudaError_t launch_w(const DecodeArgs& a, int grid, cudaStream_t st) {
    if constexpr (KIND == 2) {
        if (a.ev_xhat) return launch_wx<M, KIND, true>(a, grid, st);  // trace with x_hat
    }
    return launch_wx<M, KIND, false>(a, grid, st);
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

template <int M, int KIND>
static int occ_w() {
    int nb = 0;
    constexpr int W = wk::Plan<M>::WARPS;
    const size_t smem = W * sizeof(typename wk::Dec<M, KIND>::Smem) + wk::extra_smem<M, KIND>();
    cudaFuncSetAttribute(wk::bp_warp_kernel<M, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, wk::bp_warp_kernel<M, KIND>, 32 * W, smem) != cudaSuccess)
        return 0;
    return nb;
}

template <int M>
static int occ_m(int kind) {
    return kind == 0 ? occ_w<M, 0>() : kind == 1 ? occ_w<M, 1>() : occ_w<M, 2>();
}

int warp_blocks_per_sm(int m, int kind) {
    switch (m) {
        case 7: return occ_m<7>(kind);
        case 8: return occ_m<8>(kind);
        case 9: return occ_m<9>(kind);
        case 10: return occ_m<10>(kind);
    }
    return 0;
}

}  // namespace pbp
