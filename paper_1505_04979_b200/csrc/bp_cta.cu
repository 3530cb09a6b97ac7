// CTA-per-frame BP decoder for n = 2048 .. 16384 (configs 3 and 4).
//
// The reference schedule (src/bp_core.cpp:58-86, csfg_freeze.cpp:99-152):
// every stage's PEs under the is_pe_active mask (inactive PEs keep their
// state), at most one candidate check/commit per stage in stage order, and
// the pinned G-check after each sweep. What is B200-specific is where the
// state lives and when the checks run:
//
// * T threads own P = n/T rows each (one frame per CTA; three CTAs per SM at
//   n = 2048, two at 4096, one beyond). A pass is K = log2 P consecutive stages
//   whose PE distances are register bits of the thread's rows, so R(s) is
//   carried in registers from stage to stage and crosses shared memory
//   (Rx) only between passes.
// * L(s) for a stage s inside a pass is produced and consumed by the same
//   thread (stage s writes it, stage s-1 reads it, both in the pass's row
//   layout): those levels live in registers, or where registers run out in
//   shared memory or as thread-major (coalesced) L2 arrays. Levels at pass
//   boundaries are exchanged between layouts in row-indexed shared memory
//   (L2 for some at n >= 8192); L(m) in {0, +-CAP} is two bit masks.
// * csfg checks are deferred to the end of each pass: its stages run as if
//   none of its checks commits; then one batched polar transform of the
//   stages' hard decisions (csfg_freeze.cpp:18-39: register bits in-thread,
//   lane bits by shuffles, warp bits by one shared-memory superset XOR) and
//   one OR-reduction decide every candidate for every frontier an earlier
//   commit of the pass can produce, and the commits (apply_freeze,
//   csfg_freeze.cpp:82-93) are applied in stage order by the owners of the
//   block's rows, with the PE count corrected for the PEs the reference
//   would have skipped. Rows of a committed block pair only with each other
//   at later stages, so their speculative values are never observed.
//   Frontier and event count are uniform registers.
//
// Arithmetic as in the warp-resident kernel (one min.xorsign.abs per
// min-with-sign, every product and sum rounded on its own, r_top =
// fma(alpha, m, +0) so R is never -0); frames with |LLR| beyond the
// clamp-free bound or non-finite are re-routed to the generic kernel, which
// keeps every clamp.
//
// Levels that the register file cannot hold live in tensor memory where the
// layout allocates it (thread-private levels: one tcgen05.ld/st of P columns
// per stage): n = 4096 at two CTAs per SM (256 columns each; the occupancy
// API reports one CTA per SM for a TMEM kernel, but CTAs whose columns fit the
// SM's 512 co-reside), n = 8192 and 16384 at one. R(0) stays in TMEM where a
// column slot is free.
//
// n = 16384 csfg runs as a 2-CTA thread-block cluster per frame (SP = true,
// bp_pair_kernel): each CTA holds half of the frame in the n = 8192 layout on
// its own SM, so every level is on chip; only the frame's stage 0 couples the
// halves (row r of both halves at the same thread of both CTAs: one term per
// row through distributed shared memory per sweep), the half holding the
// frontier checks the candidates (the first CTA posts its frontier to the
// second), and the pinned G-check splits along the transform's top level with
// one cluster barrier per iteration.
#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "pbp_common.cuh"
#include "tmem.cuh"

namespace pbp {
namespace cta {

constexpr unsigned kFull = 0xffffffffu;
// kTmem: a thread-private (inner) level in tensor memory: the thread's P rows are
// P columns of its TMEM lane (one tcgen05.ld/st per stage instead of P L2 accesses)
enum : int { kReg = 0, kSmem = 1, kGlob = 2, kBits = 3, kTmem = 4 };

// Per-size plan: threads (LOGT), rows per thread (2^K), where each L level
// lives, whether R(0) stays in registers, whether Rx is double-buffered.
template <int M, bool SP = false>
struct Cfg;
template <>
struct Cfg<11> {  // 128 threads x 16 rows, 3 CTAs per SM: four levels in registers, the rest in shared memory
    static constexpr int LOGT = 7, K = 4, MINB = 3;
    static constexpr bool r0reg = false, rx2 = false;
    static constexpr int TMEM_COLS = 0;
    static constexpr int where(int s) { return s == 11 ? kBits : (s <= 3 || s == 5) ? kReg : kSmem; }
};
template <>
struct Cfg<12> {  // 256 x 16, two frames per SM, every level on chip: three in registers, two in shared memory, six in TMEM
    static constexpr int LOGT = 8, K = 4, MINB = 2;
    // rx2: the pass-boundary R exchange double-buffered (no barrier before its
    // stores; measured +0.6 % csfg at n = 4096, +2.5 % at n = 8192)
    static constexpr bool r0reg = false, rx2 = true;
    // 256 columns per CTA: two CTAs per SM share the 512 (the occupancy API reports one
    // CTA per SM for a kernel that allocates TMEM; a grid of two per SM co-resides:
    // cta_blocks_per_sm). Against levels 6..9 in shared memory and 10, 11 in L2: +3 %.
    static constexpr int TMEM_COLS = 256;
    static constexpr bool TPROT_REG = false;
    static constexpr bool PACK(int kind) { return kind != 2; }
    // level 5 in TMEM too (16 registers freed: +1.8 % csfg, +3.6 % G-stop over registers)
    // (level 3 in TMEM as well measured 1.4 % slower here)
    static constexpr int where(int s) { return s == 12 ? kBits : (s <= 3) ? kReg : (s == 4 || s == 8) ? kSmem : kTmem; }
};
#if 0  // round-1 layout (two levels in L2)
template <>
struct Cfg<12> {  // 256 x 16, two frames per SM: four levels in registers, five in shared memory, two in L2
    static constexpr int LOGT = 8, K = 4, MINB = 2;
    static constexpr bool r0reg = false, rx2 = false;
    // no TMEM: a kernel that allocates tensor memory gets one CTA per SM
    // (tools/micro/tmem_occupancy.cu), and n = 4096 needs two frames per SM
    static constexpr int TMEM_COLS = 0;
    static constexpr int where(int s) {
        return s == 12 ? kBits : (s <= 3 || s == 5) ? kReg : (s == 10 || s == 11) ? kGlob : kSmem;
    }
};
#endif
template <>
struct Cfg<13> {  // 512 x 16: two levels in registers, three in shared memory, seven in TMEM (all on chip)
    static constexpr int LOGT = 9, K = 4, MINB = 1;
    // rx2: the pass-boundary R exchange double-buffered (no barrier before its
    // stores; measured +0.6 % csfg at n = 4096, +2.5 % at n = 8192)
    static constexpr bool r0reg = false, rx2 = true;
    static constexpr int TMEM_COLS = 512;  // 16 warps: 128 columns of its lane quarter per warp
    static constexpr bool TPROT_REG = false;
    static constexpr bool PACK(int) { return true; }
    // every inner level from 3 on in TMEM (5 and 6 in shared memory measured 1.8 % slower,
    // level 3 in registers 2.4 % slower)
    static constexpr int where(int s) { return s == 13 ? kBits : (s <= 2) ? kReg : (s % 4 == 0) ? kSmem : kTmem; }
};
template <>
struct Cfg<14> {  // 1024 x 16: one level in shared memory, four in TMEM, the rest in L2
    static constexpr int LOGT = 10, K = 4, MINB = 1;
    static constexpr bool r0reg = false, rx2 = false;
    static constexpr int TMEM_COLS = 512;  // 32 warps: 64 columns per warp = four levels
    static constexpr bool TPROT_REG = false;
    // L(12) joins two layouts with lane strides > 1 row (uncoalesced in L2); the TMEM
    // levels are inner levels whose blocks freeze rarely (first-pass stages), so their
    // boundary fix-up after the sweep seldom runs; 148 frames x 8 L2 levels fit the L2
    static constexpr int where(int s) {
        return s == 14 ? kBits : (s == 12) ? kSmem : (s == 1 || s == 2 || s == 3 || s == 5) ? kTmem : kGlob;
    }
};

// SP (split pair): one CTA of a 2-CTA cluster holding half of a frame of
// length 2^(M+1): its local stages 0..M-1 are the frame's stages 1..M, the
// frame's stage 0 (distance 2^M) is the cross stage between the pair.
template <>
struct Cfg<13, true> {  // half of n = 16384: 512 x 16, one CTA per SM; inner levels 5..11 in TMEM, L(1) of the frame too
    static constexpr int LOGT = 9, K = 4, MINB = 1;
    static constexpr bool r0reg = false, rx2 = false;
    static constexpr int TMEM_COLS = 512;  // 16 warps: 128 columns per warp = six levels + L(1) of the frame
    static constexpr bool TPROT_REG = false;
    static constexpr int where(int s) { return s == 13 ? kBits : (s <= 3) ? kReg : (s % 4 == 0) ? kSmem : kTmem; }
};

template <>
struct Cfg<11, true> {  // half of n = 4096 (A/B experiment, PBP_PAIR=2): the n = 2048 layout, L(1) of the frame in registers
    static constexpr int LOGT = 7, K = 4, MINB = 2;
    static constexpr bool r0reg = false, rx2 = false;
    static constexpr int TMEM_COLS = 0;
    static constexpr bool L0REG = true;
    static constexpr int where(int s) { return s == 11 ? kBits : (s <= 3 || s == 5) ? kReg : kSmem; }
};

template <class C, typename = void>
struct L0Reg { static constexpr bool value = false; };
// packed fp32x2 PE math per layout and decoder (PACK(kind)); scalar where the
// packed pairs' register pressure spills (measured: n = 8192 +2.5 %, n = 4096
// G-stop +5.5 %, n = 4096 csfg -0.8 %, the pair -2.9 %, n = 16384 G-stop -10 %)
template <class C, typename = void>
struct Pack { static constexpr bool on(int) { return false; } };
template <class C>
struct Pack<C, std::void_t<decltype(C::PACK(0))>> { static constexpr bool on(int kind) { return C::PACK(kind); } };
template <class C>
struct L0Reg<C, std::void_t<decltype(C::L0REG)>> { static constexpr bool value = C::L0REG; };

template <int M_, bool SP_ = false>
struct Plan {
    using C = Cfg<M_, SP_>;
    static constexpr bool SP = SP_;
    static constexpr int M = M_;
    static constexpr int N = 1 << M;
    static constexpr int LOGT = C::LOGT;
    static constexpr int T = 1 << LOGT;
    static constexpr int NWARP = T / 32;
    static constexpr int K = C::K;
    static constexpr int P = 1 << K;
    static constexpr int Q = (M + K - 1) / K;
    static constexpr int NW = N / 32;
    static_assert(K + LOGT == M, "rows per thread x threads = n");
    static_assert(P <= 16, "a thread's rows are a sub-word group");
    static_assert(M - K >= 5, "pass 0 keeps row bits [0, 5) in the lane index");
    // pass q: register j holds row bits [b, b+K); thread bits fill the rest
    static constexpr int base(int q) { return (M - K * (q + 1)) > 0 ? (M - K * (q + 1)) : 0; }
    static constexpr int last(int q) { return ((q + 1) * K < M ? (q + 1) * K : M) - 1; }
    static constexpr int pass_of(int s) { return s / K; }
    static constexpr int count(int kind, int below) {
        int c = 0;
        for (int s = 1; s < below; ++s) c += C::where(s) == kind;
        return c;
    }
    static constexpr int slot(int s) { return count(C::where(s), s); }
    static constexpr int NREG = count(kReg, M + 1), NSM = count(kSmem, M + 1), NGL = count(kGlob, M + 1);
    static constexpr int NTM = count(kTmem, M + 1);
    // TMEM: each warp owns TMEM_COLS * 4 / NWARP columns of its lane quarter, P per level
    static constexpr int TM_WCOLS = C::TMEM_COLS > 0 ? C::TMEM_COLS * 4 / NWARP : 0;
    // SP: the frame's L(1) (local L(0), thread-private in pass 0's layout) in TMEM slot NTM
    // (L0T), else in registers
    static constexpr bool L0T = SP && !L0Reg<C>::value;
    // (with L0T, this half's R(0) in TMEM slot NTM + 1)
    static constexpr int L0S = NTM, R0S = NTM + 1;
    // one CTA per frame: R(0) in TMEM slot NTM when a TMEM layout has the columns
    // (one tcgen05.ld per sweep instead of P global loads)
    static constexpr bool R0T = !SP && NTM > 0 && (NTM + 1) * P <= TM_WCOLS;
    static constexpr bool TMEM = NTM > 0 || L0T;
    static constexpr bool tm_ok() {
        for (int s = 1; s <= M; ++s)
            if (C::where(s) == kTmem && !(s < M && s / K == (s - 1) / K)) return false;  // inner levels only
        return (NTM + (L0T ? 2 : 0)) * P <= TM_WCOLS || !TMEM;
    }
    static_assert(tm_ok(), "TMEM levels: thread-private (inner) levels that fit the warp's columns");
    static constexpr int pad(int row) { return row + (row >> 5); }
    static constexpr int NX = N + N / 32;
    // L(s) is produced (stage s) and consumed (stage s-1, commits of stage
    // s-1) in one pass layout: only its owner threads touch it
    static constexpr bool inner(int s) { return s < M && pass_of(s) == pass_of(s - 1); }
};

__device__ __forceinline__ float xsmin(float a, float b) {
    float d;
    asm("min.xorsign.abs.f32 %0, %1, %2;" : "=f"(d) : "f"(a), "f"(b));
    return d;
}

// packed fp32x2 arithmetic (FADD2 / FFMA2), round-to-nearest per half
__device__ __forceinline__ void add2(float& d0, float& d1, float a0, float a1, float b0, float b1) {
    asm("{ .reg .b64 a, b, d; mov.b64 a, {%2, %3}; mov.b64 b, {%4, %5}; add.rn.f32x2 d, a, b; mov.b64 {%0, %1}, d; }"
        : "=f"(d0), "=f"(d1) : "f"(a0), "f"(a1), "f"(b0), "f"(b1));
}
// s * a + (+0): the single-rounded product, never -0
__device__ __forceinline__ void fma2s0(float& d0, float& d1, float s, float a0, float a1) {
    asm("{ .reg .b64 a, b, c, d; mov.b64 a, {%2, %2}; mov.b64 b, {%3, %4}; mov.b64 c, 0; "
        "fma.rn.f32x2 d, a, b, c; mov.b64 {%0, %1}, d; }"
        : "=f"(d0), "=f"(d1) : "f"(s), "f"(a0), "f"(a1));
}

// thread-block cluster (SP pair): rank, barrier, distributed shared memory
__device__ __forceinline__ int cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return (int)r;
}
__device__ __forceinline__ void cluster_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }
__device__ __forceinline__ void cluster_sync() {
    cluster_arrive();
    cluster_wait();
}
// cluster window address of the same shared-memory object in CTA `rank`
__device__ __forceinline__ uint32_t cluster_map(const void* p, int rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"((uint32_t)__cvta_generic_to_shared(p)), "r"(rank));
    return r;
}
__device__ __forceinline__ void st_peer(uint32_t addr, uint32_t v) {
    asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t addr, int v) {
    asm volatile("st.shared::cluster.s32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t addr, float v) {
    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t addr, long long v) {
    asm volatile("st.shared::cluster.s64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ void st_peer(uint32_t addr, unsigned long long v) {
    asm volatile("st.shared::cluster.u64 [%0], %1;" ::"r"(addr), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_volatile(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"((uint32_t)__cvta_generic_to_shared(p)) : "memory");
    return v;
}

// bit i (i & h == 0) absorbs bit i + h for h < 2^NB: the in-thread levels of
// the polar transform (polar_code.cpp:13-20) over a thread's register rows
template <int NB>
__device__ __forceinline__ uint32_t bits_transform(uint32_t w) {
    if constexpr (NB > 0) w ^= (w >> 1) & 0x5555u;
    if constexpr (NB > 1) w ^= (w >> 2) & 0x3333u;
    if constexpr (NB > 2) w ^= (w >> 4) & 0x0F0Fu;
    if constexpr (NB > 3) w ^= (w >> 8) & 0x00FFu;
    return w;
}

template <class C, typename = void>
struct TprotReg { static constexpr bool value = false; };
template <class C>
struct TprotReg<C, std::void_t<decltype(C::TPROT_REG)>> { static constexpr bool value = C::TPROT_REG; };

template <int M, bool SP = false>
struct Smem {
    using PL = Plan<M, SP>;
    using C = Cfg<M, SP>;
    float Ls[PL::NSM > 0 ? PL::NSM : 1][PL::NX];  // shared-memory L levels, row-indexed (padded)
    float Rx[C::rx2 ? 2 : 1][PL::NX];         // R at pass boundaries
    typename std::conditional<(PL::Q * PL::P > 32), unsigned long long, uint32_t>::type buf[PL::T];  // cross-warp words
    uint32_t vw[3];                                // verdict words of the pass checks
    uint32_t dec[PL::NW];                          // decided_u
    uint32_t xh[PL::NW];                           // x_hat = (R(0) + L(0) < 0) of the last sweep
    uint8_t fst[PL::N];                            // freeze_stage per row
    long long frame;
    // TMEM levels: per thread and level, rows whose L is a frozen-block boundary
    // (bits 0..P-1) and their signs (bits 16..16+P-1), restored after each sweep
    uint32_t tprot[(PL::NTM > 0 && !TprotReg<C>::value) ? PL::NTM : 1][(PL::NTM > 0 && !TprotReg<C>::value) ? PL::T : 1];
    uint32_t tbase;                                // TMEM allocation
    // SP: what the peer CTA of the pair writes here (st.shared::cluster)
    // double-buffered by iteration parity: the peer writes sweep t's while this CTA may still read t-1's
    // the peer's stage-0 term at pass-0 thread positions: from the first CTA
    // alpha * min-with-sign(L(1), R(0)) (the PE's cross term), from the second L(1) + R(0)
    float mb[SP ? 2 : 1][SP ? PL::P : 1][SP ? PL::T : 1];
    uint32_t gx[SP ? 2 : 1][SP ? PL::NW : 1];     // G-check words from the peer (first CTA: t1; second: t0 ^ x_hat0)
    int pst[2][4];                                 // the peer's frontier (global), completion stage, mismatch of its half
    long long pfin[3];                             // frame end (from the second CTA): bit errors, PEs, events
    uint32_t tu[SP ? PL::NW : 1];                  // own transformed pinned hard output
    unsigned long long post;                       // second CTA: the first CTA's post (seq << 32 | frontier << 16 | code)
    unsigned long long postv;                      // its broadcast copy
};

// XH: also record each freeze event's x_hat (trace calls; a separate
// instantiation keeps the decode kernel's code unchanged)
template <int M, int KIND, bool XH = false, bool SP = false>
struct Dec {
    using PL = Plan<M, SP>;
    using C = Cfg<M, SP>;
    static constexpr int N = PL::N, P = PL::P, K = PL::K, Q = PL::Q, NW = PL::NW, kT = PL::T;
    static constexpr bool csfg = KIND == 2;

    Smem<M, SP>* sm;
    const DecodeArgs* a;
    float* Lg;  // L2 levels, N floats each
    uint32_t tb;  // this warp's TMEM columns (TMEM levels at tb + P * slot)
    static constexpr bool kTpReg = TprotReg<C>::value;
    uint32_t tpr[kTpReg && PL::NTM > 0 ? PL::NTM : 1];  // boundary masks of the TMEM levels (kTpReg)
    __device__ __forceinline__ uint32_t& tprot(int k) { return kTpReg ? tpr[k] : sm->tprot[k][tid]; }
    const float* llr;
    int tid, lane, warp;
    float alpha;
    float R[P];
    float R0[C::r0reg ? P : 1];
    float Lr[PL::NREG > 0 ? PL::NREG : 1][P];
    uint32_t lm_nz, lm_neg;  // L(m) of the thread's last-pass rows: 0 / +CAP / -CAP
    // frozen bits of the thread's rows, P bits per pass layout
    using FzT = typename std::conditional<(Q * P > 32), unsigned long long, uint32_t>::type;
    FzT fzp;
    int frontier, nev, it, ph;
    FzT snap;      // sign bits of R(S+1) after each stage of the current pass
    uint32_t onm;  // PE activations of the current pass, bit i * P/2 + k
    unsigned act;  // this thread's PE activations (< 2^32 per frame)
    bool ownp;     // this warp holds rows of a candidate block of the current pass (warp-uniform)
    // SP (one half of a frame on a 2-CTA cluster)
    int rank;       // 0: the frame's rows [0, N), 1: rows [N, 2N)
    int gfr;        // the frame's frontier, 0 .. 2N (frontier = this half's part of it)
    int cut;        // second CTA: first local stage the reference did not run in the final sweep (frame complete)
    int xcode;      // first CTA: 1 + stage index of the pass at which its frontier reached N, else 0
    bool hfz;       // this half frozen whole by a commit of the frame's stage 0
    bool nowait;    // second CTA: the frontier cannot reach N in the rest of this sweep
    bool xpend;     // the frame's stage-0 check of this sweep is pending (decided with pass 0's checks)
    uint32_t x0;    // its hard decisions: sign bits of R(1) of this half (pass 0's layout)
    unsigned act0;  // PE activations before this sweep's local stages
    float l0r[SP && !PL::L0T ? P : 1];  // the frame's L(1) of this half when not in TMEM
    uint32_t rsm;   // the peer's shared memory (cluster window address of its Smem)

    // the frame's frontier lies in this half: its candidate blocks are checked here
    __device__ __forceinline__ bool owner() const { return !SP || (gfr >> PL::M) == rank; }
    // the reference left the stage loop (csfg_freeze.cpp:109): the frame's frontier reached its end
    // (SP: or this half was frozen whole at the frame's stage 0 in this sweep)
    __device__ __forceinline__ bool ended() const { return SP ? (hfz || (rank == 1 && frontier >= N)) : frontier >= N; }
    template <typename F>
    __device__ __forceinline__ uint32_t peer_addr(const F* field) const {
        return rsm + (uint32_t)((const char*)field - (const char*)sm);
    }

    template <int q>
    __device__ __forceinline__ int row(int j) const {
        constexpr int b = PL::base(q);
        return (tid & ((1 << b) - 1)) | (j << b) | ((tid >> b) << (b + K));
    }

    template <int q>
    __device__ __forceinline__ void init_fz(const uint8_t* frozen_rows) {
        if constexpr (q == 0) fzp = 0;
#pragma unroll
        for (int j = 0; j < P; ++j) fzp |= (FzT)(frozen_rows[row<q>(j)] != 0) << (q * P + j);
        if constexpr (q + 1 < Q) init_fz<q + 1>(frozen_rows);
    }
    template <int q>
    __device__ __forceinline__ uint32_t fz() const {
        return (uint32_t)(fzp >> (q * P)) & low_mask(P);
    }

    // padded shared-memory index of row<q>(j): pad(row) = pad(row<q>(0)) +
    // pad(j << b) (the register bits never carry into the thread bits), so
    // every access is one per-pass base register plus an immediate
    template <int q>
    __device__ __forceinline__ int pbase() const {
        return PL::pad(row<q>(0));
    }
    template <int q>
    static constexpr int poff(int j) {
        return PL::pad(j << PL::base(q));
    }

    // L2-resident level index: thread-major for a level of one layout (every
    // warp access one coalesced line per register), row-indexed otherwise
    template <int s, int q>
    __device__ __forceinline__ size_t gidx(int j) const {
        if constexpr (PL::inner(s)) return ((size_t)PL::slot(s) * P + j) * kT + tid;
        else return (size_t)PL::slot(s) * N + row<q>(j);
    }

    template <int s, int q>
    __device__ __forceinline__ float ld(int j) const {
        constexpr int w = C::where(s);
        if constexpr (w == kReg) return Lr[PL::slot(s)][j];
        else if constexpr (w == kSmem) return sm->Ls[PL::slot(s)][pbase<q>() + poff<q>(j)];
        else if constexpr (w == kGlob) return Lg[gidx<s, q>(j)];
        else return ((lm_nz >> j) & 1u) ? (((lm_neg >> j) & 1u) ? -kCap : kCap) : 0.f;
    }
    template <int s, int q>
    __device__ __forceinline__ void st(int j, float v) {
        constexpr int w = C::where(s);
        if constexpr (w == kReg) Lr[PL::slot(s)][j] = v;
        else if constexpr (w == kSmem) sm->Ls[PL::slot(s)][pbase<q>() + poff<q>(j)] = v;
        else if constexpr (w == kGlob) Lg[gidx<s, q>(j)] = v;
        else {
            lm_nz |= 1u << j;
            lm_neg = v < 0.f ? (lm_neg | (1u << j)) : (lm_neg & ~(1u << j));
        }
    }

    // x_hat bits of the thread's rows, bit j = (R[j] < 0) (R is never -0)
    __device__ __forceinline__ uint32_t sign_bits() const {
        uint32_t w = 0u;
#pragma unroll
        for (int j = P - 1; j >= 0; --j) w = __funnelshift_l(__float_as_uint(R[j]), w, 1);
        return w;
    }

    // stage S; false when the csfg frontier covered n (the reference leaves
    // the stage loop, csfg_freeze.cpp:109). csfg checks are deferred to the
    // end of the pass (pass_check): the pass's stages run as if no check of
    // the pass commits, and the commits correct that afterwards.
    // Can this warp hold rows of a candidate block of pass q? Every frontier the
    // pass can reach lies in [f0, fend], fend = the end of f0's block at the
    // pass's first stage (later blocks nest inside it), and a candidate block of
    // the pass lies in the rows whose bits >= b + K are those of its frontier:
    // threads tid >> b = f0 >> (b + K) or fend >> (b + K), at most two warps when
    // b <= 5. With b > 5 the warp transform needs every warp.
    template <int q>
    __device__ __forceinline__ bool own_pass() const {
        constexpr int b = PL::base(q);
        if constexpr (b > 5) {
            return true;
        } else {
            const int f0 = frontier;
            const int fend = ((f0 >> (b + K - 1)) + 1) << (b + K - 1);
            const int th = tid >> b;
            return __any_sync(kFull, th == (f0 >> (b + K)) || th == (fend >> (b + K)));
        }
    }

    template <int S>
    __device__ __forceinline__ bool stage() {
        constexpr int q = PL::pass_of(S);
        constexpr int b = PL::base(q);
        constexpr int g = M - 1 - S;
        constexpr int dj = 1 << (g - b);
        constexpr int i = S - q * K;  // stage index inside the pass
        if constexpr (csfg) {
            if (ended()) return false;
            if constexpr (i == 0) {
                snap = 0;
                onm = 0u;
                ownp = own_pass<q>();
            }
        }
        float lt[P / 2], lb[P / 2];
        // is_pe_active (csfg_freeze.cpp:95-97) as a mask over the thread's
        // PEs; rows >= frontier are never frozen, and row<q>(0) is the
        // thread's lowest row
        uint32_t onb = low_mask(P / 2);
        if (csfg && row<q>(0) < frontier) {
            const uint8_t* fs = sm->fst + row<q>(0);
#pragma unroll
            for (int j = 0, k = 0; j < P; ++j) {
                if (j & dj) continue;
                if (row<q>(j) < frontier && (int)fs[j << b] < S) onb &= ~(1u << k);
                ++k;
            }
        }
        // SP: local L(0) is the frame's L(1): stored (TMEM) for the next cross stage and pushed to the peer
        constexpr bool l0out = SP && S == 0;
        constexpr bool tin = C::where(S + 1) == kTmem, tout = (S > 0 && C::where(S) == kTmem) || l0out;
        float tl[tin ? P : 1], to[tout ? P : 1];
        if constexpr (tin) {
            tm::wait_st();  // this level's store of the previous sweep / its boundary fix-up
            tm::ld16(tb + P * PL::slot(S + 1), tl);
            tm::wait_ld();
        }
#pragma unroll
        for (int j = 0, k = 0; j < P; ++j) {
            if (j & dj) continue;
            if constexpr (tin) {
                lt[k] = tl[j];
                lb[k] = tl[j + dj];
            } else {
                lt[k] = ld<S + 1, q>(j);
                lb[k] = ld<S + 1, q>(j + dj);
            }
            ++k;
        }
        // PE outputs of the pair (j, j + dj): stores / selects / stage-0 decisions
        auto emit = [&](int j, int k, float l_top, float l_bot, float n_t, float n_b) {
            const bool on = (onb >> k) & 1u;
            const float r_t = R[j], r_b = R[j + dj];
            bool xt = false, xb = false;
            if constexpr (tout) {
                // every PE's outputs (an inactive PE's only matter at a frozen block's
                // boundary L, which fixup_tmem restores after the sweep)
                to[j] = l_top;
                to[j + dj] = l_bot;
            } else if constexpr (S > 0) {
                if (on) {
                    st<S, q>(j, l_top);
                    st<S, q>(j + dj, l_bot);
                }
            } else {  // L(0) only feeds the G-check's x_hat (bp_core.cpp:99); stage 0 is always active
                xt = __fadd_rn(r_t, l_top) < 0.f;
                xb = __fadd_rn(r_b, l_bot) < 0.f;
            }
            R[j] = on ? n_t : r_t;
            R[j + dj] = on ? n_b : r_b;
            if constexpr (S == 0 && KIND != 0 && !SP) {
                // pass 0: a warp's lanes hold 32 consecutive rows of every register
                const int rt = row<q>(j), rb = rt + (1 << g);
                const uint32_t wt = __ballot_sync(kFull, xt), wb = __ballot_sync(kFull, xb);
                if (lane == 0) {
                    sm->xh[rt >> 5] = wt;
                    sm->xh[rb >> 5] = wb;
                }
            }
        };
        // every PE is computed; an inactive one keeps R and L unchanged (selects and
        // predicated stores instead of a branch per PE)
        if constexpr (dj >= 2 && Pack<C>::on(KIND)) {
            // two PEs per packed fp32x2 instruction (FADD2 / FFMA2), as the warp
            // kernel: products as fma(alpha, m, +0) (ptxas would fuse a bare
            // mul.f32x2 into the following add; the +0 addend only turns a -0
            // product into +0, which no decision distinguishes)
#pragma unroll
            for (int j = 0, k = 0; j < P; j += 2) {
                if (j & dj) continue;
                const float r_t0 = R[j], r_t1 = R[j + 1], r_b0 = R[j + dj], r_b1 = R[j + dj + 1];
                float c0, c1, s0, s1, lt0, lt1, lb0, lb1, nt0, nt1, nb0, nb1;
                fma2s0(c0, c1, alpha, xsmin(lt[k], r_t0), xsmin(lt[k + 1], r_t1));
                add2(s0, s1, lb[k], lb[k + 1], r_b0, r_b1);
                fma2s0(lt0, lt1, alpha, xsmin(lt[k], s0), xsmin(lt[k + 1], s1));
                add2(lb0, lb1, lb[k], lb[k + 1], c0, c1);
                fma2s0(nt0, nt1, alpha, xsmin(r_t0, s0), xsmin(r_t1, s1));
                add2(nb0, nb1, r_b0, r_b1, c0, c1);
                emit(j, k, lt0, lb0, nt0, nb0);
                emit(j + 1, k + 1, lt1, lb1, nt1, nb1);
                k += 2;
            }
        } else {
#pragma unroll
            for (int j = 0, k = 0; j < P; ++j) {
                if (j & dj) continue;
                const float r_t = R[j], r_b = R[j + dj];
                const float cross = __fmul_rn(alpha, xsmin(lt[k], r_t));
                const float sum_bot = __fadd_rn(lb[k], r_b);
                const float l_top = __fmul_rn(alpha, xsmin(lt[k], sum_bot));
                const float l_bot = __fadd_rn(lb[k], cross);
                emit(j, k, l_top, l_bot, __fmaf_rn(alpha, xsmin(r_t, sum_bot), 0.0f), __fadd_rn(r_b, cross));
                ++k;
            }
        }
        if constexpr (l0out) {
            if constexpr (PL::L0T) {
                tm::st16(tb + P * PL::L0S, to);
            } else {
#pragma unroll
                for (int j = 0; j < P; ++j) l0r[j] = to[j];
            }  // (pushed to the peer after the sweep: push_l1)
        } else if constexpr (tout) {
            tm::st16(tb + P * PL::slot(S), to);
        }
        act += __popc(onb);
        if constexpr (csfg) {
            onm |= onb << (i * (P / 2));
            if (ownp) snap |= (FzT)sign_bits() << (i * P);
        }
        constexpr bool pass_end = S == PL::last(q);
        constexpr bool boundary = pass_end && q + 1 < Q;
        // R(S+1) into the next pass's layout; it does not depend on the
        // verdicts, so the check's barriers also order the exchange
        if constexpr (boundary) {
            if constexpr (!C::rx2) __syncthreads();  // readers of the previous boundary are done
            float* rx = sm->Rx[C::rx2 ? (q & 1) : 0];
#pragma unroll
            for (int j = 0; j < P; ++j) rx[pbase<q>() + poff<q>(j)] = R[j];
        }
        if constexpr (csfg && pass_end) pass_check<q>();
        if constexpr (boundary) {
            if constexpr (!csfg) __syncthreads();
            const float* rx = sm->Rx[C::rx2 ? (q & 1) : 0];
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = rx[pbase<q + 1>() + poff<q + 1>(j)];
        }
        return true;
    }

    // lane bits [0, NL) of the transform by shuffles: the lower lane absorbs
    template <int NL, typename W>
    __device__ __forceinline__ W lane_transform(W w) const {
#pragma unroll
        for (int k = 0; k < NL; ++k) {
            const W v = __shfl_xor_sync(kFull, w, 1 << k);
            if (!((lane >> k) & 1)) w ^= v;
        }
        return w;
    }

    // warp-index bits [0, NWB): XOR over the supersets, through shared memory
    template <int NWB, typename W>
    __device__ __forceinline__ W warp_transform(W w) {
        sm->buf[tid] = w;
        __syncthreads();
        const int wl = warp & ((1 << NWB) - 1), wh = warp - wl;
        W acc = 0;
        const auto* col = sm->buf + wh * 32 + lane;
#pragma unroll
        for (int s = 0; s < (1 << NWB); ++s)
            if ((s & wl) == wl) acc ^= (W)col[s * 32];
        return acc;
    }

    // P-bit mask of the thread's rows (layout q) inside block `index` of size 2^g:
    // row >> g = (thread-high bits << (b + K - g)) | (j >> (g - b))
    template <int q, int g>
    __device__ __forceinline__ uint32_t block_mask(int index) const {
        constexpr int b = PL::base(q);
        constexpr int hb = b + K - g;
        const int jsel = index & ((1 << hb) - 1);
        return (index >> hb) == (tid >> b) ? low_mask(1 << (g - b)) << (jsel << (g - b)) : 0u;
    }

    // in-thread transform levels of stage index i of pass q, into the packed word
    template <int q, int i>
    __device__ __forceinline__ FzT pass_bits() const {
        constexpr int S = q * K + i;
        if constexpr (S > PL::last(q)) {
            return 0;
        } else {
            const uint32_t w = bits_transform<M - 1 - S - PL::base(q)>((uint32_t)(snap >> (i * P)) & low_mask(P));
            return ((FzT)w << (i * P)) | pass_bits<q, i + 1>();
        }
    }

    // violation bits of stage index i for every frontier the pass's earlier
    // commits can produce: bit (2^i - 1 + v), v = the set of earlier stages
    // that committed; f[] holds those frontiers (f[2^i - 1 + v]). A block of
    // 2^g rows covers nb = 2^(g-b) of the thread's registers: fold the
    // violations of each group, then a frontier fr selects group
    // (fr >> b) & (P - nb) when its thread bits (fr >> (b+K)) are the
    // thread's own (never true for fr >= n).
    template <int q, int i>
    __device__ __forceinline__ uint32_t pass_viol(FzT W, int* f) const {
        constexpr int S = q * K + i;
        if constexpr (S > PL::last(q)) {
            return 0u;
        } else {
            constexpr int b = PL::base(q);
            constexpr int g = M - 1 - S;
            constexpr int nb = 1 << (g - b);
            uint32_t u = (uint32_t)(W >> (i * P)) & fz<q>();
#pragma unroll
            for (int h = 1; h < nb; h <<= 1) u |= u >> h;
            const int th = tid >> b;
            uint32_t bad = 0u;
#pragma unroll
            for (int v = 0; v < (1 << i); ++v) {
                const int fr = f[(1 << i) - 1 + v];
                const int t = fr >> b;
                bad |= (((t >> K) == th ? u : 0u) >> (t & (P - nb)) & 1u) << ((1 << i) - 1 + v);
                // frontiers of stage i + 1: unchanged, or the end of this block
                if constexpr (S < PL::last(q)) {
                    f[(2 << i) - 1 + v] = fr;
                    f[(2 << i) - 1 + v + (1 << i)] = ((fr >> g) + 1) << g;
                }
            }
            return bad | pass_viol<q, i + 1>(W, f);
        }
    }

    // candidate_block / check_csfg / apply_freeze (csfg_freeze.cpp:8-39,
    // 82-93, 116-118) for every stage of pass q, in the reference's order.
    // The candidate transform of a stage is the same for every block of its
    // size, so one transform per stage serves every frontier; lane and warp
    // bits are shared by all of the pass's stages (their blocks span them).
    template <int q>
    __device__ __forceinline__ void pass_check() {
        constexpr int b = PL::base(q);
        constexpr int nst = PL::last(q) - q * K + 1;
        int first = 0;  // first stage index of the pass whose candidate this CTA checks
        if constexpr (SP) {
            if (q == 0 && xpend) {
                // the frame's stage-0 candidate (csfg_freeze.cpp:111-118 at stage 0), decided
                // before pass 0's candidates: an accept makes this sweep's local stages
                // void (every PE of the half inactive), so they are uncounted
                xpend = false;
                xcode = 0;
                const bool acc = cross_check();
                post<0>();  // (first CTA) its frontier after the frame's stage-0 check
                if (acc) return;
            }
            if (!owner()) {
                if (rank == 0) {  // the frontier moved to the second half
                    __syncthreads();  // (orders the pass-boundary R exchange, as the check's barriers do)
                    return;
                }
                if (nowait) {
                    __syncthreads();
                    return;
                }
                first = take_over<q>();
                if (first > nst) return;  // the first CTA still holds the frontier after this pass
            }
            xcode = 0;
        }
        FzT W = 0;
        if (ownp) {  // (warps without rows of a candidate contribute no violation)
            W = pass_bits<q, 0>();
            W = lane_transform<(b < 5 ? b : 5)>(W);
            if constexpr (b > 5) W = warp_transform<b - 5>(W);
            int f[(1 << nst) - 1 + (1 << nst)];
            f[0] = frontier;
            uint32_t bad = pass_viol<q, 0>(W, f);
            bad = __reduce_or_sync(kFull, bad);
            if (lane == 0 && bad) atomicOr(&sm->vw[ph], bad);
        }
        __syncthreads();
        uint32_t bad;
        bad = sm->vw[ph];
        if (tid == 0) sm->vw[ph == 0 ? 2 : ph - 1] = 0u;  // used two checks from now
        ph = ph == 2 ? 0 : ph + 1;
        if (bad == (1u << ((1 << nst) - 1)) - 1u) {  // every candidate rejected
            if constexpr (SP) post<q + 1>();
            return;
        }
        bool any = false;
        commit_walk<q, 0>(W, bad, 0, any, first);
        if constexpr (SP) post<q + 1>();
        // freeze stages are read in another layout by the next pass
        if (any) __syncthreads();
    }

    template <int q, int i>
    __device__ __forceinline__ void commit_walk(FzT W, uint32_t bad, int v, bool& any, int first) {
        constexpr int S = q * K + i;
        if constexpr (S <= PL::last(q)) {
            if (frontier >= N) return;
            if (i >= first && !((bad >> ((1 << i) - 1 + v)) & 1u)) {
                commit<q, i>(W);
                v |= 1 << i;
                any = true;
            }
            commit_walk<q, i + 1>(W, bad, v, any, first);
        }
    }

    // apply_freeze of stage index i's candidate by the owners of its rows, and
    // the PE activations of the pass's later stages that the commit made
    // inactive (or, when the frontier reached n, that the reference never ran)
    template <int q, int i>
    __device__ __forceinline__ void commit(FzT W) {
        constexpr int b = PL::base(q);
        constexpr int S = q * K + i;
        constexpr int g = M - 1 - S;
        constexpr int sz = 1 << g;
        const int index = frontier >> g;
        const int start = index << g;
        const uint32_t bm = block_mask<q, g>(index);
        const uint32_t u = (uint32_t)(W >> (i * P));
        const uint32_t x = (uint32_t)(snap >> (i * P));
        if (bm) {
            // L(S+1) = +-CAP: register levels by compile-time index, L(m) as
            // masks, the rest in the runtime loop below (commits are rare: the
            // loop keeps their code small in the instruction cache)
            constexpr int wl = C::where(S + 1);
            if constexpr (wl == kReg) {
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if ((bm >> j) & 1u) Lr[PL::slot(S + 1)][j] = ((x >> j) & 1u) ? -kCap : kCap;
            } else if constexpr (wl == kBits) {
                lm_nz |= bm;
                lm_neg = (lm_neg & ~bm) | (x & bm);
            } else if constexpr (wl == kTmem) {  // written into TMEM by fixup_tmem after the sweep
                uint32_t& w = tprot(PL::slot(S + 1));
                w = (w | bm) & ~(bm << 16);
                w |= (x & bm) << 16;
            }
#pragma unroll 1
            for (uint32_t left = bm; left; left &= left - 1u) {
                const int j = __ffs(left) - 1;
                const int r = row<q>(j);
                if constexpr (wl == kSmem || wl == kGlob) st<S + 1, q>(j, ((x >> j) & 1u) ? -kCap : kCap);
                if ((int)sm->fst[r] > S) sm->fst[r] = (uint8_t)S;
                const uint32_t bit = 1u << (r & 31);
                if ((u >> j) & 1u) atomicOr(&sm->dec[r >> 5], bit);
                else atomicAnd(&sm->dec[r >> 5], ~bit);
                if (XH && a->ev_xhat && nev < a->ev_cap && ((x >> j) & 1u))
                    atomicOr(&a->ev_xhat[((long long)sm->frame * a->ev_cap + nev) * NW + (r >> 5)], bit);
            }
        }
        if (!SP && tid == 0 && a->events && nev < a->ev_cap) {
            int* e = a->events + ((long long)sm->frame * a->ev_cap + nev) * 5;
            e[0] = it;
            e[1] = S;
            e[2] = index;
            e[3] = start;
            e[4] = sz;
        }
        nev += 1;
        frontier = start + sz;
        if constexpr (SP) {
            gfr = rank * N + frontier;
            if (frontier >= N) {
                if (rank == 0) xcode = i + 1;  // the second CTA checks from stage index i + 1 on
                else cut = S + 1;              // the frame is complete: its stage S + 2 (local S + 1) never ran
            }
        }
        uncount<q, i + 1>(bm, ended());
    }

    template <int q, int i>
    __device__ __forceinline__ void uncount(uint32_t bm, bool all) {
        constexpr int S = q * K + i;
        if constexpr (S <= PL::last(q)) {
            // top rows of stage S inside the block, as PE indices: the block is
            // the register run [j0, j0 + n) (n a power of two larger than the
            // stage's register distance), so its top rows are the PE run
            // [j0 / 2, j0 / 2 + n / 2)
            const uint32_t tm = bm ? low_mask(__popc(bm) >> 1) << ((__ffs(bm) - 1) >> 1) : 0u;
            const uint32_t drop = (all ? low_mask(P / 2) : tm) << (i * (P / 2)) & onm;
            act -= __popc(drop);
            onm &= ~drop;
            uncount<q, i + 1>(bm, all);
        }
    }

    // TMEM levels: the saturated boundary L(S+1) of blocks frozen at stage S,
    // overwritten by their (inactive) stage-S+1 PEs in this sweep, set back to
    // +-CAP before the next sweep's stage S reads it (csfg_freeze.cpp:84-86)
    template <int K_ = 0>
    __device__ __forceinline__ void fixup_tmem() {
        if constexpr (K_ < PL::NTM) {
            const uint32_t w = tprot(K_);
            if (__any_sync(kFull, w != 0u)) {
                float v[P];
                tm::ld16(tb + P * K_, v);
                tm::wait_ld();
#pragma unroll
                for (int j = 0; j < P; ++j)
                    if ((w >> j) & 1u) v[j] = ((w >> (16 + j)) & 1u) ? -kCap : kCap;
                tm::st16(tb + P * K_, v);
            }
            fixup_tmem<K_ + 1>();
        }
    }

    // ---- SP: the pair protocol -------------------------------------------
    // The first CTA owns the frontier until it reaches N. It posts its
    // frontier after the check of the frame's stage 0 and after each pass
    // (seq = it * (Q + 1) + phase, phase 0 = the cross stage's check, q + 1 =
    // pass q; code = 1 + the stage index at which the frontier left the first
    // half). The second CTA's checks of pass q wait for that pass's post only
    // while a crossing in pass q is possible: candidate blocks are aligned, so
    // a frontier below N - (block size of the pass's first stage) at the
    // pass's start stays below it for the rest of the sweep (every later
    // block is smaller) -- then it stops waiting until the next sweep.
    // After the frontier crossed, neither waits.

    // this half's R(0) (pass 0's layout, -0 -> +0)
    __device__ __forceinline__ void own_r0(float (&r)[P]) const {
        if constexpr (PL::L0T) {
            tm::ld16(tb + P * PL::R0S, r);
            tm::wait_ld();
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) r[j] = __fadd_rn(llr[(long long)rank * N + row<0>(j)], 0.0f);
        }
    }

    // The frame's stage-0 term the peer needs from this half's L(1) = v (local
    // L(0) of this sweep) and R(0), into its mailbox: the first CTA sends the
    // cross term alpha * min-with-sign(L(1), R(0)), the second L(1) + R(0)
    // (bp_core.cpp:21-24: the same operations on the same operands as a
    // one-CTA stage 0, so the peer needs no R(0) of this half)
    // this sweep's L(1) of the half (local stage 0's output, or +-CAP once frozen)
    __device__ __forceinline__ void push_l1() const {
        float v[P];
        if constexpr (PL::L0T) {
            tm::wait_st();
            tm::ld16(tb + P * PL::L0S, v);
            tm::wait_ld();
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) v[j] = l0r[j];
        }
        push_x(v);
    }

    __device__ __forceinline__ void push_x(const float* v) const {
        float r[P];
        own_r0(r);
#pragma unroll
        for (int j = 0; j < P; ++j) {
            const float x = rank == 0 ? __fmul_rn(alpha, xsmin(v[j], r[j])) : __fadd_rn(v[j], r[j]);
            st_peer(peer_addr(&sm->mb[it & 1][j][tid]), x);
        }
    }

    template <int PH>
    __device__ __forceinline__ void post() const {
        if (rank == 0 && tid == 0)
            st_peer(peer_addr(&sm->post), ((unsigned long long)(it * (Q + 1) + PH) << 32) |
                                              ((unsigned long long)frontier << 16) | (unsigned long long)xcode);
    }

    // second CTA before owning the frontier: the first stage index of pass q
    // it checks (> the pass's stage count: none, the first half still holds it)
    template <int q>
    __device__ __forceinline__ int take_over() {
        const uint32_t s0 = (uint32_t)it * (Q + 1), sq0 = s0 + q, sq1 = sq0 + 1;
        constexpr int bound = N - (N >> (q * K + 1));  // a frontier below it cannot cross in pass q or later
        if (tid == 0) {
            unsigned long long w;
            do {  // the frontier at the start of pass q (or a crossing of this sweep)
                w = ld_volatile(&sm->post);
            } while ((uint32_t)(w >> 32) < sq0 && !((w & 0xffffu) && (uint32_t)(w >> 32) >= s0));
            if ((uint32_t)(w >> 32) == sq0 && !(w & 0xffffu) && (int)((w >> 16) & 0xffffu) >= bound) {
                do {  // a crossing in pass q is possible: its verdict
                    w = ld_volatile(&sm->post);
                } while ((uint32_t)(w >> 32) < sq1);
            }
            sm->postv = w;
        }
        __syncthreads();
        const unsigned long long w = sm->postv;
        const uint32_t seq = (uint32_t)(w >> 32);
        const int code = (int)(w & 0xffffu);
        if (code && (seq == sq1 || (q == 0 && seq == s0))) {
            gfr = N;  // the frame's frontier is this half's row 0
            return seq == s0 ? 0 : code;
        }
        if (seq == sq0 && !code) nowait = true;  // (the bound held: no crossing in this sweep)
        return 1 << 30;
    }

    // The frame's stage 0 (distance N, bp_core.cpp:18-32, always active): row r
    // of both halves meets at the same thread position of both CTAs. R(1) of
    // this half goes to R (pass 0's layout), x_hat = (R(0) + L(0) < 0) of this
    // half to sm->xh (bp_core.cpp:99); its PEs are counted by the first CTA.
    __device__ __forceinline__ void cross_stage() {
        float lo[P], r0[P];
        if constexpr (PL::L0T) {
            tm::wait_st();
            tm::ld16(tb + P * PL::L0S, lo);
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) lo[j] = l0r[j];
        }
        own_r0(r0);
#pragma unroll
        for (int j = 0; j < P; ++j) {
            // the first CTA: l_top and R(1) of the top rows from the peer's L(1) + R(0)
            // (sum_bot); the second: l_bot and R(1) of the bottom rows from the cross term
            const float pm = sm->mb[(it - 1) & 1][j][tid];
            float rn, x;
            if (rank == 0) {
                const float l_top = __fmul_rn(alpha, xsmin(lo[j], pm));
                rn = __fmaf_rn(alpha, xsmin(r0[j], pm), 0.0f);
                x = __fadd_rn(r0[j], l_top);
            } else {
                const float l_bot = __fadd_rn(lo[j], pm);
                rn = __fadd_rn(r0[j], pm);
                x = __fadd_rn(r0[j], l_bot);
            }
            R[j] = rn;
            const uint32_t w = __ballot_sync(kFull, x < 0.f);
            if (lane == 0) sm->xh[row<0>(j) >> 5] = w;
        }
        if (rank == 0) act += P;
    }

    // candidate_block of the frame's stage 0 (this half, size N) and its
    // check/commit (csfg_freeze.cpp:18-39, 82-93) on R(1): the transform over
    // every row bit of the half (register, lane and warp bits of pass 0)
    __device__ __forceinline__ bool cross_check() {
        const uint32_t x = x0;
        uint32_t u = bits_transform<K>(x);
        u = lane_transform<5>(u);
        u = warp_transform<PL::LOGT - 5>(u);
        if (__syncthreads_or((u & fz<0>()) != 0u)) return false;
        // apply_freeze: L(1) = +-CAP over the half (over the speculative values
        // local stage 0 stored and pushed), freeze stage 0 (every later stage of
        // the half inactive: its local sweeps stop), decided_u = u
        hfz = true;
        act = act0;
        float v[P];
#pragma unroll
        for (int j = 0; j < P; ++j) {
            v[j] = ((x >> j) & 1u) ? -kCap : kCap;
            const uint32_t w = __ballot_sync(kFull, (u >> j) & 1u);
            if (lane == 0) sm->dec[row<0>(j) >> 5] = w;
        }
        if constexpr (PL::L0T) {
            tm::wait_st();
            tm::st16(tb + P * PL::L0S, v);
        } else {
#pragma unroll
            for (int j = 0; j < P; ++j) l0r[j] = v[j];
        }
        nev += 1;
        frontier = N;
        gfr = rank * N + N;
        if (rank == 1) {
            cut = 0;  // the frame is complete: no stage after its stage 0 ran
        } else {
            xcode = 1;
        }
        return true;
    }

    // PE activations of local stages >= l0 under the final freeze stages
    // (first CTA, when the second half completed the frame mid-sweep)
    __device__ __forceinline__ unsigned recount_from(int l0) const {
        unsigned c = 0;
        for (int l = l0; l < M; ++l) {
            const int g = M - 1 - l;
            for (int p = tid; p < N / 2; p += kT) {
                const int r = ((p >> g) << (g + 1)) | (p & ((1 << g) - 1));
                c += (int)sm->fst[r] >= l ? 1u : 0u;
            }
        }
        return c;
    }

    template <int S>
    __device__ __forceinline__ bool sweep_from() {
        if (!stage<S>()) return false;
        if constexpr (S + 1 < M) return sweep_from<S + 1>();
        return true;
    }

    // hard_output with frozen rows 0 and rows < pin from decided_u, as the
    // thread's P-bit group (rows P*tid + j; R in the last pass's layout)
    __device__ __forceinline__ uint32_t u_group(int pin) const {
        uint32_t u = sign_bits() & ~fz<Q - 1>();
        const int r0 = P * tid;
        if (pin > r0) {
            const uint32_t pm = pin - r0 >= P ? low_mask(P) : low_mask(pin - r0);
            const uint32_t d = (sm->dec[r0 >> 5] >> (r0 & 31)) & low_mask(P);
            u = (u & ~pm) | (d & pm);
        }
        return u;
    }

    // gmatrix_converged (bp_core.cpp:95-102) with the pinned prefix
    // (csfg_freeze.cpp:120-135): the transform over all n row bits (register
    // bits [0, K), lane bits [K, K+5), warp bits above), compared to x_hat
    __device__ __forceinline__ bool gcheck(int pin) {
        uint32_t u = bits_transform<K>(u_group(pin));
        u = lane_transform<5>(u);
        u = warp_transform<PL::LOGT - 5>(u);
        const int r0 = P * tid;
        const uint32_t x = (sm->xh[r0 >> 5] >> (r0 & 31)) & low_mask(P);
        return !__syncthreads_or(u != x);
    }

    __device__ void run(const DecodeArgs& args, Smem<M, SP>* s) {
        a = &args;
        sm = s;
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        alpha = args.alpha;
        Lg = args.scratch + (long long)blockIdx.x * args.scratch_stride;
        init_fz<0>(args.frozen_rows);
        for (;;) {
            __syncthreads();
            if (tid == 0) {
                const unsigned long long idx = atomicAdd(args.queue, 1ull);
                sm->frame = (long long)idx < args.frames ? (long long)idx : -1;
            }
            __syncthreads();
            const long long f = sm->frame;
            if (f < 0) break;
            // channel LLRs (R(0), -0 -> +0) in pass 0's layout; frames beyond
            // the clamp-free bound go to the generic kernel
            llr = args.llr + f * (long long)N;
            bool bad = false;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                const float v = llr[row<0>(j)];
                bad |= !(fabsf(v) <= kClampFreeBound);
                if constexpr (C::r0reg) R0[j] = __fadd_rn(v, 0.0f);
            }
            if (__syncthreads_or(bad)) {
                if (tid == 0) {
                    const unsigned long long slot = atomicAdd(args.list_len, 1ull);
                    args.list[slot] = f + args.frame_base;
                }
                continue;
            }
            // init_state (bp_core.cpp:43-56)
#pragma unroll
            for (int l = 0; l < PL::NREG; ++l)
#pragma unroll
                for (int j = 0; j < P; ++j) Lr[l][j] = 0.f;
            lm_nz = fz<Q - 1>();
            lm_neg = 0u;
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = 0.f;  // R(m) = 0 until the first sweep (max_iter = 0)
            for (int i = tid; i < PL::NSM * PL::NX; i += kT) (&sm->Ls[0][0])[i] = 0.f;
            for (int i = tid; i < PL::NGL * N; i += kT) Lg[i] = 0.f;
            if constexpr (PL::NTM > 0) {
                float z[P];
#pragma unroll
                for (int j = 0; j < P; ++j) z[j] = 0.f;
#pragma unroll
                for (int k = 0; k < PL::NTM; ++k) {
                    tm::st16(tb + P * k, z);
                    tprot(k) = 0u;
                }
                if constexpr (PL::R0T) {
#pragma unroll
                    for (int j = 0; j < P; ++j) z[j] = __fadd_rn(llr[row<0>(j)], 0.0f);
                    tm::st16(tb + P * PL::NTM, z);
                }
            }
            for (int r = tid; r < N; r += kT) sm->fst[r] = kNotFrozen;
            for (int w = tid; w < NW; w += kT) sm->dec[w] = 0u;
            frontier = 0;
            nev = 0;
            ph = 0;
            if (tid < 3) sm->vw[tid] = 0u;
            act = 0;
            __syncthreads();
            int iters = (KIND == 0) ? args.max_iter : 0;
            int stop = 0;
            bool converged = false;
            for (int t = 1; t <= args.max_iter; ++t) {
                if constexpr (csfg) {
                    if (frontier >= N || converged) break;
                    iters = t;
                }
                it = t;
                // keep the per-stage row/address arithmetic inside the loop
                // (hoisted for every stage it would not fit in the registers)
                asm volatile("" : "+r"(tid));
                if constexpr (PL::R0T) {
                    tm::wait_st();
                    tm::ld16(tb + P * PL::NTM, R);
                    tm::wait_ld();
                } else {
#pragma unroll
                    for (int j = 0; j < P; ++j) {
                        if constexpr (C::r0reg) R[j] = R0[j];
                        else R[j] = __fadd_rn(llr[row<0>(j)], 0.0f);
                    }
                }
                sweep_from<0>();
                if constexpr (csfg && PL::NTM > 0) fixup_tmem();
                if constexpr (KIND == 0) {
                    __syncthreads();  // Rx buffers are reused by the next sweep
                } else if constexpr (KIND == 1) {
                    if (gcheck(0)) {
                        iters = t;
                        stop = 1;
                        break;
                    }
                } else {
                    if (frontier < N) converged = gcheck(frontier);
                }
            }
            if constexpr (KIND == 1) {
                if (stop == 0) iters = args.max_iter;
            }
            if constexpr (csfg) stop = (frontier >= N) ? 2 : (converged ? 1 : 0);
            // DecodeOutcome (bp_core.cpp:106-115, csfg_freeze.cpp:137-151)
            __syncthreads();  // decided_u of the last commits
            uint32_t u;
            const int r0 = P * tid;
            if (csfg && frontier >= N) u = (sm->dec[r0 >> 5] >> (r0 & 31)) & low_mask(P);
            else u = u_group(csfg ? frontier : 0);
            // the P-bit groups of 32/P consecutive threads form one word
            uint32_t word = u << (r0 & 31);
#pragma unroll
            for (int o = 1; o < 32 / P; o <<= 1) word |= __shfl_xor_sync(kFull, word, o);
            int berr = 0;
            if ((r0 & 31) == 0) {
                const int wi = r0 >> 5;
                if (args.u_bits) args.u_bits[f * NW + wi] = word;
                if (args.truth_u) berr = __popc((word ^ args.truth_u[f * NW + wi]) & ~args.frozen_bits[wi]);
            }
            berr = __reduce_add_sync(kFull, berr);
            const unsigned wact = __reduce_add_sync(kFull, act);
            // per-CTA sums through shared memory (buf: no transform is pending)
            if (lane == 0) {
                sm->buf[2 * warp] = (uint32_t)berr;
                sm->buf[2 * warp + 1] = wact;
            }
            __syncthreads();
            if (tid == 0) {
                long long pe = 0;
                int be = 0;
                for (int w = 0; w < PL::NWARP; ++w) {
                    be += (int)sm->buf[2 * w];
                    pe += sm->buf[2 * w + 1];
                }
                if (args.iters) args.iters[f] = iters;
                if (args.pe) args.pe[f] = pe;
                if (args.stop) args.stop[f] = (uint8_t)stop;
                if (args.nev) args.nev[f] = nev;
                if (args.counters) {
                    unsigned long long* cs = counter_set(args, f);
                    atomicAdd(&cs[kCntFrames], 1ull);
                    atomicAdd(&cs[kCntBitErr], (unsigned long long)be);
                    atomicAdd(&cs[kCntFrameErr], be > 0 ? 1ull : 0ull);
                    atomicAdd(&cs[kCntIters], (unsigned long long)iters);
                    atomicAdd(&cs[kCntItersSq], (unsigned long long)iters * iters);
                    atomicAdd(&cs[kCntPe], (unsigned long long)pe);
                    atomicAdd(&cs[kCntEvents], (unsigned long long)nev);
                    atomicAdd(&cs[kCntStop0 + stop], 1ull);
                }
            }
        }
    }

    // SP: one half of each frame of length 2N on a 2-CTA cluster (csfg; G-stop and
    // fixed-iteration decodes run the same loop without the frontier).
    // Per iteration: the cross stage (the frame's stage 0) from the peer's
    // L(1) in the mailbox, the check of the frame's stage-0 candidate by the
    // half holding the frontier, the local sweep (the frame's stages 1..m-1,
    // whose local stage 0 pushes the new L(1) into the peer's mailbox), the
    // pinned G-check over both halves (csfg_freeze.cpp:120-135: the frame's
    // transform is the halves' local transforms plus one XOR level across
    // the pair). Two cluster barriers per iteration: after the cross stage
    // (the mailbox is consumed before the peer refills it) and at the end
    // (mailbox, G-check words and frontier exchanged).
    __device__ void run_pair(const DecodeArgs& args, Smem<M, SP>* s) {
        a = &args;
        sm = s;
        tid = threadIdx.x;
        lane = tid & 31;
        warp = tid >> 5;
        alpha = args.alpha;
        rank = cluster_rank();
        rsm = cluster_map(sm, rank ^ 1);
        constexpr int N2 = 2 * N;
        init_fz<0>(args.frozen_rows + (long long)rank * N);
        for (;;) {
            // the previous frame is done in both CTAs: reset what the peer writes
            if (rank == 1 && tid == 0) sm->post = 0u;
            cluster_sync();
            if (rank == 0 && tid == 0) {
                const unsigned long long idx = atomicAdd(args.queue, 1ull);
                const long long v = (long long)idx < args.frames ? (long long)idx : -1;
                sm->frame = v;
                st_peer(peer_addr(&sm->frame), v);
            }
            cluster_sync();
            const long long f = sm->frame;
            if (f < 0) break;
            // both CTAs test the whole frame (their own rows and the peer's at
            // the same positions), so they agree without an exchange
            llr = args.llr + f * (long long)N2;
            bool bad = false;
#pragma unroll
            for (int j = 0; j < P; ++j) {
                bad |= !(fabsf(llr[row<0>(j)]) <= kClampFreeBound);
                bad |= !(fabsf(llr[N + row<0>(j)]) <= kClampFreeBound);
            }
            if (__syncthreads_or(bad)) {
                if (rank == 0 && tid == 0) {
                    const unsigned long long slot = atomicAdd(args.list_len, 1ull);
                    args.list[slot] = f + args.frame_base;
                }
                continue;
            }
            // init_state (bp_core.cpp:43-56)
#pragma unroll
            for (int l = 0; l < PL::NREG; ++l)
#pragma unroll
                for (int j = 0; j < P; ++j) Lr[l][j] = 0.f;
            lm_nz = fz<Q - 1>();
            lm_neg = 0u;
#pragma unroll
            for (int j = 0; j < P; ++j) R[j] = 0.f;
            for (int i = tid; i < PL::NSM * PL::NX; i += kT) (&sm->Ls[0][0])[i] = 0.f;
            {
                float z[P];
#pragma unroll
                for (int j = 0; j < P; ++j) z[j] = 0.f;
#pragma unroll
                for (int k = 0; k < PL::NTM; ++k) {
                    tm::st16(tb + P * k, z);
                    tprot(k) = 0u;
                }
                if constexpr (PL::L0T) {
                    tm::st16(tb + P * PL::L0S, z);
                    float r[P];
#pragma unroll
                    for (int j = 0; j < P; ++j) r[j] = __fadd_rn(llr[(long long)rank * N + row<0>(j)], 0.0f);
                    tm::st16(tb + P * PL::R0S, r);
                } else {
#pragma unroll
                    for (int j = 0; j < P; ++j) l0r[j] = 0.f;
                }
                tm::wait_st();
                // sweep 1's stage-0 terms (L(1) = 0) into the peer's mailbox slot 0
                it = 0;
                push_x(z);
            }
            for (int r = tid; r < N; r += kT) sm->fst[r] = kNotFrozen;
            for (int w = tid; w < NW; w += kT) sm->dec[w] = 0u;
            frontier = 0;
            gfr = 0;
            cut = M;
            xcode = 0;
            hfz = false;
            nev = 0;
            ph = 0;
            if (tid < 3) sm->vw[tid] = 0u;
            act = 0;
            cluster_sync();  // (and the peer's sweep-1 terms are in the mailbox)
            int iters = 0;
            bool converged = false;
            for (int t = 1; t <= args.max_iter; ++t) {
                if (gfr >= N2 || converged) break;
                iters = t;
                it = t;
                asm volatile("" : "+r"(tid));
                cross_stage();
                nowait = false;
                x0 = sign_bits();
                act0 = act;
                xpend = owner() && !hfz;  // checked with pass 0's candidates
                if (!hfz) {
                    sweep_from<0>();
                    if constexpr (PL::NTM > 0) fixup_tmem();
                }
                push_l1();
                if constexpr (KIND == 0) {  // fixed iterations: no G-check, only the exchange's ordering
                    cluster_sync();
                    continue;
                }
                // pinned G-check inputs: this half's hard output (rows < frontier
                // from decided_u; G-stop: frontier 0), transformed over the half's row bits
                uint32_t g = bits_transform<K>(u_group(frontier));
                g = lane_transform<5>(g);
                g = warp_transform<PL::LOGT - 5>(g);
                const int r0 = P * tid;
                uint32_t word = g << (r0 & 31);
#pragma unroll
                for (int o = 1; o < 32 / P; o <<= 1) word |= __shfl_xor_sync(kFull, word, o);
                // x = the frame's transform: first half t0 ^ t1, second half t1;
                // the first CTA sends t0 ^ x_hat0, the second t1 and whether its
                // half mismatches (t1 != x_hat1): both then decide the same
                if ((r0 & 31) == 0) sm->tu[r0 >> 5] = word;
                __syncthreads();
                const int gs = it & 1;
                bool mm1 = false;
                if (tid < NW) {
                    const uint32_t t = sm->tu[tid];
                    st_peer(peer_addr(&sm->gx[gs][tid]), rank == 0 ? t ^ sm->xh[tid] : t);
                    mm1 = rank == 1 && t != sm->xh[tid];
                }
                mm1 = __syncthreads_or(mm1);
                if (tid == 0) {
                    st_peer(peer_addr(&sm->pst[gs][0]), gfr);
                    st_peer(peer_addr(&sm->pst[gs][1]), cut);
                    st_peer(peer_addr(&sm->pst[gs][2]), (int)mm1);
                }
                cluster_sync();
                const int pg = sm->pst[gs][0];
                if (rank == 0) {
                    cut = sm->pst[gs][1];
                    mm1 = sm->pst[gs][2] != 0;
                }
                gfr = max(gfr, pg);
                if (gfr < N2) {
                    bool mm = false;
                    if (tid < NW) {
                        const uint32_t g = sm->gx[gs][tid];
                        mm = rank == 0 ? ((sm->tu[tid] ^ g) != sm->xh[tid]) : ((g ^ sm->tu[tid]) != 0u);
                    }
                    converged = !__syncthreads_or(mm || mm1);
                }
            }
            const int stop = (gfr >= N2) ? 2 : (converged ? 1 : 0);
            // the second half completed the frame mid-sweep: the first half's
            // stages after that point are not the reference's
            if (rank == 0 && gfr >= N2 && !hfz && cut < M) act -= recount_from(cut);
            __syncthreads();  // decided_u of the last commits
            uint32_t u;
            const int r0 = P * tid;
            if (gfr >= N2) u = (sm->dec[r0 >> 5] >> (r0 & 31)) & low_mask(P);
            else u = u_group(frontier);
            uint32_t word = u << (r0 & 31);
#pragma unroll
            for (int o = 1; o < 32 / P; o <<= 1) word |= __shfl_xor_sync(kFull, word, o);
            int berr = 0;
            if ((r0 & 31) == 0) {
                const int wi = rank * NW + (r0 >> 5);
                if (args.u_bits) args.u_bits[f * 2 * NW + wi] = word;
                if (args.truth_u) berr = __popc((word ^ args.truth_u[f * 2 * NW + wi]) & ~args.frozen_bits[wi]);
            }
            berr = __reduce_add_sync(kFull, berr);
            const unsigned wact = __reduce_add_sync(kFull, act);
            if (lane == 0) {
                sm->buf[2 * warp] = (uint32_t)berr;
                sm->buf[2 * warp + 1] = wact;
            }
            __syncthreads();
            long long pe = 0;
            int be = 0;
            if (tid == 0) {
                for (int w = 0; w < PL::NWARP; ++w) {
                    be += (int)sm->buf[2 * w];
                    pe += sm->buf[2 * w + 1];
                }
                if (rank == 1) {
                    st_peer(peer_addr(&sm->pfin[0]), (long long)be);
                    st_peer(peer_addr(&sm->pfin[1]), pe);
                    st_peer(peer_addr(&sm->pfin[2]), (long long)nev);
                }
            }
            cluster_sync();
            if (rank == 0 && tid == 0) {
                be += (int)sm->pfin[0];
                pe += sm->pfin[1];
                const int ne = nev + (int)sm->pfin[2];
                if (args.iters) args.iters[f] = iters;
                if (args.pe) args.pe[f] = pe;
                if (args.stop) args.stop[f] = (uint8_t)stop;
                if (args.nev) args.nev[f] = ne;
                if (args.counters) {
                    unsigned long long* cs = counter_set(args, f);
                    atomicAdd(&cs[kCntFrames], 1ull);
                    atomicAdd(&cs[kCntBitErr], (unsigned long long)be);
                    atomicAdd(&cs[kCntFrameErr], be > 0 ? 1ull : 0ull);
                    atomicAdd(&cs[kCntIters], (unsigned long long)iters);
                    atomicAdd(&cs[kCntItersSq], (unsigned long long)iters * iters);
                    atomicAdd(&cs[kCntPe], (unsigned long long)pe);
                    atomicAdd(&cs[kCntEvents], (unsigned long long)ne);
                    atomicAdd(&cs[kCntStop0 + stop], 1ull);
                }
            }
        }
    }
};

// SP kernel: a 2-CTA cluster per frame of length 2^(M+1), each CTA one half
template <int M, int KIND>
__global__ void __launch_bounds__(Plan<M, true>::T, Cfg<M, true>::MINB) bp_pair_kernel(const __grid_constant__ DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char csm[];
    using PL = Plan<M, true>;
    Dec<M, KIND, false, true> dec;
    Smem<M, true>* sm = reinterpret_cast<Smem<M, true>*>(csm);
    if constexpr (PL::TMEM) {
        constexpr int COLS = Cfg<M, true>::TMEM_COLS;
        const int warp = threadIdx.x >> 5;
        if (warp == 0) tm::alloc<COLS>(&sm->tbase);
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        dec.tb = sm->tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(PL::TM_WCOLS * (warp >> 2));
        dec.run_pair(a, sm);
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        if (warp == 0) tm::dealloc<COLS>(sm->tbase);
    } else {
        dec.tb = 0;
        dec.run_pair(a, sm);
    }
}

template <int M, int KIND, bool XH = false>
__global__ void __launch_bounds__(Plan<M>::T, Cfg<M>::MINB) bp_cta_kernel(const __grid_constant__ DecodeArgs a) {
    extern __shared__ __align__(16) unsigned char csm[];
    Dec<M, KIND, XH> dec;
    Smem<M>* sm = reinterpret_cast<Smem<M>*>(csm);
    if constexpr (Plan<M>::NTM > 0) {
        constexpr int COLS = Cfg<M>::TMEM_COLS;
        const int warp = threadIdx.x >> 5;
        if (warp == 0) tm::alloc<COLS>(&sm->tbase);
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        dec.tb = sm->tbase + ((uint32_t)(32 * (warp & 3)) << 16) + (uint32_t)(Plan<M>::TM_WCOLS * (warp >> 2));
        dec.run(a, sm);
        tm::fence_before();
        __syncthreads();
        tm::fence_after();
        if (warp == 0) tm::dealloc<COLS>(sm->tbase);
    } else {
        dec.run(a, sm);
    }
}

template <int M, int KIND, bool XH>
static cudaError_t launch_tx(const DecodeArgs& a, int grid, cudaStream_t st) {
    const size_t smem = sizeof(Smem<M>);
    cudaError_t e = cudaFuncSetAttribute(bp_cta_kernel<M, KIND, XH>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    bp_cta_kernel<M, KIND, XH><<<grid, Plan<M>::T, smem, st>>>(a);
    return cudaGetLastError();
}

template <int M, int KIND>
static cudaError_t launch_t(const DecodeArgs& a, int grid, cudaStream_t st) {
    if constexpr (KIND == 2) {
        if (a.ev_xhat) return launch_tx<M, KIND, true>(a, grid, st);  // trace with x_hat
    }
    return launch_tx<M, KIND, false>(a, grid, st);
}

template <int M>
static cudaError_t launch_m(const DecodeArgs& a, int grid, cudaStream_t st) {
    switch (a.kind) {
        case 0: return launch_t<M, 0>(a, grid, st);
        case 1: return launch_t<M, 1>(a, grid, st);
        default: return launch_t<M, 2>(a, grid, st);
    }
}

// SP launch: clusters of two CTAs, as many as can be resident (one per SM
// pair), each taking frames from the queue
template <int M, int KIND>
static cudaError_t launch_pair(const DecodeArgs& a, cudaStream_t st) {
    auto k = bp_pair_kernel<M, KIND>;
    const size_t smem = sizeof(Smem<M, true>);
    static_assert(sizeof(Smem<M, true>) <= 227 * 1024, "one half-frame CTA per SM");
    cudaError_t e = cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(Plan<M, true>::T);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    // resident clusters per device, cached (host threads of pbp_simulate_sweep_multi launch concurrently)
    static std::atomic<int> cache[64];
    int dev = 0;
    e = cudaGetDevice(&dev);
    if (e != cudaSuccess) return e;
    int max_clusters = dev < 64 ? cache[dev].load(std::memory_order_relaxed) : 0;
    if (!max_clusters) {
        cfg.gridDim = dim3(2 * 148 * 4);
        int nc = 0;
        e = cudaOccupancyMaxActiveClusters(&nc, k, &cfg);
        if (e != cudaSuccess) return e;
        if (nc < 1) return cudaErrorInvalidConfiguration;
        max_clusters = nc;
        if (dev < 64) cache[dev].store(nc, std::memory_order_relaxed);
        if (getenv("PBP_PAIR_INFO")) fprintf(stderr, "pbp: bp_pair_kernel %zu B shared/CTA, %d resident clusters\n", smem, nc);
    }
    long long ncl = std::min<long long>(max_clusters, a.frames);
    if (const char* gc = getenv("PBP_GRID_CAP")) ncl = std::max(1ll, std::min(ncl, atoll(gc) / 2));  // experiments
    cfg.gridDim = dim3((unsigned)(2 * ncl));
    e = cudaLaunchKernelEx(&cfg, k, a);
    if (e != cudaSuccess) return e;
    return cudaGetLastError();
}

template <int M, int KIND>
static int occ_t() {
    int nb = 0;
    const size_t smem = sizeof(Smem<M>);
    cudaFuncSetAttribute(bp_cta_kernel<M, KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, bp_cta_kernel<M, KIND>, Plan<M>::T, smem) != cudaSuccess)
        return 0;
    return nb;
}

template <int M>
static int occ_m(int kind) {
    const int nb = kind == 0 ? occ_t<M, 0>() : kind == 1 ? occ_t<M, 1>() : occ_t<M, 2>();
    if constexpr (Plan<M>::TMEM) {
        // the occupancy API counts one CTA per SM for a kernel that allocates tensor
        // memory; CTAs whose columns fit the SM's 512 together do co-reside
        static_assert(Cfg<M>::MINB * Cfg<M>::TMEM_COLS <= 512, "TMEM columns of the resident CTAs");
        static_assert(Cfg<M>::MINB * (sizeof(Smem<M>) + 1024) <= 228 * 1024, "shared memory of the resident CTAs");
        return nb > 0 ? std::max(nb, (int)Cfg<M>::MINB) : 0;
    }
    return nb;
}

}  // namespace cta

int cta_kernel_supported(int m) { return m >= 11 && m <= 14; }

// L2-resident L levels per CTA (at least one level, so the pointer is valid)
long long cta_scratch_floats(int m) {
    switch (m) {
        case 11: return (long long)std::max(1, cta::Plan<11>::NGL) << 11;
        case 12: return (long long)std::max(1, cta::Plan<12>::NGL) << 12;
        case 13: return (long long)std::max(1, cta::Plan<13>::NGL) << 13;
        case 14: return (long long)std::max(1, cta::Plan<14>::NGL) << 14;
    }
    return 0;
}

// n = 16384 csfg decodes (no event trace) on 2-CTA clusters, one half of the
// frame per SM: every message level on chip (PBP_PAIR=0: one CTA per frame)
bool cta_pair_on(int m, int kind) {
    const char* e = getenv("PBP_PAIR");  // read per launch: tests compare both layouts in one process
    const int v = e ? atoi(e) : 1;
    // n = 4096 on pairs only as an experiment (PBP_PAIR=2, csfg): slower, see DESIGN.md section 5
    return (v && m == 14 && kind >= 0 && kind <= 2) || (v >= 2 && m == 12 && kind == 2);
}
static bool cta_pair(const DecodeArgs& a) { return cta_pair_on(a.m, a.kind) && !a.events && !a.ev_xhat; }
template <int M>
static int pair_occ() {
    auto k = cta::bp_pair_kernel<M, 2>;
    const size_t smem = sizeof(cta::Smem<M, true>);
    int nb = 0;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k, cta::Plan<M, true>::T, smem) != cudaSuccess) return 0;
    return nb;
}
int cta_pair_warps_per_sm(int m) {
    return m == 12 ? pair_occ<11>() * cta::Plan<11, true>::NWARP : pair_occ<13>() * cta::Plan<13, true>::NWARP;
}
size_t cta_pair_smem_bytes(int m) { return m == 12 ? sizeof(cta::Smem<11, true>) : sizeof(cta::Smem<13, true>); }

cudaError_t launch_cta(const DecodeArgs& a, int grid, cudaStream_t st) {
    if (cta_pair(a)) {
        if (a.m == 12) return cta::launch_pair<11, 2>(a, st);
        return a.kind == 0 ? cta::launch_pair<13, 0>(a, st)
                           : (a.kind == 1 ? cta::launch_pair<13, 1>(a, st) : cta::launch_pair<13, 2>(a, st));
    }
    switch (a.m) {
        case 11: return cta::launch_m<11>(a, grid, st);
        case 12: return cta::launch_m<12>(a, grid, st);
        case 13: return cta::launch_m<13>(a, grid, st);
        case 14: return cta::launch_m<14>(a, grid, st);
    }
    return cudaErrorInvalidValue;
}

size_t cta_smem_bytes(int m) {
    switch (m) {
        case 11: return sizeof(cta::Smem<11>);
        case 12: return sizeof(cta::Smem<12>);
        case 13: return sizeof(cta::Smem<13>);
        case 14: return sizeof(cta::Smem<14>);
    }
    return 0;
}

int cta_warps(int m) { return m >= 11 && m <= 14 ? 1 << (m - 4 - 5) : 0; }  // 16 rows per thread

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
