// Shared device-side definitions for the B200 polar BP decoder.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace pbp {

// LLR_CAP (include/polarbp/bp_core.hpp:21) as fp32, the "ref32" value.
constexpr float kCap = 1e30f;
// |LLR| bound under which no clamp of the reference can bind (DESIGN.md
// "clamp elision"): |R(s)| <= 2^s * max|LLR| <= 2^24 * 1e14 < 3.8e22 =
// ulp(CAP)/2, so every CAP +- finite sum rounds back to +-CAP and every
// product term stays <= alpha * CAP. Frames outside it (or non-finite) are
// decoded by the generic kernel, which keeps every clamp.
constexpr float kClampFreeBound = 1e14f;
constexpr uint8_t kNotFrozen = 0x7f;  // kNotFrozen (csfg_freeze.hpp:37) as a byte

// Counter slots (pbp_counters in include/pbp.h)
enum : int {
    kCntFrames = 0, kCntBitErr, kCntFrameErr, kCntIters, kCntItersSq, kCntPe, kCntEvents,
    kCntStop0, kCntStop1, kCntStop2, kNumCounters
};

struct DecodeArgs {
    int n, m, kind, max_iter;
    float alpha;
    const uint32_t* frozen_bits;  // device, ceil(n/32) words
    const uint8_t* frozen_rows;   // device, n bytes
    const float* llr;             // frames x n
    const double* llr64;          // frames x n: decode in fp64 (generic kernel only)
    double alpha64;
    long long frames;
    // per-frame outputs (device, nullable)
    uint32_t* u_bits;
    int* iters;
    long long* pe;
    uint8_t* stop;
    int* nev;
    int* events;  // frames x ev_cap x 5 (nullable)
    int ev_cap;
    // frames x ev_cap x ceil(n/32) words, zeroed (nullable): each event's x_hat,
    // the block's hard decisions at its rows (FreezeEvent::x_hat)
    uint32_t* ev_xhat;
    // counters mode (nullable)
    const uint32_t* truth_u;          // frames x ceil(n/32)
    unsigned long long* counters;     // kNumCounters (cnt_batch > 0: one set per cnt_batch frames)
    int cnt_batch;                    // 0: one counter set; > 0: set f / cnt_batch for frame f
    // work distribution
    unsigned long long* queue;        // atomic frame counter (zeroed before launch)
    // re-route list: the fast kernel appends frames it cannot take; the
    // generic kernel consumes it when list_mode != 0.
    long long* list;                  // frame indices + frame_base
    unsigned long long* list_len;
    long long frame_base;             // index of this launch's frame 0 in the list's numbering
    int list_mode;
    float* r0s;                       // warp kernel: per-CTA channel LLRs (n floats each)
    float* scratch;                   // generic kernel: per-CTA message arrays
    long long scratch_stride;         // floats per CTA
};

// channel generation (channel.cu)
struct GenArgs {
    int n, k;
    unsigned long long seed;
    long long first, count;
    double sigma, scale;  // sqrt(sigma^2), 2/sigma^2 from the host (channel.cpp:53-55)
    int noiseless;
    const int* info_rows;  // k entries: row of the b-th info bit
    float* llr;            // count x n (nullable)
    double* llr64;         // count x n (nullable)
    uint32_t* u_out;       // count x ceil(n/32) (nullable)
    unsigned long long* mt0;  // count x 312 scratch: the seeded mt19937_64 states
};

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// counter set of frame f (its run_point batch when the caller asked for
// per-batch sums: the host applies the reference's stop rule on them)
__device__ __forceinline__ unsigned long long* counter_set(const DecodeArgs& a, long long f) {
    return a.cnt_batch > 0 ? a.counters + (f / a.cnt_batch) * kNumCounters : a.counters;
}

// XOR butterfly of the polar transform (polar_code.cpp:13-20) restricted to
// bit positions h < nbits inside one 32-bit word: bit i (with i&h == 0)
// absorbs bit i+h.
__device__ __forceinline__ uint32_t word_transform(uint32_t w, int nbits) {
    if (nbits > 1) w ^= (w >> 1) & 0x55555555u;
    if (nbits > 2) w ^= (w >> 2) & 0x33333333u;
    if (nbits > 4) w ^= (w >> 4) & 0x0F0F0F0Fu;
    if (nbits > 8) w ^= (w >> 8) & 0x00FF00FFu;
    if (nbits > 16) w ^= (w >> 16) & 0x0000FFFFu;
    return w;
}

__device__ __forceinline__ uint32_t low_mask(int nbits) {
    return nbits >= 32 ? 0xffffffffu : ((1u << nbits) - 1u);
}

}  // namespace pbp
