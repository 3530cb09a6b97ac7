// On-device frame generation, identical stream layout to the reference's
// decode_trial (src/sim_harness.cpp:67-73):
//   TrialRng(seed, trial) = std::mt19937_64(mix64(seed + 0x9E37..15 * (trial+1)))
//                                                       (src/channel.cpp:20-32)
//   K draws -> info bits (top bit, channel.cpp:41), placed on the unfrozen
//   rows in ascending order and encoded (polar_code.cpp:82-91);
//   then per symbol two draws -> Box-Muller cosine branch (channel.cpp:34-39),
//   y = s + sigma * g, LLR = (2/sigma^2) * y in fp64 (channel.cpp:49-60).
// Seeding the 312-word state is a serial recurrence per trial, so it runs
// lane-per-trial in channel_seed_kernel (32 trials per warp, states written
// trial-major to a scratch through a shared-memory transpose); the generation
// kernel then runs one warp per trial: coalesced state load, the twist
// warp-parallel in the three phases of libstdc++'s _M_gen_rand, tempering and
// consumption lane-parallel. Integer state is
// bit-exact; the fp64 log/cos are CUDA's (<= 2 ulp), which the parity tests
// compare against glibc on the host (fp32 LLRs are what the decoder sees).
#include "pbp_common.cuh"

namespace pbp {


namespace {

constexpr int kMtN = 312, kMtM = 156;
constexpr unsigned long long kUpper = ~0ull << 31, kLower = ~kUpper;
constexpr unsigned long long kMatA = 0xB5026F5AA96619E9ull;
constexpr int kGenWarps = 4;

__device__ __forceinline__ unsigned long long mix64(unsigned long long z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}

__device__ __forceinline__ unsigned long long twist1(unsigned long long a, unsigned long long b) {
    const unsigned long long y = (a & kUpper) | (b & kLower);
    return (y >> 1) ^ ((y & 1ull) ? kMatA : 0ull);
}

__device__ __forceinline__ unsigned long long temper(unsigned long long z) {
    z ^= (z >> 29) & 0x5555555555555555ull;
    z ^= (z << 17) & 0x71D67FFFEDA60000ull;
    z ^= (z << 37) & 0xFFF7EEE000000000ull;
    z ^= z >> 43;
    return z;
}

// warp-parallel _M_gen_rand: read-all / syncwarp / write-all per phase
__device__ void mt_twist(unsigned long long* mt, int lane) {
    unsigned long long v[5];
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const int i = lane + 32 * c;
        if (i < kMtN - kMtM) v[c] = mt[i + kMtM] ^ twist1(mt[i], mt[i + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const int i = lane + 32 * c;
        if (i < kMtN - kMtM) mt[i] = v[c];
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const int i = kMtN - kMtM + lane + 32 * c;
        if (i < kMtN - 1) v[c] = mt[i - (kMtN - kMtM)] ^ twist1(mt[i], mt[i + 1]);
    }
    __syncwarp();
#pragma unroll
    for (int c = 0; c < 5; ++c) {
        const int i = kMtN - kMtM + lane + 32 * c;
        if (i < kMtN - 1) mt[i] = v[c];
    }
    __syncwarp();
    if (lane == 0) mt[kMtN - 1] = mt[kMtM - 1] ^ twist1(mt[kMtN - 1], mt[0]);
    __syncwarp();
}

// polar transform of nbits bits in nw words of shared memory, one warp
__device__ void warp_transform_words(uint32_t* w, int nbits, int lane) {
    const int nw = (nbits + 31) >> 5;
    for (int q = lane; q < nw; q += 32) w[q] = word_transform(w[q], nbits);
    __syncwarp();
    for (int h = 1; h < nw; h <<= 1) {
        for (int p = lane; p < nw / 2; p += 32) {
            const int q = ((p / h) * 2 * h) + (p % h);
            w[q] ^= w[q + h];
        }
        __syncwarp();
    }
}

__device__ __forceinline__ double box_muller(unsigned long long d1, unsigned long long d2) {
    const double u1 = __dmul_rn((double)((d1 >> 11) + 1ull), 0x1.0p-53);
    const double u2 = __dmul_rn((double)(d2 >> 11), 0x1.0p-53);
    // 2.0 * pi * u2 evaluated left to right: 2*pi is exact.
    return __dmul_rn(sqrt(__dmul_rn(-2.0, log(u1))),
                     cos(__dmul_rn(6.283185307179586476925286766559, u2)));
}

}  // namespace

// std::mt19937_64 seeding (x_i = 6364136223846793005 (x ^ x >> 62) + i) of
// TrialRng(seed, first + t) for t < count, one lane per trial; mt_out[t][312].
// Each lane produces 8 words at a time into a padded shared tile, then the warp
// stores 4 trials x 64 contiguous bytes per instruction.
__global__ void __launch_bounds__(kGenWarps * 32) channel_seed_kernel(unsigned long long seed, long long first,
                                                                       long long count, unsigned long long* mt_out) {
    __shared__ unsigned long long tile[kGenWarps][32][9];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long long t0 = ((long long)blockIdx.x * kGenWarps + warp) * 32;
    if (t0 >= count) return;
    const unsigned long long trial = (unsigned long long)(first + t0 + lane);
    unsigned long long x = mix64(seed + 0x9E3779B97F4A7C15ull * (trial + 1ull));
    auto& tl = tile[warp];
    for (int i0 = 0; i0 < kMtN; i0 += 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (i0 + j > 0) x = 6364136223846793005ull * (x ^ (x >> 62)) + (unsigned long long)(i0 + j);
            tl[lane][j] = x;
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            const int tt = 4 * q + (lane >> 3), j = lane & 7;
            if (t0 + tt < count) mt_out[(t0 + tt) * kMtN + i0 + j] = tl[tt][j];
        }
        __syncwarp();
    }
}

__global__ void __launch_bounds__(kGenWarps * 32) channel_gen_kernel(GenArgs g) {
    extern __shared__ unsigned long long gsm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nw = (g.n + 31) >> 5;
    unsigned long long* mt = gsm + warp * (2 * kMtN + 1);
    unsigned long long* outv = mt + kMtN;
    unsigned long long* carry = outv + kMtN;
    uint32_t* words = reinterpret_cast<uint32_t*>(gsm + kGenWarps * (2 * kMtN + 1)) + warp * 2 * nw;
    uint32_t* uw = words;
    uint32_t* xw = words + nw;
    const long long total_warps = (long long)gridDim.x * kGenWarps;
    const int draws = g.k + 2 * g.n;

    for (long long it = (long long)blockIdx.x * kGenWarps + warp; it < g.count; it += total_warps) {
        for (int i = lane; i < kMtN; i += 32) mt[i] = __ldcs(g.mt0 + it * kMtN + i);
        for (int q = lane; q < nw; q += 32) uw[q] = 0u;
        __syncwarp();
        bool encoded = false;
        for (int base = 0; base < draws; base += kMtN) {
            mt_twist(mt, lane);
            for (int i = lane; i < kMtN; i += 32) outv[i] = temper(mt[i]);
            __syncwarp();
            // info bits: draws [0, k)
            for (int i = lane; i < kMtN; i += 32) {
                const int d = base + i;
                if (d < g.k && (outv[i] >> 63)) {
                    const int r = g.info_rows[d];
                    atomicOr(&uw[r >> 5], 1u << (r & 31));
                }
            }
            __syncwarp();
            if (!encoded && base + kMtN >= g.k) {
                for (int q = lane; q < nw; q += 32) {
                    xw[q] = uw[q];
                    if (g.u_out) g.u_out[(long long)it * nw + q] = uw[q];
                }
                __syncwarp();
                warp_transform_words(xw, g.n, lane);
                encoded = true;
            }
            // symbols: symbol j uses draws k+2j (u1) and k+2j+1 (u2)
            const int j_lo = (base + 0 - g.k) >= 0 ? (base - g.k) >> 1 : 0;
            for (int j = j_lo + lane;; j += 32) {
                const int d1 = g.k + 2 * j;
                if (d1 >= base + kMtN || j >= g.n) break;
                if (d1 + 1 < base) continue;
                unsigned long long v1, v2;
                if (d1 < base) {  // u1 in the previous block (saved)
                    v1 = *carry;
                    v2 = outv[d1 + 1 - base];
                } else if (d1 + 1 >= base + kMtN) {
                    continue;  // u2 in the next block: handled there
                } else {
                    v1 = outv[d1 - base];
                    v2 = outv[d1 + 1 - base];
                }
                const double sym = ((xw[j >> 5] >> (j & 31)) & 1u) ? -1.0 : 1.0;
                const double y = g.noiseless ? sym : __dadd_rn(sym, __dmul_rn(g.sigma, box_muller(v1, v2)));
                const double l = __dmul_rn(g.scale, y);
                if (g.llr) g.llr[(long long)it * g.n + j] = __double2float_rn(l);
                if (g.llr64) g.llr64[(long long)it * g.n + j] = l;
            }
            __syncwarp();
            if (lane == 0) *carry = outv[kMtN - 1];
            __syncwarp();
        }
    }
}

size_t channel_smem_bytes(int n) {
    const int nw = (n + 31) / 32;
    return (size_t)kGenWarps * (2 * kMtN + 1) * 8 + (size_t)kGenWarps * 2 * nw * 4;
}

long long channel_seed_words(long long count) { return count * kMtN; }

cudaError_t launch_channel(const GenArgs& g, int grid, cudaStream_t stream) {
    {
        const long long warps = (g.count + 31) / 32;
        channel_seed_kernel<<<(unsigned)((warps + kGenWarps - 1) / kGenWarps), kGenWarps * 32, 0, stream>>>(
            g.seed, g.first, g.count, g.mt0);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return e;
    }
    const size_t smem = channel_smem_bytes(g.n);
    if (smem > 48 * 1024) {
        cudaError_t e = cudaFuncSetAttribute(channel_gen_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
    }
    channel_gen_kernel<<<grid, kGenWarps * 32, smem, stream>>>(g);
    return cudaGetLastError();
}

}  // namespace pbp
