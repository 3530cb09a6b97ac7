/*
 * TEST INFRASTRUCTURE ONLY -- see pbp_oracle.h. Plain-C restatement of the
 * reference's code construction, channel and BP decoders. Not product code.
 */
#include "pbp_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdatomic.h>
#include <stdlib.h>
#include <string.h>

static int is_pow2(int v) { return v > 0 && (v & (v - 1)) == 0; }

static int log2i(int n) {
    int m = 0;
    while ((1 << m) < n) ++m;
    return m;
}

/* polar_code.cpp:13-20 -- natural-order butterfly x = u F^{(x)m}: for each
 * half = 1, 2, 4, ..., every index i with bit `half` clear absorbs i+half. */
int orc_polar_transform(uint8_t* v, int n) {
    if (!is_pow2(n)) return -1;
    for (int half = 1; half < n; half <<= 1)
        for (int i = 0; i < n; ++i)
            if (!(i & half)) v[i] ^= v[i + half];
    return 0;
}

/* polar_code.cpp:27-43 -- Bhattacharyya recursion, strides n/2 .. 1;
 * the lower index of each pair receives 2z - z^2, the upper z^2. */
static void bhattacharyya(int n, double z0, double* z) {
    for (int i = 0; i < n; ++i) z[i] = z0;
    for (int half = n / 2; half >= 1; half /= 2)
        for (int i = 0; i < n; ++i) {
            if (i & half) continue;
            const double zi = z[i];
            z[i] = 2.0 * zi - zi * zi;
            z[i + half] = zi * zi;
        }
}

static const double* g_sort_z;
/* polar_code.cpp:57-60 -- descending z, ties by ascending index */
static int worse_first(const void* a, const void* b) {
    const int ia = *(const int*)a, ib = *(const int*)b;
    const double za = g_sort_z[ia], zb = g_sort_z[ib];
    if (za != zb) return za > zb ? -1 : 1;
    return ia < ib ? -1 : (ia > ib);
}

/* polar_code.cpp:53-66 -- freeze the n-k least reliable rows.
 * (qsort with a total order gives the same set as std::sort.) */
int orc_construct(int n, int k, double design_z, uint8_t* frozen_out) {
    if (!is_pow2(n) || k < 1 || k > n || !(design_z > 0.0 && design_z < 1.0)) return -1;
    double* z = (double*)malloc(sizeof(double) * (size_t)n);
    int* order = (int*)malloc(sizeof(int) * (size_t)n);
    bhattacharyya(n, design_z, z);
    for (int i = 0; i < n; ++i) order[i] = i;
    g_sort_z = z;
    qsort(order, (size_t)n, sizeof(int), worse_first);
    memset(frozen_out, 0, (size_t)n);
    for (int i = 0; i < n - k; ++i) frozen_out[order[i]] = 1;
    free(z);
    free(order);
    return 0;
}

/* polar_code.cpp:82-91 -- info bits fill unfrozen rows in ascending order */
int orc_encode(int n, const uint8_t* frozen, const uint8_t* info, uint8_t* u_out, uint8_t* x_out) {
    if (!is_pow2(n)) return -1;
    int next = 0;
    for (int i = 0; i < n; ++i) u_out[i] = frozen[i] ? 0 : info[next++];
    memcpy(x_out, u_out, (size_t)n);
    return orc_polar_transform(x_out, n);
}

/* ---- channel.cpp ------------------------------------------------------- */

/* channel.cpp:20-27 -- splitmix64 finalizer */
static uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ULL;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBULL;
    z ^= z >> 31;
    return z;
}

/* std::mt19937_64 (libstdc++ GCC 13 random.tcc: seed() and _M_gen_rand()),
 * parameters w=64 n=312 m=156 r=31 a=0xb5026f5aa96619e9 u=29
 * d=0x5555555555555555 s=17 b=0x71d67fffeda60000 t=37
 * c=0xfff7eee000000000 l=43 f=6364136223846793005. */
#define MT_N 312
#define MT_M 156
static void mt_seed(orc_mt64* g, uint64_t s) {
    g->mt[0] = s;
    for (int i = 1; i < MT_N; ++i)
        g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = MT_N;
}

static void mt_twist(orc_mt64* g) {
    const uint64_t upper = ~(uint64_t)0 << 31, lower = ~upper;
    for (int i = 0; i < MT_N; ++i) {
        const uint64_t y = (g->mt[i] & upper) | (g->mt[(i + 1) % MT_N] & lower);
        g->mt[i] = g->mt[(i + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1) ? 0xB5026F5AA96619E9ULL : 0);
    }
    g->idx = 0;
}

uint64_t orc_mt64_next(orc_mt64* g) {
    if (g->idx >= MT_N) mt_twist(g);
    uint64_t z = g->mt[g->idx++];
    z ^= (z >> 29) & 0x5555555555555555ULL;
    z ^= (z << 17) & 0x71D67FFFEDA60000ULL;
    z ^= (z << 37) & 0xFFF7EEE000000000ULL;
    z ^= z >> 43;
    return z;
}

/* channel.cpp:31-32 -- one stream per (master seed, trial) */
void orc_trial_rng(orc_mt64* g, uint64_t master_seed, uint64_t trial) {
    mt_seed(g, mix64(master_seed + 0x9E3779B97F4A7C15ULL * (trial + 1)));
}

/* channel.cpp:34-39 -- Box-Muller cosine branch, two draws per sample:
 * u1 in (0,1], u2 in [0,1), 53-bit mantissas, glibc libm log/cos/sqrt. */
double orc_gaussian(orc_mt64* g) {
    const double u1 = (double)((orc_mt64_next(g) >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(orc_mt64_next(g) >> 11) * 0x1.0p-53;
    return sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
}

/* channel.cpp:9-15 */
double orc_noise_variance(double ebn0_db, double rate) {
    return 1.0 / (2.0 * rate * pow(10.0, ebn0_db / 10.0));
}

/* sim_harness.cpp:67-73 -> channel.cpp:41 (bit = top bit of a draw),
 * polar_code.cpp:82-91 (encode), channel.cpp:43-60 (BPSK 0->+1, AWGN,
 * LLR = (2/sigma^2) * y). */
int orc_trial_frame(uint64_t seed, uint64_t trial, int n, const uint8_t* frozen, double ebn0_db,
                    int noiseless, uint8_t* info_out, double* llr_out) {
    if (!is_pow2(n)) return -1;
    int k = 0;
    for (int i = 0; i < n; ++i) k += frozen[i] ? 0 : 1;
    orc_mt64 g;
    orc_trial_rng(&g, seed, trial);
    uint8_t* info = (uint8_t*)malloc((size_t)k + 1);
    uint8_t* u = (uint8_t*)malloc((size_t)n);
    uint8_t* x = (uint8_t*)malloc((size_t)n);
    for (int b = 0; b < k; ++b) info[b] = (uint8_t)(orc_mt64_next(&g) >> 63);
    orc_encode(n, frozen, info, u, x);
    const double sigma2 = orc_noise_variance(ebn0_db, (double)k / n);
    const double sigma = sqrt(sigma2);
    const double scale = 2.0 / sigma2;
    for (int i = 0; i < n; ++i) {
        const double s = x[i] ? -1.0 : 1.0;
        const double y = noiseless ? s : s + sigma * orc_gaussian(&g);
        llr_out[i] = scale * y;
    }
    if (info_out) memcpy(info_out, info, (size_t)k);
    free(info);
    free(u);
    free(x);
    return 0;
}

/* ---- decoders, instantiated for float and double ------------------------ */

#define REAL float
#define SUF(name) name##_f32
#define CAP_VALUE 1e30f
#include "pbp_oracle_real.inc"
#undef REAL
#undef SUF
#undef CAP_VALUE

#define REAL double
#define SUF(name) name##_f64
#define CAP_VALUE 1e30
#include "pbp_oracle_real.inc"
#undef REAL
#undef SUF
#undef CAP_VALUE
