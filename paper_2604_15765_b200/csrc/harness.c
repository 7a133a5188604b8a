/*
 * harness.c -- seeded synthetic inputs for the BASELINE.json configs.
 *
 * Host-only C, no CUDA: shared by the GPU arm (which uploads psi / Pauli data and lets
 * hs_state_fill_* build the payload on the device), the CPU reference arm and the tests, so
 * every engine sees bit-identical inputs.  Compiled with -ffp-contract=off: the payload
 * builders below perform exactly the rounded operations of the device generators in
 * engine.cu (fill_mixture_kernel, fill_pauli_kernel).
 *
 * RNG: the reference's counter-based gaussian_entry (storage.cpp:22-44), restated.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

static uint64_t splitmix64(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}

void hsg_gaussian_entry(uint64_t seed, uint64_t counter, double out[2]) {
    const uint64_t base = splitmix64(seed ^ 0xD6E8FEB86659FD93ull);
    const uint64_t r1 = splitmix64(base + 2 * counter);
    const uint64_t r2 = splitmix64(base + 2 * counter + 1);
    const double u1 = (double)((r1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    const double phi = 2.0 * 3.141592653589793238462643383279502884 * u2;
    out[0] = r * cos(phi);
    out[1] = r * sin(phi);
}

/* Uniform double in [0, 1) from a (seed, counter) stream. */
double hsg_uniform(uint64_t seed, uint64_t counter) {
    const uint64_t r = splitmix64(splitmix64(seed ^ 0x5851F42D4C957F2Dull) + counter);
    return (double)(r >> 11) * 0x1.0p-53;
}

/* psi_i[x] = gaussian_entry(seed + i, x) / ||.||, i < rank; norms summed in index order. */
void hsg_rank_psi(int n, uint64_t seed, int rank, double* psi) {
    const uint64_t N = UINT64_C(1) << n;
    for (int i = 0; i < rank; ++i) {
        double* p = psi + 2 * (uint64_t)i * N;
        double ss = 0.0;
        for (uint64_t x = 0; x < N; ++x) {
            hsg_gaussian_entry(seed + (uint64_t)i, x, p + 2 * x);
            ss += p[2 * x] * p[2 * x] + p[2 * x + 1] * p[2 * x + 1];
        }
        const double nrm = sqrt(ss);
        for (uint64_t x = 0; x < 2 * N; ++x)
            p[x] /= nrm;
    }
}

static uint64_t payload_count(int n, int m, uint64_t* grid) {
    const uint64_t N = UINT64_C(1) << n, M = UINT64_C(1) << m;
    const uint64_t G = N >= M ? N / M : 1;
    if (grid)
        *grid = G;
    return G * (G + 1) / 2 * M * M;
}

uint64_t hsg_payload_count(int n, int m) { return payload_count(n, m, NULL); }

/* Tiled payload of rho = (1/rank) sum_i |psi_i><psi_i| over tiles [t0, t1) (storage.hpp:60-96
 * layout); every element directly (diagonal tiles included), same rounding as the device. */
void hsg_rho_payload_range(int n, int m, int rank, const double* psi, double* payload, uint64_t t0, uint64_t t1) {
    const uint64_t N = UINT64_C(1) << n, M = UINT64_C(1) << m;
    const double inv = 1.0 / rank;
    uint64_t ti = 0, tj = 0;
    {  /* decode t0 */
        uint64_t r = (uint64_t)((sqrt(1.0 + 8.0 * (double)t0) - 1.0) * 0.5);
        while (r * (r + 1) / 2 > t0)
            --r;
        while ((r + 1) * (r + 2) / 2 <= t0)
            ++r;
        ti = r;
        tj = t0 - r * (r + 1) / 2;
    }
    for (uint64_t t = t0; t < t1; ++t) {
        double* tp = payload + 2 * (t - t0) * M * M;
        for (uint64_t r = 0; r < M; ++r)
            for (uint64_t c = 0; c < M; ++c) {
                const uint64_t i = ti * M + r, j = tj * M + c;
                double ar = 0.0, ai = 0.0;
                if (i < N && j < N) {
                    for (int a = 0; a < rank; ++a) {
                        const double* p = psi + 2 * ((uint64_t)a * N + i);
                        const double* q = psi + 2 * ((uint64_t)a * N + j);
                        const double re = p[0] * q[0] + p[1] * q[1];
                        const double im = p[1] * q[0] - p[0] * q[1];
                        ar = ar + re;
                        ai = ai + im;
                    }
                    ar = ar * inv;
                    ai = ai * inv;
                }
                tp[2 * (r * M + c)] = ar;
                tp[2 * (r * M + c) + 1] = ai;
            }
        if (++tj > ti) {
            ++ti;
            tj = 0;
        }
    }
}

void hsg_rho_payload(int n, int m, int rank, const double* psi, double* payload) {
    uint64_t G;
    payload_count(n, m, &G);
    hsg_rho_payload_range(n, m, rank, psi, payload, 0, G * (G + 1) / 2);
}

/* Isometry V (rows x cols, rows >= cols, V^dagger V = I): modified Gram-Schmidt QR of
 * Z = gaussian_entry(seed, r * cols + c) / sqrt2 (row-major), columns orthonormalised in order;
 * R's diagonal is then real positive, i.e. the phase-fixed Q = Q diag(R_ii / |R_ii|) of Mezzadri's
 * recipe.  Returns 0, or -1 for an invalid shape. */
int hsg_isometry(int rows, int cols, uint64_t seed, double* u) {
    if (rows < 1 || cols < 1 || cols > rows || rows > 4096)
        return -1;
    double* z = (double*)malloc((size_t)rows * cols * 2 * sizeof(double));
    if (!z)
        return -1;
#define Z(r, c) z[((size_t)(r) * cols + (c)) * 2]
#define ZI(r, c) z[((size_t)(r) * cols + (c)) * 2 + 1]
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
            double g[2];
            hsg_gaussian_entry(seed, (uint64_t)r * cols + c, g);
            Z(r, c) = g[0] / sqrt(2.0);
            ZI(r, c) = g[1] / sqrt(2.0);
        }
    for (int c = 0; c < cols; ++c) {
        for (int p = 0; p < c; ++p) { /* z[:,c] -= <q_p, z[:,c]> q_p */
            double dr = 0.0, di = 0.0;
            for (int r = 0; r < rows; ++r) { /* conj(q) * z */
                const double qr = Z(r, p), qi = ZI(r, p), vr = Z(r, c), vi = ZI(r, c);
                dr += qr * vr + qi * vi;
                di += qr * vi - qi * vr;
            }
            for (int r = 0; r < rows; ++r) {
                const double qr = Z(r, p), qi = ZI(r, p);
                Z(r, c) -= dr * qr - di * qi;
                ZI(r, c) -= dr * qi + di * qr;
            }
        }
        double ss = 0.0;
        for (int r = 0; r < rows; ++r)
            ss += Z(r, c) * Z(r, c) + ZI(r, c) * ZI(r, c);
        const double nrm = sqrt(ss);
        for (int r = 0; r < rows; ++r) {
            Z(r, c) /= nrm;
            ZI(r, c) /= nrm;
        }
    }
#undef Z
#undef ZI
    memcpy(u, z, (size_t)rows * cols * 2 * sizeof(double));
    free(z);
    return 0;
}

/* Haar-random 2^k x 2^k unitary (k <= 6): the square isometry. */
void hsg_haar(int k, uint64_t seed, double* u) {
    const int d = 1 << k;
    (void)hsg_isometry(d, d, seed, u);
}

/* Fisher-Yates permutation of [0, n) from the (seed, counter) uniform stream. */
void hsg_permutation(int n, uint64_t seed, uint32_t* out) {
    for (int i = 0; i < n; ++i)
        out[i] = (uint32_t)i;
    for (int i = n - 1; i > 0; --i) {
        const int j = (int)(hsg_uniform(seed, (uint64_t)i) * (double)(i + 1));
        const uint32_t t = out[i];
        out[i] = out[j];
        out[j] = t;
    }
}

/* `count` Pauli strings on n qubits: per qubit uniform I/X/Y/Z from the uniform stream,
 * coefficient Re gaussian_entry(seed, s) (N(0,1)); x = X|Y mask, z = Z|Y mask, ny = #Y. */
void hsg_pauli_strings(int n, int count, uint64_t seed, uint64_t* x, uint64_t* z, int32_t* ny, double* coef) {
    for (int s = 0; s < count; ++s) {
        uint64_t xm = 0, zm = 0;
        int y = 0;
        for (int q = 0; q < n; ++q) {
            const int code = (int)(hsg_uniform(seed + 1, (uint64_t)s * 64 + q) * 4.0);
            if (code == 1 || code == 2)
                xm |= UINT64_C(1) << q;
            if (code == 3 || code == 2)
                zm |= UINT64_C(1) << q;
            if (code == 2)
                ++y;
        }
        double g[2];
        hsg_gaussian_entry(seed, (uint64_t)s, g);
        x[s] = xm;
        z[s] = zm;
        ny[s] = y;
        coef[s] = g[0];
    }
}

/* Tiled payload of O = sum_s coef_s P_s, P_s(i, j) = [i ^ j == x_s] i^ny (-1)^popcount(j & z_s),
 * strings summed in index order (bit-identical to fill_pauli_kernel). */
void hsg_pauli_payload(int n, int m, int count, const uint64_t* x, const uint64_t* z, const int32_t* ny,
                       const double* coef, double* payload) {
    uint64_t G;
    const uint64_t cnt = payload_count(n, m, &G);
    const uint64_t N = UINT64_C(1) << n, M = UINT64_C(1) << m;
    memset(payload, 0, cnt * 16);
    for (uint64_t ti = 0; ti < G; ++ti)
        for (uint64_t tj = 0; tj <= ti; ++tj) {
            double* tp = payload + 2 * (ti * (ti + 1) / 2 + tj) * M * M;
            for (uint64_t r = 0; r < M; ++r)
                for (uint64_t c = 0; c < M; ++c) {
                    const uint64_t i = ti * M + r, j = tj * M + c;
                    if (i >= N || j >= N)
                        continue;
                    double ar = 0.0, ai = 0.0;
                    for (int s = 0; s < count; ++s) {
                        if (x[s] != (i ^ j))
                            continue;
                        double v = coef[s];
                        if (__builtin_popcountll(j & z[s]) & 1)
                            v = -v;
                        switch (ny[s] & 3) {
                        case 0: ar = ar + v; break;
                        case 1: ai = ai + v; break;
                        case 2: ar = ar + -v; break;
                        default: ai = ai + -v; break;
                        }
                    }
                    tp[2 * (r * M + c)] = ar;
                    tp[2 * (r * M + c) + 1] = ai;
                }
        }
}
