// engine_convert.cuh -- part of engine.cu (one translation unit; included after the state type).
// Format conversions on the device: the reference's to_dense / convert
// (storage.cpp:241-292) between the tiled lower triangle and the dense row-major N x N matrix or the
// column-major packed lower triangle, and between tiled layouts of different tile exponents.
//
// Semantics follow the reference exactly (so results are bit-identical, not just close):
//   to_dense(tiled):  d(i, j) = tile element for i, j in the same (diagonal) tile -- "diagonal tile
//                     holds both halves" (storage.cpp:271-273) -- else the stored lower element or
//                     the conjugate of its mirror;
//   convert(.., packed / tiled):  fill_from_lower(gen = to_dense(src).at) (storage.cpp:149-189,
//                     285-292): stored (i >= j) = d(i, j); a tiled target's diagonal-tile upper half
//                     = conj(d(j, i)); padding (N < M) = 0;
//   to_dense(packed): d(i, j) = P(i, j), d(j, i) = conj(P(i, j)), so d(i, i) = conj(P(i, i)).
// HBM layout: every kernel moves whole 32 x 32 (or M x M) blocks through shared memory so both the
// read and the write side are coalesced rows of >= 128 B (the transposed half of a dense matrix is
// written from the staged stored tile, the packed columns are read / written along rows i).  Pure
// streams: algorithmic bytes = read once + write once of each side.
#pragma once

namespace {
constexpr int CV_T = 256;  // threads per CTA of the conversion kernels

__device__ __forceinline__ uint64_t packed_off(uint64_t N, uint64_t j) { return j * N - j * (j - 1) / 2; }

// element (i, j) of the logical matrix as to_dense reads it from a tiled payload (m: tile exponent)
__device__ __forceinline__ double2 tiled_at(const double2* __restrict__ d, uint32_t m, uint64_t i, uint64_t j) {
    const uint64_t ti = i >> m, tj = j >> m, mk = (1ull << m) - 1;
    if (ti >= tj)
        return d[((tri(ti) + tj) << (2 * m)) + ((i & mk) << m) + (j & mk)];
    return cconj(d[((tri(tj) + ti) << (2 * m)) + ((j & mk) << m) + (i & mk)]);
}

// Tiled -> dense rows [ti0 * M, ti1 * M) (out points at row ti0 * M).  Work items: (a) every stored
// tile of tile rows [ti0, ti1) written in place (direct), (b) every stored tile (T, t) with t in
// [ti0, ti1), T > t, written conjugate-transposed into rows of tile row t.  E = min(M, N).
__global__ void __launch_bounds__(CV_T) to_dense_kernel(const double2* __restrict__ src, uint32_t m, uint64_t N,
                                                        uint64_t G, uint64_t ti0, uint64_t ti1, double2* out) {
    __shared__ double2 s[32][33];
    const uint32_t M = 1u << m, E = (uint32_t)min((uint64_t)M, N);
    const uint64_t na = tri(ti1) - tri(ti0), nb = (ti1 - ti0) * G;
    const uint64_t row0 = ti0 * M;
    for (uint64_t w = blockIdx.x; w < na + nb; w += gridDim.x) {
        uint64_t ti, tj;
        bool adj;
        if (w < na) {
            tri_loose(tri(ti0) + w, ti, tj);
            adj = false;
        } else {
            const uint64_t u = w - na;
            tj = ti0 + u / G;  // stored (ti, tj) with ti > tj, written into tile row tj
            ti = u % G;
            if (ti <= tj)
                continue;
            adj = true;
        }
        const double2* tp = src + ((tri(ti) + tj) << (2 * m));
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
            const uint32_t r = e / E, c = e % E;
            s[r][c] = tp[r * M + c];
        }
        __syncthreads();
        if (!adj) {
            for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
                const uint32_t r = e / E, c = e % E;
                out[(ti * M + r - row0) * N + tj * M + c] = s[r][c];
            }
        } else {  // logical (tj * M + c, ti * M + r) = conj(stored (ti * M + r, tj * M + c)), rows along r
            for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
                const uint32_t c = e / E, r = e % E;
                out[(tj * M + c - row0) * N + ti * M + r] = cconj(s[r][c]);
            }
        }
    }
}

// Tiled -> packed columns [tj0 * M, tj1 * M) (out points at column tj0 * M): every stored tile (ti, tj)
// with tj in [tj0, tj1); column tj * M + c receives rows i >= j, contiguous along i.
__global__ void __launch_bounds__(CV_T) to_packed_kernel(const double2* __restrict__ src, uint32_t m, uint64_t N,
                                                         uint64_t G, uint64_t tj0, uint64_t tj1, double2* out) {
    __shared__ double2 s[32][33];
    const uint32_t M = 1u << m, E = (uint32_t)min((uint64_t)M, N);
    const uint64_t base = packed_off(N, tj0 * M);
    for (uint64_t w = blockIdx.x; w < (tj1 - tj0) * G; w += gridDim.x) {
        const uint64_t tj = tj0 + w / G, ti = w % G;
        if (ti < tj)
            continue;
        const double2* tp = src + ((tri(ti) + tj) << (2 * m));
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
            const uint32_t r = e / E, c = e % E;
            s[r][c] = tp[r * M + c];
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
            const uint32_t c = e / E, r = e % E;
            const uint64_t i = ti * M + r, j = tj * M + c;
            if (i >= j)
                out[packed_off(N, j) - base + (i - j)] = s[r][c];
        }
    }
}

// Dense rows [ti0 * M, ti1 * M) (in points at row ti0 * M) -> the stored tiles of tile rows
// [ti0, ti1): off-diagonal tiles are the dense block; a diagonal tile's upper half is conj(d(j, i)).
__global__ void __launch_bounds__(CV_T) from_dense_kernel(double2* dst, uint32_t m, uint64_t N, uint64_t ti0,
                                                          uint64_t ti1, const double2* __restrict__ in) {
    __shared__ double2 s[32][33];
    const uint32_t M = 1u << m, E = (uint32_t)min((uint64_t)M, N);
    const uint64_t row0 = ti0 * M;
    for (uint64_t w = blockIdx.x; w < tri(ti1) - tri(ti0); w += gridDim.x) {
        const uint64_t t = tri(ti0) + w;
        uint64_t ti, tj;
        tri_loose(t, ti, tj);
        double2* tp = dst + (t << (2 * m));
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
            const uint32_t r = e / E, c = e % E;
            s[r][c] = in[(ti * M + r - row0) * N + tj * M + c];
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < M * M; e += CV_T) {
            const uint32_t r = e >> m, c = e & (M - 1);
            double2 v = make_double2(0.0, 0.0);
            if (r < E && c < E)
                v = (ti != tj || r >= c) ? s[r][c] : cconj(s[c][r]);
            tp[e] = v;
        }
    }
}

// Packed columns [tj0 * M, tj1 * M) (in points at column tj0 * M) -> the stored tiles (ti, tj),
// tj in [tj0, tj1): lower elements read along i (contiguous in the packed column), a diagonal tile's
// upper half = conj(lower mirror).  The matrix diagonal is conj(P(i, i)): the reference's
// to_dense(packed) sets d(i, j) = v, then d(j, i) = conj(v), which for i == j leaves conj(v)
// (storage.cpp:249-256; only visible for a payload whose diagonal is not real).
__global__ void __launch_bounds__(CV_T) from_packed_kernel(double2* dst, uint32_t m, uint64_t N, uint64_t G,
                                                           uint64_t tj0, uint64_t tj1, const double2* __restrict__ in) {
    __shared__ double2 s[32][33];
    const uint32_t M = 1u << m, E = (uint32_t)min((uint64_t)M, N);
    const uint64_t base = packed_off(N, tj0 * M);
    for (uint64_t w = blockIdx.x; w < (tj1 - tj0) * G; w += gridDim.x) {
        const uint64_t tj = tj0 + w / G, ti = w % G;
        if (ti < tj)
            continue;
        double2* tp = dst + ((tri(ti) + tj) << (2 * m));
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < E * E; e += CV_T) {
            const uint32_t c = e / E, r = e % E;
            const uint64_t i = ti * M + r, j = tj * M + c;
            if (i >= j)
                s[r][c] = in[packed_off(N, j) - base + (i - j)];
        }
        __syncthreads();
        for (uint32_t e = threadIdx.x; e < M * M; e += CV_T) {
            const uint32_t r = e >> m, c = e & (M - 1);
            double2 v = make_double2(0.0, 0.0);
            if (r < E && c < E)
                v = (ti != tj || r > c) ? s[r][c] : cconj(s[c][r]);
            tp[e] = v;
        }
    }
}

// Tiled (m1) -> tiled (m2), same n: fill_from_lower over to_dense(src) element by element; threads
// run along stored rows of the target, whose lower elements read source rows (coalesced); a target
// diagonal tile's upper half reads the mirror.
__global__ void __launch_bounds__(CV_T) retile_kernel(double2* dst, uint32_t m2, uint64_t cnt2, uint64_t N,
                                                      const double2* __restrict__ src, uint32_t m1) {
    const uint64_t M2 = 1ull << m2;
    for (uint64_t e = blockIdx.x * (uint64_t)CV_T + threadIdx.x; e < cnt2; e += (uint64_t)gridDim.x * CV_T) {
        uint64_t ti, tj;
        tri_loose(e >> (2 * m2), ti, tj);
        const uint64_t i = ti * M2 + ((e >> m2) & (M2 - 1)), j = tj * M2 + (e & (M2 - 1));
        double2 v = make_double2(0.0, 0.0);
        if (i < N && j < N)
            v = i >= j ? tiled_at(src, m1, i, j) : cconj(tiled_at(src, m1, j, i));
        dst[e] = v;
    }
}
}  // namespace
