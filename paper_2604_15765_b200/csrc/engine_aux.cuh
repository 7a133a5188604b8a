// engine_aux.cuh -- part of engine.cu (one translation unit; included in order).
// Deterministic reductions (tr(rho O), trace, Frobenius) and device-side input generators.
#pragma once

namespace {
// ------------------------------------------------------------------------- reductions
// Per-CTA partial sums over a contiguous tile range, fixed order, then a single-CTA
// ordered sum: deterministic for a given grid (SPEC.md observables: fixed-order reduction).
constexpr int RED_BLOCKS = 1184;  // 8 x 148 SMs

struct SD {  // shard descriptor of a state's local payload
    uint32_t Plog, logB, shard;
};

__device__ double block_sum(double v, double* sh) {
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int s = NTHR / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            sh[threadIdx.x] += sh[threadIdx.x + s];
        __syncthreads();
    }
    const double r = sh[0];
    __syncthreads();
    return r;
}

// kind 0: Re<a, b>_F (expectation); kind 1: |a|^2 (frobenius); kind 2: trace (diagonal elements)
__global__ void __launch_bounds__(NTHR) reduce_kernel(const double2* __restrict__ a, const double2* __restrict__ b,
                                                      uint64_t ntiles, uint32_t logM, int kind, double* partials, SD sd) {
    __shared__ double sh[NTHR];
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = blockIdx.x * per, t1 = min(ntiles, t0 + per);
    const uint32_t MM = 1u << (2 * logM), M = 1u << logM;
    double dsum = 0.0, osum = 0.0;
    if (t0 < t1) {
        for (uint64_t t = t0; t < t1; ++t) {
            uint64_t ti, tj;
            shard_decode(sd.Plog, sd.logB, sd.shard, t, ti, tj);
            const double2* pa = a + (t << (2 * logM));
            const double2* pb = b + (t << (2 * logM));
            double acc = 0.0;
            if (kind == 2) {
                if (ti == tj)
                    for (uint32_t p = threadIdx.x; p < M; p += NTHR)
                        acc += pa[p * M + p].x;
            } else {
                for (uint32_t p = threadIdx.x; p < MM; p += NTHR) {
                    const double2 x = pa[p], y = pb[p];
                    acc = fma(x.x, y.x, acc);
                    acc = fma(x.y, y.y, acc);
                }
            }
            if (ti == tj)
                dsum += acc;
            else
                osum += acc;
        }
    }
    dsum = block_sum(dsum, sh);
    osum = block_sum(osum, sh);
    if (threadIdx.x == 0) {
        partials[2 * blockIdx.x] = dsum;
        partials[2 * blockIdx.x + 1] = osum;
    }
}

__global__ void finish_kernel(const double* partials, int nparts, int kind, double* out) {
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        double d = 0.0, o = 0.0;
        for (int i = 0; i < nparts; ++i) {
            d += partials[2 * i];
            o += partials[2 * i + 1];
        }
        out[0] = kind == 2 ? d : d + 2.0 * o;
    }
}

// ------------------------------------------------------------------------- generators
// rho(i, j) = (1/rank) sum_a psi_a[i] conj(psi_a[j]) with explicit rounding (no contraction),
// bit-identical to hsg_rho_payload (harness.c).
__global__ void fill_mixture_kernel(double2* st, uint64_t count, uint32_t logM, uint64_t N, const double2* psi,
                                    int rank, double inv, SD sd) {
    const uint32_t M = 1u << logM;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = e >> (2 * logM);
        const uint32_t r = (uint32_t)((e >> logM) & (M - 1)), c = (uint32_t)(e & (M - 1));
        uint64_t ti, tj;
        shard_decode(sd.Plog, sd.logB, sd.shard, t, ti, tj);
        const uint64_t i = ti * M + r, j = tj * M + c;
        double2 acc = make_double2(0.0, 0.0);
        if (i < N && j < N) {
            for (int a = 0; a < rank; ++a) {
                const double2 p = psi[(uint64_t)a * N + i], q = psi[(uint64_t)a * N + j];
                const double re = __dadd_rn(__dmul_rn(p.x, q.x), __dmul_rn(p.y, q.y));
                const double im = __dsub_rn(__dmul_rn(p.y, q.x), __dmul_rn(p.x, q.y));
                acc.x = __dadd_rn(acc.x, re);
                acc.y = __dadd_rn(acc.y, im);
            }
            acc.x = __dmul_rn(acc.x, inv);
            acc.y = __dmul_rn(acc.y, inv);
        }
        st[e] = acc;
    }
}


// The reference's seeded operators (storage.cpp:22-55,195-239) generated where they live: the
// counter-based gaussian_entry (splitmix64 + Box-Muller) per element, H = (A + A^dagger) / 2.  The
// integer stream is exact; CUDA's log / sqrt / sincos may differ from glibc's in the last ulp, so
// elements agree with the reference to ~1e-16 relative (tests/test_gpu_parity.py).
__device__ __forceinline__ uint64_t splitmix64_d(uint64_t x) {
    x += 0x9E3779B97F4A7C15ull;
    x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
    x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
    return x ^ (x >> 31);
}
__device__ __forceinline__ double2 gaussian_entry_d(uint64_t base, uint64_t counter) {
    const uint64_t r1 = splitmix64_d(base + 2 * counter), r2 = splitmix64_d(base + 2 * counter + 1);
    const double u1 = (double)((r1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = (double)(r2 >> 11) * 0x1.0p-53;
    const double r = sqrt(-2.0 * log(u1));
    double sn, cs;
    sincos(2.0 * 3.141592653589793238462643383279502884 * u2, &sn, &cs);
    return make_double2(r * cs, r * sn);
}
// kind 0: random_hermitian(seed); kind 1: basis_projector(basis = seed)
__global__ void fill_seeded_kernel(double2* st, uint64_t count, uint32_t logM, uint64_t N, uint64_t seed, int kind,
                                   SD sd) {
    const uint32_t M = 1u << logM;
    const uint64_t base = splitmix64_d(seed ^ 0xD6E8FEB86659FD93ull);
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = e >> (2 * logM);
        const uint32_t r = (uint32_t)((e >> logM) & (M - 1)), c = (uint32_t)(e & (M - 1));
        uint64_t ti, tj;
        shard_decode(sd.Plog, sd.logB, sd.shard, t, ti, tj);
        const uint64_t i = ti * M + r, j = tj * M + c;
        double2 v = make_double2(0.0, 0.0);
        if (i < N && j < N) {
            if (kind == 0) {
                const double2 a = gaussian_entry_d(base, i * N + j), b = gaussian_entry_d(base, j * N + i);
                v = make_double2(0.5 * (a.x + b.x), 0.5 * (a.y - b.y));
            } else if (i == seed && j == seed) {
                v.x = 1.0;
            }
        }
        st[e] = v;
    }
}

// max_e |st[e] - rho_psi(e)| over the stored payload, rho_psi = (1/rank) sum |psi_i><psi_i| built
// exactly as fill_mixture_kernel (verification of full-size states without a second copy)
__global__ void dist_mixture_kernel(const double2* st, uint64_t count, uint32_t logM, uint64_t N, const double2* psi,
                                    int rank, double inv, double* out, SD sd) {
    __shared__ double sh[NTHR];
    const uint32_t M = 1u << logM;
    double mx = 0.0;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = e >> (2 * logM);
        const uint32_t r = (uint32_t)((e >> logM) & (M - 1)), c = (uint32_t)(e & (M - 1));
        uint64_t ti, tj;
        shard_decode(sd.Plog, sd.logB, sd.shard, t, ti, tj);
        const uint64_t i = ti * M + r, j = tj * M + c;
        double2 acc = make_double2(0.0, 0.0);
        if (i < N && j < N) {
            for (int a = 0; a < rank; ++a) {
                const double2 p = psi[(uint64_t)a * N + i], q = psi[(uint64_t)a * N + j];
                acc.x = __dadd_rn(acc.x, __dadd_rn(__dmul_rn(p.x, q.x), __dmul_rn(p.y, q.y)));
                acc.y = __dadd_rn(acc.y, __dsub_rn(__dmul_rn(p.y, q.x), __dmul_rn(p.x, q.y)));
            }
            acc.x = __dmul_rn(acc.x, inv);
            acc.y = __dmul_rn(acc.y, inv);
        }
        const double2 v = st[e];
        mx = fmax(mx, fmax(fabs(v.x - acc.x), fabs(v.y - acc.y)));
    }
    sh[threadIdx.x] = mx;
    __syncthreads();
    for (int s = NTHR / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s)
            sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + s]);
        __syncthreads();
    }
    if (threadIdx.x == 0)
        out[blockIdx.x] = sh[0];
}

struct PauliArgs {
    const uint64_t* x;
    const uint64_t* z;
    const int32_t* ny;
    const double* coef;
    int count;
};

__global__ void fill_pauli_kernel(double2* st, uint64_t count, uint32_t logM, uint64_t N, PauliArgs pa, SD sd) {
    const uint32_t M = 1u << logM;
    for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < count;
         e += (uint64_t)gridDim.x * blockDim.x) {
        const uint64_t t = e >> (2 * logM);
        const uint32_t r = (uint32_t)((e >> logM) & (M - 1)), c = (uint32_t)(e & (M - 1));
        uint64_t ti, tj;
        shard_decode(sd.Plog, sd.logB, sd.shard, t, ti, tj);
        const uint64_t i = ti * M + r, j = tj * M + c;
        double2 acc = make_double2(0.0, 0.0);
        if (i < N && j < N) {
            const uint64_t ij = i ^ j;
            for (int s = 0; s < pa.count; ++s) {
                if (pa.x[s] != ij)
                    continue;
                double v = pa.coef[s];
                if (__popcll(j & pa.z[s]) & 1)
                    v = -v;
                const int ph = pa.ny[s] & 3;  // i^ny
                if (ph == 0)
                    acc.x = __dadd_rn(acc.x, v);
                else if (ph == 1)
                    acc.y = __dadd_rn(acc.y, v);
                else if (ph == 2)
                    acc.x = __dadd_rn(acc.x, -v);
                else
                    acc.y = __dadd_rn(acc.y, -v);
            }
        }
        st[e] = acc;
    }
}

// ---------------------------------------------------------------- CX layer (fusion)
// A product of CX gates on disjoint (control, target) pairs is an involutive, GF(2)-linear basis
// permutation pi (x -> x ^ sum_k x_ck e_tk), and rho'(i, j) = rho(pi(i), pi(j)).  In place, one pass:
// every canonical slot (off-diagonal tiles, the lower half of diagonal tiles) pairs with the
// canonical slot of (pi(i), pi(j)) -- conjugated when that logical element lies above the diagonal
// -- and the lower slot of each pair swaps both (pi is an involution, so the pairing is symmetric).
// The upper half of a diagonal tile is written with its canonical mirror.  pi splits over the
// tile and in-tile bits (linearity), so an element costs two XORs with a per-tile and an in-tile
// (shared-memory) image.
struct CxLayer {
    uint32_t n;
    uint32_t c[32], t[32];
    // Tile-column bits that are CX targets of low in-tile controls (at most two bits): along a tile
    // row the partners of such a control's two values alternate in runs of 16 / 32 / 64 B between
    // tile columns tq and tq ^ bit, and the sibling tile (ti, tj ^ bit) holds the complementary runs.
    uint32_t gmask;
};
__device__ __forceinline__ uint64_t cx_pi(const CxLayer& L, uint64_t x) {
    uint64_t y = x;
    for (uint32_t k = 0; k < L.n; ++k)
        y ^= ((x >> L.c[k]) & 1ull) << L.t[k];
    return y;
}
__global__ void __launch_bounds__(256, 3) cx_layer_kernel(double2* __restrict__ st, uint64_t ntiles, uint32_t logM,
                                                       uint32_t nq, const CxLayer L) {
    constexpr uint32_t CXB = 4;   // positions a thread has in flight
    constexpr uint32_t NMEM = 4;  // tiles of a sibling group, at most
    __shared__ uint64_t tab[32];  // pi of the in-tile offsets
    // per tile: pi of its rows x (tile row rT, in-tile row rX, tri(rT)) and, per group member, of its columns y
    __shared__ uint64_t rT[32], rTri[32], cT[NMEM * 32], cTri[NMEM * 32];
    __shared__ uint32_t rX[32], cY[NMEM * 32];
    const uint32_t M = 1u << logM, lMM = 2 * logM, nel = 1u << lMM;
    if (threadIdx.x < M)
        tab[threadIdx.x] = cx_pi(L, threadIdx.x);
    auto put = [&](uint64_t slot, bool diag, uint32_t x, uint32_t y, double2 v) {
        st[slot] = v;
        if (diag && x > y)  // mirror in the upper half of a diagonal tile
            st[slot - ((uint64_t)x << logM) - y + ((uint64_t)y << logM) + x] = make_double2(v.x, -v.y);
    };
    const uint32_t gmask = L.gmask, glo = gmask & (0u - gmask), ghi = gmask ^ glo;
    const uint32_t lgn = gmask ? (ghi ? 2u : 1u) : 0u;  // log2 of a group's tile count
    // Each thread takes CXB positions at once -- one column of CXB / nm adjacent rows in each of the
    // nm tiles of a sibling group: every owner's two loads are issued before any store (memory-level
    // parallelism; pairs are disjoint, so no other thread reads or writes them; the upper halves of
    // diagonal tiles written as mirrors are never read).  Adjacent rows: where the partner tile is
    // stored transposed they are adjacent elements of one partner row.  Sibling tiles: together their
    // partners cover whole partner rows, requested back to back (DRAM moves 64-B granules, and L2 does
    // not keep the half nobody asked for).
    for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        uint64_t ti, tj;
        tri_loose(tile, ti, tj);
        // a group lies in one tile row; it is taken whole by its first tile when every member is stored
        const bool grouped = gmask && ((tj | gmask) <= ti);
        if (grouped && (tj & gmask))
            continue;
        const uint32_t lg = grouped ? lgn : 0u, nm = 1u << lg;
        __syncthreads();  // tab ready / the previous tile's tables are no longer read
        if (threadIdx.x < (1 + nm) * M) {
            const bool col = threadIdx.x >= M;
            const uint32_t v = threadIdx.x & (M - 1), mem = col ? (threadIdx.x >> logM) - 1 : 0;
            const uint64_t tjm = tj | ((mem & 1u) ? glo : 0u) | ((mem & 2u) ? ghi : 0u);
            const uint64_t pq = cx_pi(L, (col ? tjm : ti) << logM) ^ tab[v], t = pq >> logM;
            if (col) {
                cT[mem * 32 + v] = t;
                cTri[mem * 32 + v] = t * (t + 1) / 2;
                cY[mem * 32 + v] = (uint32_t)(pq & (M - 1));
            } else {
                rT[v] = t;
                rTri[v] = t * (t + 1) / 2;
                rX[v] = (uint32_t)(pq & (M - 1));
            }
        }
        __syncthreads();
        // Ownership of a pair {e, s2}: the slot whose canonical (row, column) comes first owns it.  Rows
        // decide except on the 2^-npairs of rows pi fixes, so a warp (one tile row) owns all of its
        // elements or none: owned rows are read and written as whole 512-B runs, the other warps leave
        // before any per-element arithmetic.
        const uint32_t ti32 = (uint32_t)ti, tj32 = (uint32_t)tj, I0 = ti32 << logM;
        const uint32_t rpi = CXB >> lg;  // rows per thread and iteration
        const uint32_t nbase = ((M + rpi - 1) / rpi) << logM;
        for (uint32_t pos0 = threadIdx.x; pos0 < nbase; pos0 += blockDim.x) {
            uint64_t s2o[CXB];
            // bit 0: active pair, 1: self-pair, 2: conjugate, 3: partner in a diagonal tile; bits 8-15 / 16-23: the
            // partner's in-tile column / row
            uint32_t meta[CXB];
            double2 av[CXB], bv[CXB];
            auto where = [&](uint32_t k, uint32_t& x, uint32_t& y, uint32_t& mem, uint32_t& tjm) {
                mem = k & (nm - 1);
                x = (pos0 >> logM) * rpi + (k >> lg);
                y = pos0 & (M - 1);
                tjm = tj32 | ((mem & 1u) ? glo : 0u) | ((mem & 2u) ? ghi : 0u);
            };
#pragma unroll
            for (uint32_t k = 0; k < CXB; ++k) {
                uint32_t x, y, mem, tjm;
                where(k, x, y, mem, tjm);
                meta[k] = 0;
                if (x >= M)
                    continue;
                const uint32_t I = I0 | x, J = (tjm << logM) | y;
                if ((ti32 == tjm && x < y) || (I >> nq) || (J >> nq))
                    continue;  // mirror half, or zero padding (n < m): left as it is
                const uint32_t cy = mem * 32 + y;
                const uint64_t tp = rT[x], tq = cT[cy];
                const uint32_t px = rX[x], qy = cY[cy];
                const uint32_t pI = ((uint32_t)tp << logM) | px, pJ = ((uint32_t)tq << logM) | qy;
                const bool cj = pI < pJ;
                const uint32_t I2 = cj ? pJ : pI, J2 = cj ? pI : pJ;  // canonical (row, column) of the partner
                if (I2 != I ? I2 < I : (J2 < J || (J2 == J && !cj)))
                    continue;  // the partner's thread owns the pair; or a fixed point
                // canonical slot of (pi(i), pi(j)): (tp, tq, px, qy), or its transpose when above the diagonal
                const uint64_t s2 = ((cj ? cTri[cy] + tp : rTri[x] + tq) << lMM) +
                                    (cj ? ((uint64_t)qy << logM) + px : ((uint64_t)px << logM) + qy);
                const uint64_t e = ((tile + (tjm - tj32)) << lMM) + (x << logM) + y;
                s2o[k] = s2;
                meta[k] = 1u | (s2 == e ? 2u : 0u) | (cj ? 4u : 0u) | (tp == tq ? 8u : 0u) |
                          ((cj ? (qy << 8) | px : (px << 8) | qy) << 8);
                av[k] = st[e];
                if (s2 != e)
                    bv[k] = st[s2];
            }
#pragma unroll
            for (uint32_t k = 0; k < CXB; ++k) {
                if (!(meta[k] & 1u))
                    continue;
                uint32_t x, y, mem, tjm;
                where(k, x, y, mem, tjm);
                const bool diag = ti32 == tjm;
                const uint64_t e = ((tile + (tjm - tj32)) << lMM) + (x << logM) + y;
                double2 a = av[k];
                if (meta[k] & 2u) {  // rho'(i, j) = rho(j, i)
                    put(e, diag, x, y, make_double2(a.x, -a.y));
                    continue;
                }
                double2 b = bv[k];
                if (meta[k] & 4u) {
                    a.y = -a.y;
                    b.y = -b.y;
                }
                put(e, diag, x, y, b);
                put(s2o[k], (meta[k] & 8u) != 0, meta[k] >> 16, (meta[k] >> 8) & 0xffu, a);
            }
        }
    }
}
}  // namespace
