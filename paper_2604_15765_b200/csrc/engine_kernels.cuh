// engine_kernels.cuh -- part of engine.cu (one translation unit; included in order).
// Block transforms and the streaming kernels: the slab kernel (paths U and D, the wedge
// rule for diagonal units) and the persistent TMA-bulk pipeline (pipe_kernel).
#pragma once

namespace {
// ------------------------------------------------------------------- block transforms
// The transforms see a block through (base, off[]) : element (rho, gamma) lives at
// sm[base + off[rho * D + gamma]].  They are shared by paths U and D.

// S-form, k = 1 (TransferQuad, kernels.cpp:66-77): v row-stacked (h00, h01, h10, h11)
template <int MODE>
__device__ __forceinline__ void xf_quad(double2* sm, uint32_t base, const uint16_t* off, const Coef<16>& cf) {
    double2 v0 = sm[base + off[0]], v1 = sm[base + off[1]], v2 = sm[base + off[2]], v3 = sm[base + off[3]];
    double2 w0, w1, w2, w3;
    if (MODE == M_HAD) {  // HadamardQuad (native.cpp:332-339)
        const double2 a = make_double2(v0.x + v1.x, v0.y + v1.y), b = make_double2(v0.x - v1.x, v0.y - v1.y);
        const double2 c = make_double2(v2.x + v3.x, v2.y + v3.y), d = make_double2(v2.x - v3.x, v2.y - v3.y);
        w0 = make_double2(0.5 * (a.x + c.x), 0.5 * (a.y + c.y));
        w1 = make_double2(0.5 * (b.x + d.x), 0.5 * (b.y + d.y));
        w2 = make_double2(0.5 * (a.x - c.x), 0.5 * (a.y - c.y));
        w3 = make_double2(0.5 * (b.x - d.x), 0.5 * (b.y - d.y));
    } else if (cf.xpat) {
        const double2* s = cf.s;
        w0 = cfma(s[3], v3, cmul(s[0], v0));
        w3 = cfma(s[15], v3, cmul(s[12], v0));
        w1 = cfma(s[6], v2, cmul(s[5], v1));
        w2 = cfma(s[10], v2, cmul(s[9], v1));
    } else {
        const double2* s = cf.s;
        w0 = cmul(s[0], v0); w0 = cfma(s[1], v1, w0); w0 = cfma(s[2], v2, w0); w0 = cfma(s[3], v3, w0);
        w1 = cmul(s[4], v0); w1 = cfma(s[5], v1, w1); w1 = cfma(s[6], v2, w1); w1 = cfma(s[7], v3, w1);
        w2 = cmul(s[8], v0); w2 = cfma(s[9], v1, w2); w2 = cfma(s[10], v2, w2); w2 = cfma(s[11], v3, w2);
        w3 = cmul(s[12], v0); w3 = cfma(s[13], v1, w3); w3 = cfma(s[14], v2, w3); w3 = cfma(s[15], v3, w3);
    }
    sm[base + off[0]] = w0;
    sm[base + off[1]] = w1;
    sm[base + off[2]] = w2;
    sm[base + off[3]] = w3;
}

// S-form, k = 2 (matvec<16>, kernels.cpp:39-48)
__device__ __forceinline__ void xf_s16(double2* sm, uint32_t base, const uint16_t* off, const Coef<256>& cf) {
    double2 v[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        v[i] = sm[base + off[i]];
#pragma unroll 4
    for (int r = 0; r < 16; ++r) {
        double2 acc = cmul(cf.s[r * 16], v[0]);
#pragma unroll
        for (int c = 1; c < 16; ++c)
            acc = cfma(cf.s[r * 16 + c], v[c], acc);
        sm[base + off[r]] = acc;
    }
}

// Direct form, stage 1: row rho of B <- B[rho, :] L^dagger  (Y = B L^dagger)
template <int K, int NS>
__device__ __forceinline__ void xf_row(double2* sm, uint32_t base, const uint16_t* off, uint32_t rho,
                                       const double2* L) {
    constexpr int D = 1 << K;
    double2 v[D];
#pragma unroll
    for (int c = 0; c < D; ++c)
        v[c] = sm[base + off[rho * D + c]];
#pragma unroll
    for (int c = 0; c < D; ++c) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < D; ++t)
            acc = cfmaconj(v[t], L[c * D + t], acc);  // sum_t B[rho][t] conj(L[c][t])
        sm[base + off[rho * D + c]] = acc;
    }
}
// Direct form, stage 2: column gamma <- L Y[:, gamma]
template <int K>
__device__ __forceinline__ void xf_col(double2* sm, uint32_t base, const uint16_t* off, uint32_t gamma,
                                       const double2* L) {
    constexpr int D = 1 << K;
    double2 v[D];
#pragma unroll
    for (int r = 0; r < D; ++r)
        v[r] = sm[base + off[r * D + gamma]];
#pragma unroll
    for (int r = 0; r < D; ++r) {
        double2 acc = make_double2(0.0, 0.0);
#pragma unroll
        for (int t = 0; t < D; ++t)
            acc = cfma(L[r * D + t], v[t], acc);
        sm[base + off[r * D + gamma]] = acc;
    }
}

// Kraus sum (k = 3 generic, r > 1): out = sum_a L_a B L_a^dagger, per block, with the block
// held in shared memory: X (input) -> T (= X L_a^dagger) -> O (+= L_a T).  Runs the row/column
// stages over three buffers.
// (handled inline in the kernels; see run_compute)

// --------------------------------------------------------------------------- kernel body
struct KrausArgs {
    const double2* ops;  // nops x D x D (device)
    int nops;
};

// Block base for path U: ((uu << logNT) * SR + xb_tab[xbi]) * Mp + yb_tab[ybi]
struct UAddr {
    const Geo* G;
    const uint8_t* xb;
    const uint8_t* yb;
    __device__ __forceinline__ uint32_t base(uint32_t b) const {
        const uint32_t ybi = b & (G->nyb - 1);
        const uint32_t xbi = (b >> G->logNyb) & (G->nxb - 1);
        const uint32_t uu = b >> (G->logNyb + G->logNxb);
        return (((uu << G->logNT) * G->SR) + xb[xbi]) * G->Mp + yb[ybi];
    }
    __device__ __forceinline__ uint32_t unit(uint32_t b) const { return b >> (G->logNyb + G->logNxb); }
};
struct DAddr {
    uint32_t shift;  // 2K
    __device__ __forceinline__ uint32_t base(uint32_t b) const { return b << shift; }
};

// Runs the compute stage(s) of MODE over `nblk` blocks addressed by A; valid(b) filters.
template <int K, int MODE, int NS, class A, class V>
__device__ __forceinline__ void compute_blocks(double2* sm, double2* sm2, double2* sm3, const uint16_t* off,
                                               uint32_t nblk, const A& addr, const V& valid, const Coef<NS>& cf,
                                               const KrausArgs& ka, uint32_t stage_order_nyb_log, double2* lsm) {
    constexpr int D = 1 << K;
    const int tid = threadIdx.x;
    if constexpr (MODE == M_S1 || MODE == M_HAD) {
        for (uint32_t b = tid; b < nblk; b += NTHR)
            if (valid(b))
                xf_quad<MODE>(sm, addr.base(b), off, *reinterpret_cast<const Coef<16>*>(&cf));
    } else if constexpr (MODE == M_S2) {
        for (uint32_t b = tid; b < nblk; b += NTHR)
            if (valid(b))
                xf_s16(sm, addr.base(b), off, *reinterpret_cast<const Coef<256>*>(&cf));
    } else if constexpr (MODE == M_DIRECT) {
        // items (b, rho): keep the fastest-varying block index innermost so lanes hit
        // consecutive columns; stage_order_nyb_log = log2 of that fastest extent.
        const uint32_t lo = stage_order_nyb_log, lomask = (1u << lo) - 1;
        const uint32_t items = nblk * D;
        for (uint32_t w = tid; w < items; w += NTHR) {
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
            const uint32_t rho = (w >> lo) % D;
            if (valid(b))
                xf_row<K, NS>(sm, addr.base(b), off, rho, cf.s);
        }
        __syncthreads();
        for (uint32_t w = tid; w < items; w += NTHR) {
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
            const uint32_t gamma = (w >> lo) % D;
            if (valid(b))
                xf_col<K>(sm, addr.base(b), off, gamma, cf.s);
        }
    } else if constexpr (MODE == M_KRAUS) {
        // sm = X (input), sm2 = T, sm3 = O; all share the same addressing.
        const uint32_t lo = stage_order_nyb_log, lomask = (1u << lo) - 1;
        const uint32_t items = nblk * D;
        for (uint32_t w = tid; w < items; w += NTHR) {
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
            const uint32_t r = (w >> lo) % D;
            if (valid(b)) {
                const uint32_t base = addr.base(b);
#pragma unroll
                for (int c = 0; c < D; ++c)
                    sm3[base + off[r * D + c]] = make_double2(0.0, 0.0);
            }
        }
        double2* Lr = lsm;  // L_a staged in shared memory (after the three block buffers)
        for (int a = 0; a < ka.nops; ++a) {
            __syncthreads();
            for (int i = tid; i < D * D; i += NTHR)
                Lr[i] = ka.ops[(size_t)a * D * D + i];
            __syncthreads();
            for (uint32_t w = tid; w < items; w += NTHR) {  // T = X L^dagger (rows)
                const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
                const uint32_t rho = (w >> lo) % D;
                if (!valid(b))
                    continue;
                const uint32_t base = addr.base(b);
                double2 v[D];
#pragma unroll
                for (int c = 0; c < D; ++c)
                    v[c] = sm[base + off[rho * D + c]];
#pragma unroll
                for (int c = 0; c < D; ++c) {
                    double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                    for (int t = 0; t < D; ++t)
                        acc = cfmaconj(v[t], Lr[c * D + t], acc);
                    sm2[base + off[rho * D + c]] = acc;
                }
            }
            __syncthreads();
            for (uint32_t w = tid; w < items; w += NTHR) {  // O += L T (columns)
                const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
                const uint32_t gamma = (w >> lo) % D;
                if (!valid(b))
                    continue;
                const uint32_t base = addr.base(b);
                double2 v[D];
#pragma unroll
                for (int r = 0; r < D; ++r)
                    v[r] = sm2[base + off[r * D + gamma]];
#pragma unroll
                for (int r = 0; r < D; ++r) {
                    double2 acc = sm3[base + off[r * D + gamma]];
#pragma unroll
                    for (int t = 0; t < D; ++t)
                        acc = cfma(Lr[r * D + t], v[t], acc);
                    sm3[base + off[r * D + gamma]] = acc;
                }
            }
        }
        __syncthreads();
        for (uint32_t w = tid; w < items; w += NTHR) {  // copy O back into X
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo);
            const uint32_t r = (w >> lo) % D;
            if (valid(b)) {
                const uint32_t base = addr.base(b);
#pragma unroll
                for (int c = 0; c < D; ++c)
                    sm[base + off[r * D + c]] = sm3[base + off[r * D + c]];
            }
        }
    }
}

// ---------------------------------------------------------------------------- path U
template <int K, int MODE, int NS>
__device__ void path_u(const Geo& G, const Tabs& T, const Coef<NS>& cf, const KrausArgs& ka,
                       double2* __restrict__ st, uint64_t item, double2* sm, uint64_t* ttab, uint16_t* off) {
    const int tid = threadIdx.x;
    constexpr int D = 1 << K;
    const uint64_t ug = item >> G.logSlabs;
    const uint32_t slab = (uint32_t)(item & (G.slabs - 1));
    const uint32_t x0 = G.sdep[slab];
    const uint64_t u0 = ug << G.logU;
    const uint32_t ntt = G.U << G.logNT;
    const uint32_t NGm = (1u << G.logNG) - 1;

    for (uint32_t i = tid; i < ntt; i += NTHR) {
        const uint32_t uu = i >> G.logNT, lt = i & ((1u << G.logNT) - 1);
        const uint64_t u = u0 + uu;
        uint64_t ent;
        if (u >= G.nU_units) {
            ent = F_BAD;
        } else if (!G.offdiag) {
            ent = u;
        } else {
            uint64_t tbi, tbj;
            unit_decode(G, u, true, tbi, tbj);
            const uint32_t R = lt >> G.logNG, C = lt & NGm;
            const uint64_t tr = ins_bits(tbi, R, G.gr_pos, G.g), tc = ins_bits(tbj, C, G.gr_pos, G.g);
            ent = tile_entry(G, tr, tc);
        }
        if (MODE == M_MONO && !((G.active >> lt) & 1ull))
            ent |= F_SKIP;
        ttab[i] = ent;
    }
    for (uint32_t i = tid; i < (uint32_t)(D * D); i += NTHR)
        off[i] = G.comp_off[i];
    __syncthreads();

    const uint32_t logTE = G.logSR + G.logM, TEm = (1u << logTE) - 1;
    const uint32_t Mm = G.M - 1, SRm = G.SR - 1;
    const uint32_t Mp = G.Mp;

    // ---- load: HBM -> shared (logical layout, adjoint tiles transposed + conjugated)
    for (uint32_t e0 = 0; e0 < G.E; e0 += NTHR * 8) {
        double2 v[8];
        uint32_t dst[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t e = e0 + j * NTHR + tid;
            dst[j] = 0xffffffffu;
            if (e < G.E) {
                const uint32_t tt = e >> logTE, l = e & TEm;
                const uint64_t ent = ttab[tt];
                if (!(ent & (F_BAD | F_SKIP))) {
                    const uint64_t tb = (ent & F_MASK) << (2 * G.logM);
                    uint32_t xs, y;
                    uint64_t src;
                    if (!(ent & F_ADJ)) {
                        xs = l >> G.logM;
                        y = l & Mm;
                        src = tb + ((uint64_t)(x0 | T.xdep[xs]) << G.logM) + y;
                    } else {
                        y = l >> G.logSR;
                        xs = l & SRm;
                        src = tb + ((uint64_t)y << G.logM) + (x0 | T.xdep[xs]);
                    }
                    v[j] = ldg2(tile_base(G, ent, st) + src);
                    if (ent & F_ADJ)
                        v[j].y = -v[j].y;
                    dst[j] = (tt * G.SR + xs) * Mp + y;
                }
            }
        }
#pragma unroll
        for (int j = 0; j < 8; ++j)
            if (dst[j] != 0xffffffffu)
                sm[dst[j]] = v[j];
    }
    __syncthreads();

    // ---- transform
    if constexpr (MODE != M_MONO) {
        UAddr A{&G, T.xb, T.yb};
        const uint32_t nblk = G.U << (G.logNxb + G.logNyb);
        const uint64_t nU = G.nU_units;
        auto valid = [&](uint32_t b) { return u0 + A.unit(b) < nU; };
        double2* sm2 = sm + G.Epad;
        double2* sm3 = sm + 2 * G.Epad;
        compute_blocks<K, MODE, NS>(sm, sm2, sm3, off, nblk, A, valid, cf, ka, G.logNyb, sm + 3 * G.Epad);
        __syncthreads();
    }

    // ---- store: shared -> HBM
    for (uint32_t e0 = 0; e0 < G.E; e0 += NTHR * 8) {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t e = e0 + j * NTHR + tid;
            if (e >= G.E)
                continue;
            const uint32_t tt = e >> logTE, l = e & TEm;
            const uint64_t ent = ttab[tt];
            if (ent & (F_BAD | F_SKIP | F_NOSTORE))
                continue;
            const uint64_t tb = (ent & F_MASK) << (2 * G.logM);
            const bool adj = (ent & F_ADJ) != 0;
            uint32_t xs, y;
            uint64_t dstg;
            if (!adj) {
                xs = l >> G.logM;
                y = l & Mm;
                dstg = tb + ((uint64_t)(x0 | T.xdep[xs]) << G.logM) + y;
            } else {
                y = l >> G.logSR;
                xs = l & SRm;
                dstg = tb + ((uint64_t)y << G.logM) + (x0 | T.xdep[xs]);
            }
            double2 w;
            if constexpr (MODE == M_MONO) {
                const uint32_t uu = tt >> G.logNT, lt = tt & ((1u << G.logNT) - 1);
                const uint32_t R = lt >> G.logNG, C = lt & NGm;
                const uint32_t rho = (R << G.kin) | T.xs_rin[xs], gam = (C << G.kin) | T.y_cin[y];
                const uint32_t rs = cf.pinv[rho], gs = cf.pinv[gam];
                const uint32_t kinm = (1u << G.kin) - 1;
                const uint32_t src = (((uu << G.logNT) + ((rs >> G.kin) << G.logNG) + (gs >> G.kin)) * G.SR +
                                      (T.xs_base[xs] | T.xs_in[rs & kinm])) * Mp +
                                     (T.y_base[y] | T.y_in[gs & kinm]);
                w = sm[src];
                const uint32_t fi = rho * D + gam;
                if (!((cf.fone >> fi) & 1ull))
                    w = cmul(cf.s[fi], w);
            } else {
                w = sm[(tt * G.SR + xs) * Mp + y];
            }
            if (adj)
                w.y = -w.y;
            G.out[dstg] = w;
        }
    }
}

// ---------------------------------------------------------------------------- path D
template <int K, int MODE, int NS>
__device__ void path_d(const Geo& G, const Tabs& T, const Coef<NS>& cf, const KrausArgs& ka,
                       double2* __restrict__ st, uint64_t item, double2* sm, uint64_t* tabs, uint32_t* bpos,
                       uint16_t* off) {
    constexpr int D = 1 << K, DD = D * D;
    const int tid = threadIdx.x;
    const uint64_t tb = item / G.itemsD;
    const uint64_t b0 = (item % G.itemsD) * G.BPI;
    uint64_t* trow = tabs;  // NG entries: tr[R]
    const uint32_t NG = 1u << G.logNG;
    for (uint32_t i = tid; i < NG; i += NTHR)
        trow[i] = ins_bits(tb, i, G.gr_pos, G.g);
    for (uint32_t i = tid; i < G.BPI; i += NTHR) {
        const uint64_t b = b0 + i;
        uint32_t v = 0xffffffffu;
        if (b < G.nblkD) {
            uint64_t xi, yi;
            tri_loose(b, xi, yi);
            v = ((uint32_t)xi << 16) | (uint32_t)yi;
        }
        bpos[i] = v;
    }
    for (uint32_t i = tid; i < (uint32_t)DD; i += NTHR)
        off[i] = (uint16_t)i;
    __syncthreads();
    const uint32_t kinm = (1u << G.kin) - 1;
    const uint32_t E = G.BPI * DD;
    const uint32_t logM = G.logM;

    // ---- gather (monomial permutation applied here)
    for (uint32_t e = tid; e < E; e += NTHR) {
        const uint32_t lb = e / DD, comp = e % DD;
        const uint32_t bp = bpos[lb];
        if (bp == 0xffffffffu)
            continue;
        uint32_t rho = comp / D, gam = comp % D;
        double2 f = make_double2(1.0, 0.0);
        bool one = true;
        if constexpr (MODE == M_MONO) {
            one = (cf.fone >> comp) & 1ull;
            f = cf.s[comp];
            rho = cf.pinv[rho];
            gam = cf.pinv[gam];
        }
        const uint32_t xb = T.yb[bp >> 16], yb = T.yb[bp & 0xffffu];
        const uint32_t R = rho >> G.kin, C = gam >> G.kin;
        const uint32_t x = xb | T.y_in[rho & kinm], y = yb | T.y_in[gam & kinm];
        double2 v;
        if (R >= C) {
            const uint64_t ent = tile_entry(G, trow[R], trow[C]);
            v = (ent & F_SKIP) ? make_double2(0.0, 0.0)
                               : tile_base(G, ent, st)[((ent & F_MASK) << (2 * logM)) + ((uint64_t)x << logM) + y];
        } else {
            const uint64_t ent = tile_entry(G, trow[C], trow[R]);
            v = (ent & F_SKIP) ? make_double2(0.0, 0.0)
                               : tile_base(G, ent, st)[((ent & F_MASK) << (2 * logM)) + ((uint64_t)y << logM) + x];
            v.y = -v.y;
        }
        if (!one)
            v = cmul(f, v);
        sm[e] = v;
    }
    __syncthreads();
    if constexpr (MODE != M_MONO) {
        DAddr A{2u * K};
        auto valid = [&](uint32_t b) { return bpos[b] != 0xffffffffu; };
        compute_blocks<K, MODE, NS>(sm, sm + E, sm + 2 * E, off, G.BPI, A, valid, cf, ka, 0, sm + 3 * E);
        __syncthreads();
    }
    // ---- scatter with the wedge rules (see file header)
    for (uint32_t e = tid; e < E; e += NTHR) {
        const uint32_t lb = e / DD, comp = e % DD;
        const uint32_t bp = bpos[lb];
        if (bp == 0xffffffffu)
            continue;
        const uint32_t xbi = bp >> 16, ybi = bp & 0xffffu;
        const uint32_t rho = comp / D, gam = comp % D;
        if (xbi == ybi && rho < gam)
            continue;
        const uint32_t xb = T.yb[xbi], yb = T.yb[ybi];
        const uint32_t R = rho >> G.kin, C = gam >> G.kin;
        const uint32_t x = xb | T.y_in[rho & kinm], y = yb | T.y_in[gam & kinm];
        const double2 w = sm[e];
        const uint64_t ent = R >= C ? tile_entry(G, trow[R], trow[C]) : tile_entry(G, trow[C], trow[R]);
        if (ent & F_REMOTE)
            continue;  // the partner shard stores this tile
        const uint64_t t0 = (ent & F_MASK) << (2 * logM);
        if (R > C) {
            G.out[t0 + ((uint64_t)x << logM) + y] = w;
        } else if (R < C) {
            G.out[t0 + ((uint64_t)y << logM) + x] = cconj(w);
        } else {
            G.out[t0 + ((uint64_t)x << logM) + y] = w;
            if (x != y)
                G.out[t0 + ((uint64_t)y << logM) + x] = cconj(w);
        }
    }
}

template <int K, int MODE, int NS>
__global__ void __launch_bounds__(NTHR) conj_kernel(const Geo G, const Coef<NS> cf, const KrausArgs ka,
                                                    double2* __restrict__ st) {
    extern __shared__ __align__(16) double2 smem[];
    __shared__ uint64_t tabs[MAX_TT];
    __shared__ uint32_t bpos[CAPD / 4];
    __shared__ uint16_t off[64];
    __shared__ Tabs T;
    // index tables are read with per-thread indices: stage them in shared memory (indexed
    // kernel-parameter reads would serialise in the constant cache)
    {
        const int t = threadIdx.x;
        if (t < 32) {
            T.xdep[t] = G.xdep[t];
            T.xb[t] = G.xb_tab[t];
            T.yb[t] = G.yb_tab[t];
            T.xs_rin[t] = G.xs_rin[t];
            T.xs_base[t] = G.xs_base[t];
            T.y_cin[t] = G.y_cin[t];
            T.y_base[t] = G.y_base[t];
            if (t < 8) {
                T.xs_in[t] = G.xs_in[t];
                T.y_in[t] = G.y_in[t];
            }
        }
    }
    const uint64_t item = blockIdx.x + (uint64_t)blockIdx.y * gridDim.x;
    if (item < G.nD_items)
        path_d<K, MODE, NS>(G, T, cf, ka, st, item, smem, tabs, bpos, off);
    else if (item < G.nD_items + G.nU_items)
        path_u<K, MODE, NS>(G, T, cf, ka, st, item - G.nD_items, smem, tabs, off);
}

// ------------------------------------------------------------- pipelined path U (TMA bulk copies)
// Persistent CTAs (one per SM) stream U-path items through a ring of `stages` shared-memory
// buffers: warp 0 issues cp.async.bulk loads (global -> shared, completion on an mbarrier with
// expect_tx) for items i+1 .. i+stages-1 while all warps transform item i in place; warp 0 then
// issues cp.async.bulk stores (shared -> global, bulk groups) and refills the buffer freed by
// item i-1 once its store has finished reading shared memory.  Direct logical tiles keep their
// stored row-major layout (pitch M); adjoint tiles keep their STORED orientation with pitch
// SR + 1, so the transposed reads of the transform are bank-conflict free; conjugation is
// applied on read and write.  No per-element index arithmetic is spent on the HBM side.
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
// 2-D tensor-map copies (x = inner coordinate in elements of the map, y = row)
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* tm, uint32_t x, uint32_t y, uint64_t* bar) {
    asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                 ::"r"(dst), "l"(tm), "r"(x), "r"(y), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, uint32_t x, uint32_t y, uint32_t src) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(tm), "r"(x), "r"(y),
                 "r"(src) : "memory");
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {  // expect_tx without an arrival
    asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
#ifdef HS_MBAR_HINT  // A/B builds: suspend-time hint (ns) for waiting warps
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity), "r"((uint32_t)HS_MBAR_HINT)
        : "memory");
    return;
#endif
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

constexpr int MAX_STAGES = 4;

// Fills the item's logical-tile table: stored tile index | F_ADJ / F_SKIP / F_BAD.
template <int MODE>
__device__ __forceinline__ void item_tiles(const Geo& G, uint64_t item, uint64_t* gt, uint32_t lane) {
    const uint32_t grp = G.groups ? (uint32_t)(item % G.groups) : 0;
    const uint64_t u0 = G.groups ? item / G.groups : (item >> G.logSlabs) << G.logU;
    const uint32_t ntt = G.U << G.logNT, NGm = (1u << G.logNG) - 1;
    for (uint32_t i = lane; i < ntt; i += 32) {
        const uint32_t uu = i >> G.logNT, lt = i & ((1u << G.logNT) - 1);
        const uint64_t u = u0 + uu;
        uint64_t ent;
        if (u >= G.nU_units) {
            ent = F_BAD;
        } else if (!G.offdiag) {
            ent = u;
        } else {
            uint64_t tbi, tbj;
            unit_decode(G, u, !G.pipe_diag, tbi, tbj);  // pipe_diag: diagonal units too
            const uint64_t tr = ins_bits(tbi, lt >> G.logNG, G.gr_pos, G.g);
            const uint64_t tc = ins_bits(tbj, lt & NGm, G.gr_pos, G.g);
            ent = tile_entry(G, tr, tc);
            // on a diagonal unit logical (R, C), R < C, aliases stored (C, R): it is staged as a
            // separate read-only copy (input of the transform) and never written back
            if (tbi == tbj && (lt >> G.logNG) < (lt & NGm))
                ent |= F_NOSTORE;
        }
        if (MODE == M_MONO && (!((G.active >> lt) & 1ull) || (G.groups && !((G.gmask[grp] >> lt) & 1ull))))
            ent |= F_SKIP;
        gt[i] = ent;
    }
}

// Issues (STORE = false) the bulk loads of an item into stage buffer `sb` or (STORE = true) the
// bulk stores back; executed by the 32 lanes of warp 0.
template <bool STORE>
__device__ __forceinline__ void item_copies(const Geo& G, const Tabs& T, uint64_t item, const uint64_t* gt,
                                            double2* sb, double2* __restrict__ st, uint64_t* bar, uint32_t lane) {
    const uint32_t x0 = G.sdep[item & (G.slabs - 1)];
    const uint32_t ntt = G.U << G.logNT;
    const uint32_t sbase = smem_u32(sb);
    if (G.SR == G.M) {  // whole stored tiles, either orientation: one bulk copy each, lane-parallel
        const uint32_t bytes = (1u << (2 * G.logM)) << 4;
        for (uint32_t tt = lane; tt < ntt; tt += 32) {
            const uint64_t ent = gt[tt];
            if ((ent & (F_BAD | F_SKIP)) || (STORE && (ent & F_NOSTORE)))
                continue;
            const uint64_t gbase = (ent & F_MASK) << (2 * G.logM);
            const uint32_t tsm =
                sbase + ((tt >> G.logNT) * G.A + G.slot[tt & ((1u << G.logNT) - 1)]) * G.TS * 16u;
            if (STORE)
                bulk_s2g(G.out + gbase, tsm, bytes);
            else
                bulk_g2s(tsm, tile_base(G, ent, st) + gbase, bytes, bar);
        }
        return;
    }
    for (uint32_t tt = 0; tt < ntt; ++tt) {
        const uint64_t ent = gt[tt];
        if ((ent & (F_BAD | F_SKIP)) || (STORE && (ent & F_NOSTORE)))
            continue;
        const uint64_t gbase = (ent & F_MASK) << (2 * G.logM);
        const uint32_t tsm = sbase + ((tt >> G.logNT) * G.A + G.slot[tt & ((1u << G.logNT) - 1)]) * G.TS * 16u;
        const double2* src = tile_base(G, ent, st);
        if (!(ent & F_ADJ)) {
            for (uint32_t r = lane; r < G.nruns; r += 32) {
                const uint32_t xs0 = G.run_xs[r], len = G.run_len[r];
                const uint64_t g = gbase + ((uint64_t)(x0 | T.xdep[xs0]) << G.logM);
                const uint32_t s = tsm + ((xs0 << G.logM) << 4);
                const uint32_t bytes = (len << G.logM) << 4;
                if (STORE)
                    bulk_s2g(G.out + g, s, bytes);
                else
                    bulk_g2s(s, src + g, bytes, bar);
            }
        } else {
            const uint32_t nch = G.nruns << G.logM;
            for (uint32_t c = lane; c < nch; c += 32) {
                const uint32_t y = c / G.nruns, r = c - y * G.nruns;
                const uint32_t xs0 = G.run_xs[r], len = G.run_len[r];
                const uint64_t g = gbase + ((uint64_t)y << G.logM) + (x0 | T.xdep[xs0]);
                const uint32_t s = tsm + ((y * G.SRp + xs0) << 4);
                if (STORE)
                    bulk_s2g(G.out + g, s, len << 4);
                else
                    bulk_g2s(s, src + g, len << 4, bar);
            }
        }
    }
}

__device__ __forceinline__ uint32_t item_bytes(const Geo& G, const uint64_t* gt) {
    const uint32_t ntt = G.U << G.logNT;
    uint32_t n = 0;
    for (uint32_t tt = 0; tt < ntt; ++tt)
        n += !(gt[tt] & (F_BAD | F_SKIP));
    return n * ((G.SR << G.logM) << 4);
}

// Consumer-side addressing.  Component i = rho * D + gamma of a block lives in logical tile
// ttr[i] of its unit; its shared-memory offset is unit_base + (adjoint ? a0 + cadj[i] : d0 +
// cdir[i]) with d0 / a0 the block's base offset in direct (pitch M) / adjoint (pitch SR + 1)
// orientation.  cdir / cadj / ttr are per-operation constants (kernel parameters, uniform
// indices); the adjoint pattern of a unit is one 64-bit mask.
constexpr int NCONS = 512;                  // consumer threads (16 warps)
constexpr int NTHR_PIPE = NCONS + 32 * 4;   // + one producer warp per ring stage (<= MAX_STAGES)
constexpr int MAX_UA = 64;                  // units per item with adjoint masks (g >= 1)

struct CBlk {
    uint32_t ub, d0, a0;
    uint64_t am;
};
__device__ __forceinline__ CBlk cblk(const Geo& G, const Tabs& T, const uint64_t* am_tab, uint32_t b, uint32_t& uu) {
    uint32_t xbi, ybi;
    if (G.diag_map) {
        // 8 consecutive blocks take 8 distinct rows AND 8 distinct columns (mod 8): lanes of a
        // quarter-warp then hit 8 different 16-byte bank groups in row-major (direct) and in
        // transposed (adjoint) orientation alike
        const uint32_t i = b & 7, d = (b >> 3) & 7;
        uint32_t r = b >> 6;
        const uint32_t ybh = r & ((G.nyb >> 3) - 1);
        r >>= G.logNyb - 3;
        const uint32_t xbh = r & ((G.nxb >> 3) - 1);
        uu = r >> (G.logNxb - 3);
        xbi = (xbh << 3) | i;
        ybi = (ybh << 3) | ((i + d) & 7);
    } else {
        ybi = b & (G.nyb - 1);
        xbi = (b >> G.logNyb) & (G.nxb - 1);
        uu = b >> (G.logNyb + G.logNxb);
    }
    const uint32_t xs = T.xb[xbi], y = T.yb[ybi];
    CBlk c;
    c.ub = uu * G.A * G.TS;
    c.d0 = xs * G.PD + y;
    c.a0 = G.logical ? c.d0 : y * G.SRp + xs;
    c.am = G.g ? am_tab[uu] : 0ull;
    return c;
}
__device__ __forceinline__ uint32_t caddr(const Tabs& T, const CBlk& c, uint32_t i, bool& cj) {
    cj = (c.am >> T.ttr[i]) & 1ull;
    return c.ub + (cj ? c.a0 + T.cadj[i] : c.d0 + T.cdir[i]);
}
__device__ __forceinline__ double2 ldc(const double2* sb, uint32_t a, bool cj) {
    double2 v = sb[a];
    if (cj)
        v.y = -v.y;
    return v;
}
__device__ __forceinline__ void stc(double2* sb, uint32_t a, bool cj, double2 v) {
    if (cj)
        v.y = -v.y;
    sb[a] = v;
}

// One program step on a quad, row-stacked (h00, h01, h10, h11).  kind: 0 transfer matrix,
// 1 Hadamard (native.cpp:332-339), 2 diagonal transfer, 3 real transfer coupling only (00, 11) and
// (01, 10) (depolarising, amplitude damping and their compositions), 4 real (00, 11) block with a
// complex diagonal on (01, 10) (the same channels composed with Rz / phase gates: 16 FP64
// operations per quad, as kinds 2 and 3), 5 Hadamard butterfly without its factor 1/2 (the caller
// has scaled the step before it by 1/2, which is exact).
__device__ __forceinline__ void prog_quad(uint32_t kind, const double2* S, double2& v0, double2& v1, double2& v2,
                                          double2& v3) {
    double2 w0, w1, w2, w3;
    if (kind == 1) {
        const double2 aa = make_double2(v0.x + v1.x, v0.y + v1.y), b2 = make_double2(v0.x - v1.x, v0.y - v1.y);
        const double2 cc = make_double2(v2.x + v3.x, v2.y + v3.y), dd = make_double2(v2.x - v3.x, v2.y - v3.y);
        w0 = make_double2(0.5 * (aa.x + cc.x), 0.5 * (aa.y + cc.y));
        w1 = make_double2(0.5 * (b2.x + dd.x), 0.5 * (b2.y + dd.y));
        w2 = make_double2(0.5 * (aa.x - cc.x), 0.5 * (aa.y - cc.y));
        w3 = make_double2(0.5 * (b2.x - dd.x), 0.5 * (b2.y - dd.y));
    } else if (kind == 5) {  // Hadamard butterfly without the 1/2 (folded into the step before, exactly)
        const double2 aa = make_double2(v0.x + v1.x, v0.y + v1.y), b2 = make_double2(v0.x - v1.x, v0.y - v1.y);
        const double2 cc = make_double2(v2.x + v3.x, v2.y + v3.y), dd = make_double2(v2.x - v3.x, v2.y - v3.y);
        w0 = make_double2(aa.x + cc.x, aa.y + cc.y);
        w1 = make_double2(b2.x + dd.x, b2.y + dd.y);
        w2 = make_double2(aa.x - cc.x, aa.y - cc.y);
        w3 = make_double2(b2.x - dd.x, b2.y - dd.y);
    } else if (kind == 2) {
        w0 = cmul(S[0], v0);
        w1 = cmul(S[5], v1);
        w2 = cmul(S[10], v2);
        w3 = cmul(S[15], v3);
    } else if (kind == 4) {
        w0 = make_double2(S[0].x * v0.x + S[3].x * v3.x, S[0].x * v0.y + S[3].x * v3.y);
        w3 = make_double2(S[12].x * v0.x + S[15].x * v3.x, S[12].x * v0.y + S[15].x * v3.y);
        w1 = cmul(S[5], v1);
        w2 = cmul(S[10], v2);
    } else if (kind == 3) {
        w0 = make_double2(S[0].x * v0.x + S[3].x * v3.x, S[0].x * v0.y + S[3].x * v3.y);
        w3 = make_double2(S[12].x * v0.x + S[15].x * v3.x, S[12].x * v0.y + S[15].x * v3.y);
        w1 = make_double2(S[5].x * v1.x + S[6].x * v2.x, S[5].x * v1.y + S[6].x * v2.y);
        w2 = make_double2(S[9].x * v1.x + S[10].x * v2.x, S[9].x * v1.y + S[10].x * v2.y);
    } else {
        w0 = cmul(S[0], v0); w0 = cfma(S[1], v1, w0); w0 = cfma(S[2], v2, w0); w0 = cfma(S[3], v3, w0);
        w1 = cmul(S[4], v0); w1 = cfma(S[5], v1, w1); w1 = cfma(S[6], v2, w1); w1 = cfma(S[7], v3, w1);
        w2 = cmul(S[8], v0); w2 = cfma(S[9], v1, w2); w2 = cfma(S[10], v2, w2); w2 = cfma(S[11], v3, w2);
        w3 = cmul(S[12], v0); w3 = cfma(S[13], v1, w3); w3 = cfma(S[14], v2, w3); w3 = cfma(S[15], v3, w3);
    }
    v0 = w0;
    v1 = w1;
    v2 = w2;
    v3 = w3;
}
// One program step on two quads at once: the step's coefficients are fetched once and the two
// independent dependency chains interleave on the FP64 pipe.
__device__ __forceinline__ void prog_quad2(uint32_t kind, const double2* S, double2 (&a)[4], double2 (&b)[4]) {
    if (kind == 1 || kind == 5) {
        prog_quad(kind, S, a[0], a[1], a[2], a[3]);
        prog_quad(kind, S, b[0], b[1], b[2], b[3]);
    } else if (kind == 2) {
        const double2 s0 = S[0], s1 = S[5], s2 = S[10], s3 = S[15];
        a[0] = cmul(s0, a[0]); b[0] = cmul(s0, b[0]);
        a[1] = cmul(s1, a[1]); b[1] = cmul(s1, b[1]);
        a[2] = cmul(s2, a[2]); b[2] = cmul(s2, b[2]);
        a[3] = cmul(s3, a[3]); b[3] = cmul(s3, b[3]);
    } else if (kind == 4) {
        const double p00 = S[0].x, p03 = S[3].x, p30 = S[12].x, p33 = S[15].x;
        const double2 s1 = S[5], s2 = S[10];
        auto pair = [&](double& x, double& y) {
            const double tx = p03 * y, ty = p30 * x;
            x = fma(p00, x, tx);
            y = fma(p33, y, ty);
        };
        pair(a[0].x, a[3].x); pair(b[0].x, b[3].x);
        pair(a[0].y, a[3].y); pair(b[0].y, b[3].y);
        a[1] = cmul(s1, a[1]); b[1] = cmul(s1, b[1]);
        a[2] = cmul(s2, a[2]); b[2] = cmul(s2, b[2]);
    } else if (kind == 3) {
        const double p00 = S[0].x, p03 = S[3].x, p30 = S[12].x, p33 = S[15].x;
        const double p11 = S[5].x, p12 = S[6].x, p21 = S[9].x, p22 = S[10].x;
        // in place: the cross terms first, then each result into its own operand's registers
        auto pair = [&](double& x, double& y, double cxx, double cxy, double cyx, double cyy) {
            const double tx = cxy * y, ty = cyx * x;
            x = fma(cxx, x, tx);
            y = fma(cyy, y, ty);
        };
        auto one = [&](double2 (&v)[4]) {
            pair(v[0].x, v[3].x, p00, p03, p30, p33);
            pair(v[0].y, v[3].y, p00, p03, p30, p33);
            pair(v[1].x, v[2].x, p11, p12, p21, p22);
            pair(v[1].y, v[2].y, p11, p12, p21, p22);
        };
        one(a);
        one(b);
    } else {
        prog_quad(0, S, a[0], a[1], a[2], a[3]);
        prog_quad(0, S, b[0], b[1], b[2], b[3]);
    }
}

// In-tile programs: what a consumer thread needs per pass (one pass per qubit, at most MAXP), the
// same for every item -- the bases of its two quads (bits 0-15, 16-31) and the pass's last step
struct ProgPre {
    static constexpr int MAXP = 5;
    uint32_t base[MAXP], end[MAXP];
    uint32_t pairm;  // bit ps: passes ps and ps + 1 share one shared-memory round trip (pipe_compute)
    bool ok;
};
template <int K, int MODE, int NS, int NC = NCONS>
__device__ __forceinline__ void pipe_compute(const Geo& G, const Tabs& T, const Coef<NS>& cf, const uint64_t* am,
                                             uint32_t nvalid_units, double2* sb, uint32_t grp = 0, int tidv = -1,
                                             uint32_t barid = 1, const ProgPre* pre = nullptr) {
    constexpr int D = 1 << K;
    const int tid = tidv >= 0 ? tidv : (int)threadIdx.x;
    const uint32_t nblk = G.U << (G.logNxb + G.logNyb);
    const uint32_t lo = G.diag_map ? 3u : G.logNyb, lomask = (1u << lo) - 1;
    if constexpr (MODE == M_S1 || MODE == M_HAD) {
        const Coef<16>& c16 = *reinterpret_cast<const Coef<16>*>(&cf);
        for (uint32_t b = tid; b < nblk; b += NC) {
            uint32_t uu;
            const CBlk c = cblk(G, T, am, b, uu);
            if (uu >= nvalid_units)
                continue;
            bool c0, c1, c2, c3;
            const uint32_t a0 = caddr(T, c, 0, c0), a1 = caddr(T, c, 1, c1);
            const uint32_t a2 = caddr(T, c, 2, c2), a3 = caddr(T, c, 3, c3);
            const double2 v0 = ldc(sb, a0, c0), v1 = ldc(sb, a1, c1), v2 = ldc(sb, a2, c2), v3 = ldc(sb, a3, c3);
            double2 w0, w1, w2, w3;
            if (MODE == M_HAD) {  // HadamardQuad (native.cpp:332-339)
                const double2 a = make_double2(v0.x + v1.x, v0.y + v1.y), bb = make_double2(v0.x - v1.x, v0.y - v1.y);
                const double2 cc = make_double2(v2.x + v3.x, v2.y + v3.y), d = make_double2(v2.x - v3.x, v2.y - v3.y);
                w0 = make_double2(0.5 * (a.x + cc.x), 0.5 * (a.y + cc.y));
                w1 = make_double2(0.5 * (bb.x + d.x), 0.5 * (bb.y + d.y));
                w2 = make_double2(0.5 * (a.x - cc.x), 0.5 * (a.y - cc.y));
                w3 = make_double2(0.5 * (bb.x - d.x), 0.5 * (bb.y - d.y));
            } else if (c16.xpat) {  // TransferQuad with only (00, 11) / (01, 10) couplings
                const double2* s = c16.s;
                w0 = cfma(s[3], v3, cmul(s[0], v0));
                w3 = cfma(s[15], v3, cmul(s[12], v0));
                w1 = cfma(s[6], v2, cmul(s[5], v1));
                w2 = cfma(s[10], v2, cmul(s[9], v1));
            } else {  // TransferQuad (kernels.cpp:66-77)
                const double2* s = c16.s;
                w0 = cmul(s[0], v0); w0 = cfma(s[1], v1, w0); w0 = cfma(s[2], v2, w0); w0 = cfma(s[3], v3, w0);
                w1 = cmul(s[4], v0); w1 = cfma(s[5], v1, w1); w1 = cfma(s[6], v2, w1); w1 = cfma(s[7], v3, w1);
                w2 = cmul(s[8], v0); w2 = cfma(s[9], v1, w2); w2 = cfma(s[10], v2, w2); w2 = cfma(s[11], v3, w2);
                w3 = cmul(s[12], v0); w3 = cfma(s[13], v1, w3); w3 = cfma(s[14], v2, w3); w3 = cfma(s[15], v3, w3);
            }
            stc(sb, a0, c0, w0);
            stc(sb, a1, c1, w1);
            stc(sb, a2, c2, w2);
            stc(sb, a3, c3, w3);
        }
    } else if constexpr (MODE == M_S2) {
        const Coef<256>& c256 = *reinterpret_cast<const Coef<256>*>(&cf);
        for (uint32_t b = tid; b < nblk; b += NC) {
            uint32_t uu;
            const CBlk c = cblk(G, T, am, b, uu);
            if (uu >= nvalid_units)
                continue;
            double2 v[16];
            uint32_t a[16];
            uint32_t cjm = 0;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                bool cj;
                a[i] = caddr(T, c, i, cj);
                cjm |= (uint32_t)cj << i;
                v[i] = ldc(sb, a[i], cj);
            }
#pragma unroll 2
            for (int r = 0; r < 16; ++r) {
                double2 acc = cmul(c256.s[r * 16], v[0]);
#pragma unroll
                for (int q = 1; q < 16; ++q)
                    acc = cfma(c256.s[r * 16 + q], v[q], acc);
                stc(sb, a[r], (cjm >> r) & 1u, acc);
            }
        }
    } else if constexpr (MODE == M_DIRECT) {
        const uint32_t items = nblk * D;
        for (uint32_t w = tid; w < items; w += NC) {  // Y = B L^dagger, row by row
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo), rho = (w >> lo) % D;
            uint32_t uu;
            const CBlk c = cblk(G, T, am, b, uu);
            if (uu >= nvalid_units)
                continue;
            double2 v[D];
            uint32_t a[D];
            uint32_t cjm = 0;
#pragma unroll
            for (int q = 0; q < D; ++q) {
                bool cj;
                a[q] = caddr(T, c, rho * D + q, cj);
                cjm |= (uint32_t)cj << q;
                v[q] = ldc(sb, a[q], cj);
            }
#pragma unroll
            for (int q = 0; q < D; ++q) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int t = 0; t < D; ++t)
                    acc = cfmaconj(v[t], cf.s[q * D + t], acc);
                stc(sb, a[q], (cjm >> q) & 1u, acc);
            }
        }
        asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NC) : "memory");  // consumer warps only
        for (uint32_t w = tid; w < items; w += NC) {  // out = L Y, column by column
            const uint32_t b = (w & lomask) | (((w >> lo) / D) << lo), gam = (w >> lo) % D;
            uint32_t uu;
            const CBlk c = cblk(G, T, am, b, uu);
            if (uu >= nvalid_units)
                continue;
            double2 v[D];
            uint32_t a[D];
            uint32_t cjm = 0;
#pragma unroll
            for (int r = 0; r < D; ++r) {
                bool cj;
                a[r] = caddr(T, c, r * D + gam, cj);
                cjm |= (uint32_t)cj << r;
                v[r] = ldc(sb, a[r], cj);
            }
#pragma unroll
            for (int r = 0; r < D; ++r) {
                double2 acc = make_double2(0.0, 0.0);
#pragma unroll
                for (int t = 0; t < D; ++t)
                    acc = cfma(cf.s[r * D + t], v[t], acc);
                stc(sb, a[r], (cjm >> r) & 1u, acc);
            }
        }
    } else if constexpr (MODE == M_PROG) {
        // fused program: single-qubit steps on in-tile bits applied to the staged whole
        // tiles one after another (one HBM pass for the whole run; the host composes the run's
        // operations per qubit).  Quads of step p: rows (x, x + 2^a) x columns (y, y + 2^a),
        // row-stacked (h00, h01, h10, h11) as TransferQuad (kernels.cpp:66-77); consecutive threads
        // take consecutive quads along a row.
        // Consecutive steps on the same qubit share one round trip through shared memory: the quad
        // stays in registers while the chain (e.g. depolarising, Rz, H in their cheap forms) runs.
        const uint32_t lq = G.logM - 1, nq = nvalid_units << (2 * lq), M = G.M;
        // two quads per thread and pass (4 whole tiles per item, 512 consumers): both are loaded
        // before either chain runs (the compiler cannot hoist shared loads over shared stores
        // itself), the step's coefficients are fetched once and the two chains interleave; the quad
        // bases come precomputed (ProgPre)
        if (pre && pre->ok && nq == 2 * NC) {
            uint32_t p = 0;
#pragma unroll
            for (int ps = 0; ps < ProgPre::MAXP; ++ps) {
                if (ps > 0 && ((pre->pairm >> (ps - 1)) & 1u))
                    continue;  // the second pass of a pair ran with the first
                if (p < cf.nsteps) {
                    const uint32_t sa = 1u << cf.pbit[p], ba = pre->base[ps] & 0xffffu, bb = pre->base[ps] >> 16;
                    const uint32_t o1 = sa, o2 = sa * M, o3 = o2 + sa;
                    double2 va[4] = {sb[ba], sb[ba + o1], sb[ba + o2], sb[ba + o3]};
                    double2 vb[4] = {sb[bb], sb[bb + o1], sb[bb + o2], sb[bb + o3]};
                    for (uint32_t pp = p; pp < pre->end[ps]; ++pp)
                        prog_quad2(cf.pkind[pp], cf.s + 16 * pp, va, vb);
                    if (ps + 1 < ProgPre::MAXP && ((pre->pairm >> ps) & 1u)) {
                        // Paired passes (qubits a, b): lanes l and l ^ 16 hold the four a-quads of one
                        // 4 x 4 block (rows / columns x0 + {0, 2^a, 2^b, 2^a + 2^b}), this lane those of
                        // block row bit b = its role.  After the a-chains role 0 keeps the a-row-0
                        // halves of its quads and gets the partner's, role 1 the a-row-1 halves: two
                        // b-quads per lane without a trip through shared memory (16 shuffles instead of
                        // 8 stores, a barrier and 8 loads).
                        const bool r1 = (threadIdx.x & 16u) != 0;
                        auto xch = [&](double2& keep_or_send0, double2& keep_or_send1) {
                            // role 0 sends element [2] / [3] and keeps [0] / [1]; role 1 the other way round
                            double2 snd = r1 ? keep_or_send0 : keep_or_send1;
                            snd.x = __shfl_xor_sync(0xffffffffu, snd.x, 16);
                            snd.y = __shfl_xor_sync(0xffffffffu, snd.y, 16);
                            if (r1)
                                keep_or_send0 = snd;
                            else
                                keep_or_send1 = snd;
                        };
                        xch(va[0], va[2]);
                        xch(vb[0], vb[2]);
                        xch(va[1], va[3]);
                        xch(vb[1], vb[3]);
                        double2 wa[4] = {va[0], vb[0], va[2], vb[2]}, wb[4] = {va[1], vb[1], va[3], vb[3]};
                        const uint32_t p2 = pre->end[ps], e2 = pre->end[ps + 1];
                        for (uint32_t pp = p2; pp < e2; ++pp)
                            prog_quad2(cf.pkind[pp], cf.s + 16 * pp, wa, wb);
                        const uint32_t sb2 = 1u << cf.pbit[p2], qa = pre->base[ps + 1] & 0xffffu, qb = pre->base[ps + 1] >> 16;
                        const uint32_t q1 = sb2, q2 = sb2 * M, q3 = q2 + sb2;
                        sb[qa] = wa[0];
                        sb[qa + q1] = wa[1];
                        sb[qa + q2] = wa[2];
                        sb[qa + q3] = wa[3];
                        sb[qb] = wb[0];
                        sb[qb + q1] = wb[1];
                        sb[qb + q2] = wb[2];
                        sb[qb + q3] = wb[3];
                        p = e2;
                        if (p < cf.nsteps)
                            asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NC) : "memory");  // consumer warps only
                        continue;
                    }
                    sb[ba] = va[0];
                    sb[ba + o1] = va[1];
                    sb[ba + o2] = va[2];
                    sb[ba + o3] = va[3];
                    sb[bb] = vb[0];
                    sb[bb + o1] = vb[1];
                    sb[bb + o2] = vb[2];
                    sb[bb + o3] = vb[3];
                    p = pre->end[ps];
                    if (p < cf.nsteps)
                        asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NC) : "memory");  // consumer warps only
                }
            }
            return;
        }
        for (uint32_t p = 0; p < cf.nsteps;) {
            const uint32_t a = cf.pbit[p], sa = 1u << a, lo = sa - 1;
            uint32_t p1 = p + 1;
            while (p1 < cf.nsteps && cf.pbit[p1] == a)
                ++p1;
            auto quad_base = [&](uint32_t q) {
                const uint32_t u = q >> (2 * lq), r = q & ((1u << (2 * lq)) - 1);
                const uint32_t qx = r >> lq, qy = r & ((1u << lq) - 1);
                const uint32_t x = ((qx & ~lo) << 1) | (qx & lo), y = ((qy & ~lo) << 1) | (qy & lo);
                return u * G.A * G.TS + x * M + y;
            };
            for (uint32_t q = tid; q < nq; q += NC) {
                const uint32_t b0 = quad_base(q);
                const uint32_t b1 = b0 + sa, b2 = b0 + sa * M, b3 = b2 + sa;
                double2 v0 = sb[b0], v1 = sb[b1], v2 = sb[b2], v3 = sb[b3];
                for (uint32_t pp = p; pp < p1; ++pp)
                    prog_quad(cf.pkind[pp], cf.s + 16 * pp, v0, v1, v2, v3);
                sb[b0] = v0;
                sb[b1] = v1;
                sb[b2] = v2;
                sb[b3] = v3;
            }
            if (p1 < cf.nsteps)
                asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NC) : "memory");  // consumer warps only
            p = p1;
        }
    } else if constexpr (MODE == M_MONO) {
        if (cf.diag && cf.nib == 0 && !G.groups && G.SR == G.M && !G.logical) {
            // diagonal phases on grid qubits only: every element of a staged logical tile (R, C)
            // gets the tile's factor f(R, C) (adjoint tiles, in stored orientation: conj f); the
            // cycle walk below costs ~8x more instructions per element for this case
            const uint32_t lMM = 2 * G.logM, D = 1u << K;
            const uint32_t nel = nvalid_units * G.A << lMM;
            for (uint32_t e = tid; e < nel; e += NC) {
                const uint32_t st_ = e >> lMM, uu = st_ / G.A, sl = st_ - uu * G.A;
                const uint32_t t = T.slt[sl], comp = (t >> G.logNG) * D + (t & ((1u << G.logNG) - 1));
                if ((cf.fone >> comp) & 1ull)
                    continue;
                double2 f = cf.s[comp];
                if ((am[uu] >> t) & 1ull)
                    f.y = -f.y;
                const uint32_t addr = (uu * G.A + sl) * G.TS + (e & ((1u << lMM) - 1));
                sb[addr] = cmul(f, sb[addr]);
            }
            return;
        }
        // in-place cycles of the component map; untouched components cost nothing
        const uint32_t cbeg = G.groups ? cf.gcyc_off[grp] : 0;
        const uint32_t nc = G.groups ? cf.gcyc_off[grp + 1] - cbeg : cf.ncyc;
        const uint32_t items = nblk * nc;
        for (uint32_t w = tid; w < items; w += NC) {
            const uint32_t b = (w & lomask) | (((w >> lo) / nc) << lo), ci = cbeg + (w >> lo) % nc;
            uint32_t uu;
            const CBlk c = cblk(G, T, am, b, uu);
            if (uu >= nvalid_units)
                continue;
            const uint32_t c0 = cf.cyc_off[ci], len = cf.cyc_off[ci + 1] - c0;
            if (len <= 2) {  // fixed points with a factor, and transpositions (all library gates)
                const uint32_t p0 = cf.cyc[c0], p1 = cf.cyc[c0 + len - 1];
                bool j0, j1;
                const uint32_t a0 = caddr(T, c, p0, j0), a1 = caddr(T, c, p1, j1);
                const double2 v0 = ldc(sb, a0, j0), v1 = ldc(sb, a1, j1);
                double2 x0 = v1, x1 = v0;  // out[p0] = f in[p1], out[p1] = f in[p0]
                if (!((cf.fone >> p0) & 1ull))
                    x0 = cmul(cf.s[p0], x0);
                stc(sb, a0, j0, x0);
                if (len == 2) {
                    if (!((cf.fone >> p1) & 1ull))
                        x1 = cmul(cf.s[p1], x1);
                    stc(sb, a1, j1, x1);
                }
                continue;
            }
            double2 v[16];
            uint32_t a[16];
            uint32_t cjm = 0;
            for (uint32_t j = 0; j < len; ++j) {
                bool cj;
                a[j] = caddr(T, c, cf.cyc[c0 + j], cj);
                cjm |= (uint32_t)cj << j;
                v[j] = ldc(sb, a[j], cj);
            }
            for (uint32_t j = 0; j < len; ++j) {
                const uint32_t comp = cf.cyc[c0 + j];
                double2 x = v[j + 1 == len ? 0 : j + 1];
                if (!((cf.fone >> comp) & 1ull))
                    x = cmul(cf.s[comp], x);
                stc(sb, a[j], (cjm >> j) & 1u, x);
            }
        }
    }
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void bulk_wait_read0() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }

template <int K, int MODE, int NS>
__global__ void __launch_bounds__(NTHR_PIPE, 1) pipe_kernel(const Geo G, const Coef<NS> cf, double2* __restrict__ st) {
    extern __shared__ __align__(128) double2 ring[];
    __shared__ __align__(8) uint64_t full[MAX_STAGES];
    __shared__ __align__(8) uint64_t done[MAX_STAGES];
    __shared__ uint64_t gt[MAX_STAGES][MAX_TT];
    __shared__ uint64_t am[MAX_STAGES][MAX_UA];
    __shared__ uint64_t gnext[MAX_STAGES][MAX_TT];
    __shared__ Tabs T;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid < 32) {
        T.xdep[tid] = G.xdep[tid];
        T.xb[tid] = G.xb_tab[tid];
        T.yb[tid] = G.yb_tab[tid];
        T.xs_rin[tid] = G.xs_rin[tid];
        T.xs_base[tid] = G.xs_base[tid];
        T.y_cin[tid] = G.y_cin[tid];
        T.y_base[tid] = G.y_base[tid];
        if (tid < 8) {
            T.xs_in[tid] = G.xs_in[tid];
            T.y_in[tid] = G.y_in[tid];
        }
    }
    if (tid < 64) {
        T.cdir[tid] = G.cdir[tid];
        T.cadj[tid] = G.cadj[tid];
        T.ttr[tid] = G.ttr[tid];
        if ((G.active >> tid) & 1ull)
            T.slt[G.slot[tid]] = (uint8_t)tid;
    }
    if (tid == 0) {
        for (uint32_t s = 0; s < G.stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&done[s], NCONS / 32);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t nItems = G.nU_items;
    const uint32_t S = G.stages;
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;

    if (warp >= NCONS / 32) {
        // ---- producer warps: warp p owns ring stage p (items j = p, p + S, ...).  A bulk
        // store can only be awaited by the thread that issued it, so giving every stage its own
        // producer lets the stages' store-drain / metadata / load-issue latencies overlap.
        const uint32_t p = warp - NCONS / 32;
        if (p >= S)
            return;
        const uint32_t ntt = G.U << G.logNT;
        uint64_t* gn = gnext[p];
        double2* sb = ring + (size_t)p * G.stage_elems;
        for (uint64_t j = p; j < nlocal + S; j += S) {
            uint32_t bytes = 0;
            if (j < nlocal) {  // metadata of item j, prepared before the stage is free
                item_tiles<MODE>(G, sweep_item(G, nItems, j), gn, lane);
                __syncwarp();
                uint32_t cnt = 0;
                for (uint32_t t = lane; t < ntt; t += 32)
                    cnt += !(gn[t] & (F_BAD | F_SKIP));
                for (int o = 16; o; o >>= 1)
                    cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
                bytes = cnt * ((G.SR << G.logM) << 4);
            }
            if (j >= S) {
                const uint64_t jj = j - S;
                mbar_wait(&done[p], (uint32_t)((jj / S) & 1));
                item_copies<true>(G, T, sweep_item(G, nItems, jj), gt[p], sb, st, nullptr, lane);
                bulk_commit();
            }
            if (j < nlocal) {
                for (uint32_t t = lane; t < ntt; t += 32)
                    gt[p][t] = gn[t];
                __syncwarp();
                if (G.g)
                    for (uint32_t uu = lane; uu < G.U && uu < MAX_UA; uu += 32) {
                        uint64_t mask = 0;
                        for (uint32_t t = 0; t < (1u << G.logNT); ++t)
                            mask |= (uint64_t)((gn[(uu << G.logNT) + t] & F_ADJ) != 0) << t;
                        am[p][uu] = mask;
                    }
                if (j >= S)
                    bulk_wait_read0();  // the store of item j - S has left the stage
                __syncwarp();
                if (G.dbg & DBG_POISON) {  // diagnostics: the stage holds NaN until the loads land
                    poison_stage(sb, G.stage_elems, lane, 32);
                    __syncwarp();
                }
                if (lane == 0)
                    mbar_arrive_expect(&full[p], bytes);
                __syncwarp();
                item_copies<false>(G, T, sweep_item(G, nItems, j), gt[p], sb, st, &full[p], lane);
            }
        }
        bulk_wait_all();
        return;
    }
    // ---- consumer warps: transform each staged item in place
    ProgPre pre;
    pre.ok = false;
    pre.pairm = 0;
    if constexpr (MODE == M_PROG) {
        const uint32_t lq = G.logM - 1, tid = threadIdx.x;
        uint32_t p = 0;
#pragma unroll
        for (int ps = 0; ps < ProgPre::MAXP; ++ps) {
            pre.base[ps] = 0;
            pre.end[ps] = 0;
            if (p < cf.nsteps) {
                uint32_t p1 = p + 1;
                while (p1 < cf.nsteps && cf.pbit[p1] == cf.pbit[p])
                    ++p1;
                const uint32_t lo = (1u << cf.pbit[p]) - 1;
#pragma unroll
                for (uint32_t h = 0; h < 2; ++h) {
                    uint32_t q = tid + h * NCONS;
                    // skewed tiles (hs_apply_program: tile u at u * (M^2 + 1), one 16-B bank group
                    // apart): for qubits 0 and 1 a quarter-warp's 8 lanes take 4 column pairs of
                    // two tiles that are 1 / 2 bank groups apart (thread bit 2 <-> tile bit a), so
                    // their 8 loads of one quad element hit 8 distinct bank groups; otherwise they
                    // hit 4, each twice
                    if (G.logM == 5 && (G.TS & 7u) == 1u && cf.pbit[p] < 2) {
                        const uint32_t hb = 8 + cf.pbit[p], d = ((q >> 2) ^ (q >> hb)) & 1u;
                        q ^= (d << 2) | (d << hb);
                    }
                    const uint32_t u = q >> (2 * lq), r = q & ((1u << (2 * lq)) - 1);
                    const uint32_t qx = r >> lq, qy = r & ((1u << lq) - 1);
                    const uint32_t x = ((qx & ~lo) << 1) | (qx & lo), y = ((qy & ~lo) << 1) | (qy & lo);
                    pre.base[ps] |= (u * G.A * G.TS + x * G.M + y) << (16 * h);
                }
                pre.end[ps] = p1;
                p = p1;
            }
        }
        pre.ok = p >= cf.nsteps && !(G.dbg & 2048u);  // bit 11: the one-quad loop
        // Pairs of passes (0, 1), (2, 3) on skewed whole 32 x 32 tiles, two quads per thread (bit 15: off).
        // Block bits <- thread bits 0-3, 5-8 (bit 4 is the role): the free column bits below 3 first, then
        // tile bits (tiles lie 1 / 2 bank groups apart), so a quarter-warp's 8 lanes spread over the bank
        // groups as far as the pair allows; then the other column bits, the row bits, the other tile bits.
        pre.pairm = 0;
        if (pre.ok && G.logM == 5 && (G.TS & 7u) == 1u && (G.U << (2 * lq)) == 2 * NCONS && !(G.dbg & 32768u)) {
            for (int ps = 0; ps + 1 < ProgPre::MAXP; ps += 2) {
                if (!pre.end[ps + 1])
                    break;
                const uint32_t a = cf.pbit[pre.end[ps] - 1], b = cf.pbit[pre.end[ps + 1] - 1];
                if (a == b)
                    break;
                uint32_t fb[3], k = 0;
                for (uint32_t q = 0; q < 5; ++q)
                    if (q != a && q != b)
                        fb[k++] = q;
                const uint32_t tb = (tid & 15u) | ((tid >> 5) << 4), role = (tid >> 4) & 1u;
                uint32_t x0 = 0, y0 = 0, u = 0, i = 0, usedc = 0, usedu = 0;
                for (uint32_t j = 0; j < 3; ++j)
                    if (fb[j] < 3) {
                        y0 |= ((tb >> i++) & 1u) << fb[j];
                        usedc |= 1u << j;
                    }
                for (uint32_t ub = 0; ub < 2 && i < 3; ++ub) {
                    u |= ((tb >> i++) & 1u) << ub;
                    usedu |= 1u << ub;
                }
                for (uint32_t j = 0; j < 3; ++j)
                    if (!((usedc >> j) & 1u))
                        y0 |= ((tb >> i++) & 1u) << fb[j];
                for (uint32_t j = 0; j < 3; ++j)
                    x0 |= ((tb >> i++) & 1u) << fb[j];
                for (uint32_t ub = 0; ub < 2; ++ub)
                    if (!((usedu >> ub) & 1u))
                        u |= ((tb >> i++) & 1u) << ub;
                const uint32_t B = u * G.A * G.TS + x0 * G.M + y0, sa = 1u << a, sb2 = 1u << b;
                const uint32_t ba = B + role * sb2 * G.M, qa = B + role * sa * G.M;
                pre.base[ps] = ba | ((ba + sb2) << 16);
                pre.base[ps + 1] = qa | ((qa + sa) << 16);
                pre.pairm |= 1u << ps;
            }
        }
    }
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = (uint32_t)(i % S);
        double2* sb = ring + (size_t)s * G.stage_elems;
        const uint64_t item = sweep_item(G, nItems, i);
        const uint32_t grp = G.groups ? (uint32_t)(item % G.groups) : 0;
        const uint64_t u0 = G.groups ? item / G.groups : (item >> G.logSlabs) << G.logU;
        const uint32_t nvalid = G.nU_units - u0 < G.U ? (uint32_t)(G.nU_units - u0) : G.U;
        mbar_wait(&full[s], (uint32_t)((i / S) & 1));
        pipe_compute<K, MODE, NS>(G, T, cf, am[s], nvalid, sb, grp, -1, 1, &pre);
        fence_async_smem();
        __syncwarp();
        if (lane == 0)
            mbar_arrive(&done[s]);
    }
}


}  // namespace
