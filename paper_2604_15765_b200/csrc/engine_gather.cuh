// engine_gather.cuh -- part of engine.cu (one translation unit; included in order).
// Gather kernels for units that do not fit whole (g >= 2; k = 3 with g = 1): the ping-pong
// cp.async gather and the warp-specialised gather with the FP64 tensor-core (DMMA) transforms
// and grid programs.
#pragma once

namespace {
// ------------------------------------------------------------- gather kernel (g >= 2: sub-blocks)
// Units with >= 2 grid bits couple 16 or 64 stored tiles, too many for whole-tile staging.  An item
// is then one S0 x S0 sub-block of positions (closed under the in-tile target bits) of every
// logical tile of a unit (4096 elements, 64 KiB); rows of S0 elements are whole cache lines in
// both orientations.  All 512 threads gather with cp.async (16 B each, adjoint tiles transposed on
// the way in, padded pitch S0 + 1), 3-stage software pipeline (commit/wait groups), transform in
// shared memory, and write back with coalesced st.global along stored rows.
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// k = 3 direct form L B L^dagger on the FP64 tensor path (mma.sync m8n8k4 f64): one warp per 8x8
// block, 16 DMMA per block (4 real products per complex product, two k = 4 chunks, two stages) in
// place of 1024 DFMA.  The contraction index k of each chunk j is permuted to k = 2c + j (c = lane
// & 3): the stage-1 accumulator fragment (row lane >> 2, columns 2c, 2c + 1) is then exactly the
// stage-2 A fragment of chunks 0 and 1, so no data moves between lanes.  Lane (g = lane >> 2, c)
// loads B[2c + j][g] and stores Z[g][2c + j].  (B200: DMMA and DFMA share the FP64 pipe at
// ~37 TFLOP/s, tools/fp64_probe.cu; DMMA issues 8x fewer instructions.)
// (not volatile: a pure function of its operands, so the compiler may interleave independent chains)
__device__ __forceinline__ void dmma_acc(double& d0, double& d1, double a, double b) {
    asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
        : "+d"(d0), "+d"(d1)
        : "d"(a), "d"(b));
}
__device__ __forceinline__ void dmma_acc_v(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1)
                 : "d"(a), "d"(b));
}
// conjugation flag applied as a sign-bit flip on the integer pipe (a DADD negation would compete
// with the DMMA for the FP64 pipe)
__device__ __forceinline__ double flip_sign(double x, uint32_t m) {
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
// per-lane constant fragments of the transform (loaded once per kernel: the lane-dependent
// coefficient index would serialise the constant-cache reads if repeated per item)
struct DmmaFrag {
    double lr[2], li[2];
    double ls[2], ld[2];      // Lr + Li (stage 1, 3M) and Pr + Pi = Lr - Li (stage 2, 3M)
    uint32_t old[2], ost[2];  // staging offsets of the loaded / stored components (from the block base)
    uint32_t tld[2], tst[2];  // their logical tiles (adjoint mask bits)
    uint32_t oldA[2], ostA[2];  // bulk staging: the same components in an adjoint tile (stored orientation)
};
// k = 3: the 8 x 8 block itself.  k = 2: four 4 x 4 blocks (2X + R1, 2Y + C1) as the quadrants of
// one 8 x 8 matrix M, transformed by I2 (x) L: (I2 (x) L) M (I2 (x) L)^dagger applies L . L^dagger to
// every quadrant, so one tensor-core transform serves four k = 2 blocks (quadrant offsets
// (R1 * PD + C1) * qstride, folded into the component offsets).
// TMA boxes (G.tma): component (sub-block x, y) of tile t sits in the 8 x 8 box (x >> 3, y >> 3) of
// the tile, stored orientation, SWIZZLE_128B with phase phi (absolute smem address bits 7-9 of the
// box base): element offset base + xs * 8 + (ys ^ ((xs + phi) & 7)), (xs, ys) the in-box position.
// Packed per access: base (12 bits) | phi << 12 | in-box x << 15 | in-box y << 18, for a direct and
// an adjoint (transposed) placement.
__device__ __forceinline__ uint32_t tma_pack(const Geo& G, const Tabs& T, uint32_t t, uint32_t xo, uint32_t yo) {
    const uint32_t nbx = G.S0 >> 3, slot = t * nbx * nbx + (xo >> 3) * nbx + (yo >> 3);
    return T.cdir[slot] | ((uint32_t)T.tsk[slot] << 12) | ((xo & 7u) << 15) | ((yo & 7u) << 18);
}
__device__ __forceinline__ uint32_t tma_addr(uint32_t pk, uint32_t xb, uint32_t yb) {
    const uint32_t xs = xb | ((pk >> 15) & 7u), ys = yb | ((pk >> 18) & 7u);
    return (pk & 0xfffu) + xs * 8u + (ys ^ ((xs + (pk >> 12)) & 7u));
}
template <int K, int NS, bool BULK = false, bool TMAB = false>
__device__ __forceinline__ DmmaFrag dmma_frag(const Geo& G, const Tabs& T, const Coef<NS>& cf) {
    DmmaFrag f;
    const uint32_t lane = threadIdx.x & 31, gq = lane >> 2, cq = lane & 3;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
        const uint32_t c8 = 2 * cq + j;
        double2 l;
        if constexpr (K == 3)
            l = cf.s[gq * 8 + c8];
        else
            l = (gq >> 2) == (c8 >> 2) ? cf.s[(gq & 3) * 4 + (c8 & 3)] : make_double2(0.0, 0.0);
        f.lr[j] = l.x;
        f.li[j] = l.y;
        f.ls[j] = l.x + l.y;
        f.ld[j] = l.x - l.y;
        if constexpr (K == 3) {
            const uint32_t il = c8 * 8 + gq, is = gq * 8 + c8;
            f.old[j] = T.cdir[il];
            f.ost[j] = T.cdir[is];
            f.tld[j] = T.ttr[il];
            f.tst[j] = T.ttr[is];
            if constexpr (TMAB) {  // component (row, col) offsets xs_in[row], y_in[col] (kin bits)
                const uint32_t km = (1u << G.kin) - 1;
                // G.tq == 4: this warp's quadrant supplies bit 3 of the block row / column
                const uint32_t qx = G.tq == 4 ? (((threadIdx.x >> 5) & 3u) >> 1) << 3 : 0u;
                const uint32_t qy = G.tq == 4 ? ((threadIdx.x >> 5) & 1u) << 3 : 0u;
                const uint32_t xl = T.xs_in[c8 & km] | qx, yl = T.y_in[gq & km] | qy;
                const uint32_t xs = T.xs_in[gq & km] | qx, ys = T.y_in[c8 & km] | qy;
                f.old[j] = tma_pack(G, T, T.ttr[il], xl, yl);
                f.oldA[j] = tma_pack(G, T, T.ttr[il], yl, xl);
                f.ost[j] = tma_pack(G, T, T.ttr[is], xs, ys);
                f.ostA[j] = tma_pack(G, T, T.ttr[is], ys, xs);
            } else if constexpr (BULK) {
                f.oldA[j] = T.cadj[il];
                f.ostA[j] = T.cadj[is];
            }
        } else {
            // load component (row c8, column gq), store component (row gq, column c8) of M
            const uint32_t il = (c8 & 3) * 4 + (gq & 3), is = (gq & 3) * 4 + (c8 & 3);
            f.old[j] = T.cdir[il] + ((c8 >> 2) * G.PD + (gq >> 2)) * G.qstride;
            f.ost[j] = T.cdir[is] + ((gq >> 2) * G.PD + (c8 >> 2)) * G.qstride;
            f.tld[j] = T.ttr[il];
            f.tst[j] = T.ttr[is];
            if constexpr (BULK) {  // transposed quadrant offsets in stored orientation
                f.oldA[j] = T.cadj[il] + ((gq >> 2) * G.PD + (c8 >> 2)) * G.qstride;
                f.ostA[j] = T.cadj[is] + ((c8 >> 2) * G.PD + (gq >> 2)) * G.qstride;
            }
        }
    }
    return f;
}
// KS: Kraus sum sum_a L_a B L_a^dagger over nk operators whose per-lane fragment values come from
// shared memory (kf[a][8][lane]: Lr, Li, Lr + Li, Lr - Li for chunks 0, 1), accumulated in registers.
template <int NC, int K = 3, bool BULK = false, bool TMAB = false, bool KS = false, bool WIDE_REGS = false>
__device__ __forceinline__ void dmma_direct3(const Geo& G, const Tabs& T, const DmmaFrag& f, uint64_t am,
                                             double2* sb, uint32_t warp, const double* kf = nullptr,
                                             uint32_t nk = 1) {
    const uint32_t lane = threadIdx.x & 31u;
    // blocks per pass: two independent chains for the unitary; one for the Kraus sum at 80 registers
    // (its accumulators would otherwise spill), two with the 128 registers of a 512-thread CTA
    constexpr int NQ = (KS && !WIDE_REGS) ? 1 : 2;
    constexpr uint32_t sh = K == 3 ? 0u : 1u;  // k = 2: 8 x 8 matrices of 2 x 2 blocks
    const uint32_t cld0 = (uint32_t)((am >> f.tld[0]) & 1ull) << 31, cld1 = (uint32_t)((am >> f.tld[1]) & 1ull) << 31;
    const uint32_t cst0 = (uint32_t)((am >> f.tst[0]) & 1ull) << 31, cst1 = (uint32_t)((am >> f.tst[1]) & 1ull) << 31;
    const uint32_t logNy = G.logNyb - sh, ymask = (G.nyb >> sh) - 1;
    // blocks per tile; G.grp4: an item is 4 independent whole tiles (in-tile k = 3), slot bt at bt * TS
    const uint32_t lbt = (G.logNxb - sh) + logNy, nblk = (G.grp4 ? 4u : 1u) << lbt;
    // two blocks per pass: independent accumulator chains keep the FP64 tensor pipe fed (small
    // tiles, m < 5, have fewer blocks than warps: the second block of a pass may be absent and is
    // then computed on a copy of the first and not stored)
    auto pass = [&](uint32_t b0, uint32_t b1, bool two) {
        uint32_t base[2], baseA[2];
        double2 v0[2], v1[2];
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            const uint32_t bq0 = (q && two) ? b1 : b0, bq = bq0 & ((1u << lbt) - 1);
            uint32_t xbv = T.xb[(bq >> logNy) << sh], ybv = T.yb[(bq & ymask) << sh];
            base[q] = (bq0 >> lbt) * G.TS + xbv * G.PD + ybv;
            if constexpr (TMAB) {  // swizzled boxes; base carries the in-box block position (the box
                xbv &= 7u;         // row / column of a quadrant, G.tq == 4, is in the fragment constants)
                ybv &= 7u;
                base[q] = (xbv << 8) | ybv;
                v0[q] = sb[cld0 ? tma_addr(f.oldA[0], ybv, xbv) : tma_addr(f.old[0], xbv, ybv)];
                v1[q] = sb[cld1 ? tma_addr(f.oldA[1], ybv, xbv) : tma_addr(f.old[1], xbv, ybv)];
            } else if constexpr (BULK) {  // adjoint tiles in stored orientation: row y, column x
                baseA[q] = ybv * G.PD + xbv;
                v0[q] = sb[cld0 ? baseA[q] + f.oldA[0] : base[q] + f.old[0]];
                v1[q] = sb[cld1 ? baseA[q] + f.oldA[1] : base[q] + f.old[1]];
            } else {
                v0[q] = sb[base[q] + f.old[0]];
                v1[q] = sb[base[q] + f.old[1]];
            }
            v0[q].y = flip_sign(v0[q].y, cld0);
            v1[q].y = flip_sign(v1[q].y, cld1);
        }
        double zr0[2] = {0.0, 0.0}, zr1[2] = {0.0, 0.0}, zi0[2] = {0.0, 0.0}, zi1[2] = {0.0, 0.0};
        for (uint32_t op = 0; op < (KS ? nk : 1u); ++op) {
            double lr0, lr1, li0, li1, ls0, ls1, ld0, ld1;
            if constexpr (KS) {
                const double* kq = kf + op * 256 + lane;
                lr0 = kq[0];
                lr1 = kq[32];
                li0 = kq[64];
                li1 = kq[96];
                ls0 = kq[128];
                ls1 = kq[160];
                ld0 = kq[192];
                ld1 = kq[224];
            } else {
                lr0 = f.lr[0];
                lr1 = f.lr[1];
                li0 = f.li[0];
                li1 = f.li[1];
                ls0 = f.ls[0];
                ls1 = f.ls[1];
                ld0 = f.ld[0];
                ld1 = f.ld[1];
            }
            // 3M form (Gauss): three real products per complex product.  Stage 1: Y = L B with
            // T1 = Lr Br, T2 = Li Bi, T3 = (Lr + Li)(Br + Bi); Yr = T1 - T2, Yi = T3 - T1 - T2
            double yr0[2], yr1[2], yi0[2], yi1[2];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                double t1a = 0.0, t1b = 0.0, t2a = 0.0, t2b = 0.0, t3a = 0.0, t3b = 0.0;
                const double s0 = v0[q].x + v0[q].y, s1 = v1[q].x + v1[q].y;
                dmma_acc(t1a, t1b, lr0, v0[q].x);
                dmma_acc(t2a, t2b, li0, v0[q].y);
                dmma_acc(t3a, t3b, ls0, s0);
                dmma_acc(t1a, t1b, lr1, v1[q].x);
                dmma_acc(t2a, t2b, li1, v1[q].y);
                dmma_acc(t3a, t3b, ls1, s1);
                yr0[q] = t1a - t2a;
                yr1[q] = t1b - t2b;
                yi0[q] = t3a - t1a - t2a;
                yi1[q] = t3b - t1b - t2b;
            }
            // stage 2: Z = Y P, P = L^dagger (B fragment of chunk j: P[2c + j][g] = conj(L[g][2c + j]));
            // U1 = Yr Pr, U2 = Yi Pi, U3 = (Yr + Yi)(Pr + Pi); Zr = U1 - U2, Zi = U3 - U1 - U2.  With
            // Pi = -Li^T the code accumulates V2 = Yi Li^T = -U2: Zr = U1 + V2, Zi = U3 - U1 + V2
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                double u1a = 0.0, u1b = 0.0, u2a = 0.0, u2b = 0.0, u3a = 0.0, u3b = 0.0;
                const double s0 = yr0[q] + yi0[q], s1 = yr1[q] + yi1[q];
                dmma_acc(u1a, u1b, yr0[q], lr0);
                dmma_acc(u2a, u2b, yi0[q], li0);
                dmma_acc(u3a, u3b, s0, ld0);
                dmma_acc(u1a, u1b, yr1[q], lr1);
                dmma_acc(u2a, u2b, yi1[q], li1);
                dmma_acc(u3a, u3b, s1, ld1);
                if constexpr (KS) {
                    zr0[q] += u1a + u2a;
                    zr1[q] += u1b + u2b;
                    zi0[q] += u3a - u1a + u2a;
                    zi1[q] += u3b - u1b + u2b;
                } else {
                    zr0[q] = u1a + u2a;
                    zr1[q] = u1b + u2b;
                    zi0[q] = u3a - u1a + u2a;
                    zi1[q] = u3b - u1b + u2b;
                }
            }
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            if (q && !two)
                break;
            if constexpr (TMAB) {
                const uint32_t xbv = base[q] >> 8, ybv = base[q] & 0xffu;
                sb[cst0 ? tma_addr(f.ostA[0], ybv, xbv) : tma_addr(f.ost[0], xbv, ybv)] = make_double2(zr0[q], flip_sign(zi0[q], cst0));
                sb[cst1 ? tma_addr(f.ostA[1], ybv, xbv) : tma_addr(f.ost[1], xbv, ybv)] = make_double2(zr1[q], flip_sign(zi1[q], cst1));
            } else if constexpr (BULK) {
                sb[cst0 ? baseA[q] + f.ostA[0] : base[q] + f.ost[0]] = make_double2(zr0[q], flip_sign(zi0[q], cst0));
                sb[cst1 ? baseA[q] + f.ostA[1] : base[q] + f.ost[1]] = make_double2(zr1[q], flip_sign(zi1[q], cst1));
            } else {
                sb[base[q] + f.ost[0]] = make_double2(zr0[q], flip_sign(zi0[q], cst0));
                sb[base[q] + f.ost[1]] = make_double2(zr1[q], flip_sign(zi1[q], cst1));
            }
        }
    };
    if (TMAB && G.tq == 4) {
        // boxes selected by bit 3 of the block position: each warp keeps one quadrant (bit 3 of the
        // block row and column: block index bits 2 and 5 of 8 x 8 blocks), 16 blocks, NW / 4 warps
        constexpr uint32_t NWQ = NC / 32 / 4;
        const uint32_t qd = warp & 3u, wi = warp >> 2;
        for (uint32_t jb = wi; jb < 16; jb += NQ * NWQ) {
            const uint32_t j1 = jb + NWQ;
            const uint32_t b0 = ((((qd >> 1) << 2) | (jb >> 2)) << 3) | ((qd & 1u) << 2) | (jb & 3u);
            const uint32_t b1 = ((((qd >> 1) << 2) | (j1 >> 2)) << 3) | ((qd & 1u) << 2) | (j1 & 3u);
            pass(b0, b1, NQ == 2 && j1 < 16);
        }
        return;
    }
    for (uint32_t b = warp; b < nblk; b += NQ * (NC / 32))
        pass(b, b + NC / 32, NQ == 2 && b + NC / 32 < nblk);
}

// k = 2 Kraus sum through its row-stacked transfer matrix S (16 x 16 complex; kernels.cpp:27-48,
// the reference's matvec<16> per block) on the FP64 tensor path: W^T = V^T S^T for 8 blocks per warp
// pass, one mma.sync m8n8k4 per (k-step ks, n-tile nt, real product).  A fragment = the blocks'
// components (lane (g, c): block g, component sf_pi[4 ks + c]), B fragment = S^T, constant per lane
// (S[sf_sigma[8 nt + g]][sf_pi[4 ks + c]]), accumulator = outputs (lane (g, c): block g, components
// sf_sigma[8 nt + 2 c + j]).  3M form: P1 = Vr Sr^T, P2 = Vi Si^T, P3 = (Vr + Vi)(Sr + Si)^T;
// Wr = P1 - P2, Wi = P3 - P1 - P2: 24 DMMA per 8 blocks (48 FMA per element, whatever the rank;
// the direct form costs 24 per element per Kraus operator).  Staged tiles keep their stored
// orientation (bulk rows); adjoint components are addressed through cadj and conjugated.
struct SfFrag {
    double sr[2][4], si[2][4];
    uint32_t ld[4], st[4];  // component offsets: direct (low 16 bits) | adjoint (high 16 bits)
    uint32_t tl, ts;        // their logical tiles, 4 bits each (adjoint flags per item)
};
template <int NS>
__device__ __forceinline__ SfFrag sform2_frag(const Geo& G, const Tabs& T, const Coef<NS>& cf) {
    SfFrag f;
    const uint32_t lane = threadIdx.x & 31u, gq = lane >> 2, cq = lane & 3u;
    f.tl = f.ts = 0;
#pragma unroll
    for (uint32_t ks = 0; ks < 4; ++ks) {
        const uint32_t ci = G.sf_pi[4 * ks + cq];
#pragma unroll
        for (uint32_t nt = 0; nt < 2; ++nt) {
            const double2 v = cf.s[G.sf_sigma[8 * nt + gq] * 16 + ci];
            f.sr[nt][ks] = v.x;
            f.si[nt][ks] = v.y;
        }
        f.ld[ks] = (uint32_t)T.cdir[ci] | ((uint32_t)T.cadj[ci] << 16);
        f.tl |= (uint32_t)T.ttr[ci] << (4 * ks);
    }
#pragma unroll
    for (uint32_t q = 0; q < 4; ++q) {
        const uint32_t co = G.sf_sigma[8 * (q >> 1) + 2 * cq + (q & 1u)];
        f.st[q] = (uint32_t)T.cdir[co] | ((uint32_t)T.cadj[co] << 16);
        f.ts |= (uint32_t)T.ttr[co] << (4 * q);
    }
    return f;
}
template <int NC>
__device__ __forceinline__ void sform2(const Geo& G, const Tabs& T, const SfFrag& f, uint64_t am, double2* sb,
                                       uint32_t warp) {
    // passes in flight per warp: one (two independent chains spill at the 128 registers of a 512-thread
    // CTA; the eight transform warps keep the FP64 pipe fed with three chains each)
    constexpr uint32_t NQ = 1;
    const uint32_t lane = threadIdx.x & 31u, gq = lane >> 2;
    uint32_t fl = 0;  // bit ks: loaded component adjoint; bit 4 + q: stored component adjoint
#pragma unroll
    for (uint32_t i = 0; i < 4; ++i) {
        fl |= (uint32_t)((am >> ((f.tl >> (4 * i)) & 15u)) & 1ull) << i;
        fl |= (uint32_t)((am >> ((f.ts >> (4 * i)) & 15u)) & 1ull) << (4 + i);
    }
    const uint32_t lbt = G.logNxb + G.logNyb, npass = ((G.grp4 ? 4u : 1u) << lbt) >> 3;
    const uint32_t lfast = G.sf_xfast ? G.logNxb : G.logNyb, fmask = (1u << lfast) - 1;
    for (uint32_t p0 = warp; p0 < npass; p0 += NQ * (NC / 32)) {
        uint32_t base[NQ], baseA[NQ];
        double vr[NQ][4], vi[NQ][4];
#pragma unroll
        for (uint32_t q = 0; q < NQ; ++q) {
            const uint32_t p = min(p0 + q * (NC / 32), npass - 1);  // a missing pass recomputes the last one
            const uint32_t b = 8 * p + gq, bq = b & ((1u << lbt) - 1);
            const uint32_t i0 = bq & fmask, i1 = bq >> lfast;
            const uint32_t xbv = T.xb[G.sf_xfast ? i0 : i1], ybv = T.yb[G.sf_xfast ? i1 : i0];
            const uint32_t slot = (b >> lbt) * G.TS;
            base[q] = slot + xbv * G.PD + (xbv >> 3) * G.s8 + ybv;
            baseA[q] = slot + ybv * G.PD + (ybv >> 3) * G.s8 + xbv;
#pragma unroll
            for (uint32_t ks = 0; ks < 4; ++ks) {
                const uint32_t adj = (fl >> ks) & 1u;
                const double2 v = sb[adj ? baseA[q] + (f.ld[ks] >> 16) : base[q] + (f.ld[ks] & 0xffffu)];
                vr[q][ks] = v.x;
                vi[q][ks] = flip_sign(v.y, adj << 31);
            }
        }
        const bool two = p0 + (NC / 32) < npass;
#pragma unroll
        for (uint32_t nt = 0; nt < 2; ++nt) {
            double p1[NQ][2], p2[NQ][2], p3[NQ][2];
#pragma unroll
            for (uint32_t q = 0; q < NQ; ++q)
                p1[q][0] = p1[q][1] = p2[q][0] = p2[q][1] = p3[q][0] = p3[q][1] = 0.0;
#pragma unroll
            for (uint32_t ks = 0; ks < 4; ++ks) {
                const double ss = f.sr[nt][ks] + f.si[nt][ks];
#pragma unroll
                for (uint32_t q = 0; q < NQ; ++q) {
                    dmma_acc(p1[q][0], p1[q][1], vr[q][ks], f.sr[nt][ks]);
                    dmma_acc(p2[q][0], p2[q][1], vi[q][ks], f.si[nt][ks]);
                    dmma_acc(p3[q][0], p3[q][1], vr[q][ks] + vi[q][ks], ss);
                }
            }
#pragma unroll
            for (uint32_t q = 0; q < NQ; ++q) {
                if (q && !two)
                    break;
#pragma unroll
                for (uint32_t j = 0; j < 2; ++j) {
                    const uint32_t o = 2 * nt + j, adj = (fl >> (4 + o)) & 1u;
                    const double wr = p1[q][j] - p2[q][j], wi = p3[q][j] - p1[q][j] - p2[q][j];
                    sb[adj ? baseA[q] + (f.st[o] >> 16) : base[q] + (f.st[o] & 0xffffu)] =
                        make_double2(wr, flip_sign(wi, adj << 31));
                }
            }
        }
    }
}

// k = 3 Kraus sums in the hermitian basis on the FP64 tensor path.  A Kraus map S is hermiticity-
// preserving, so with B = B1 + i B2 (B1 = (B + B^dagger) / 2, B2 = (B - B^dagger) / 2i, both hermitian)
// S(B) = S(B1) + i S(B2), and on the 64 real coordinates of a hermitian 8 x 8 matrix (diagonal, Re and
// Im of the upper triangle) S is one REAL 64 x 64 matrix R.  Per block: two real products R x1, R x2
// (128 FMA per element, whatever the rank) instead of the complex 64 x 64 transfer matrix (192 FMA
// per element in 3M form, kernels.cpp:39-48's matvec generalised) or the direct sum (48 per element
// per Kraus operator).  Each lane of a quad loads the 16 block elements hf_in names -- 7 mirrored
// pairs (r, c), (c, r) and 2 diagonal elements -- so the coordinates (doubled: the 1/2 is folded into
// R) form in registers:  x1 = Re B_rc + Re B_cr | Im B_rc - Im B_cr,  x2 = Im B_rc + Im B_cr |
// Re B_cr - Re B_rc.  Outputs come out as coordinate pairs (Re, Im of H_rc) of H1 = R x1 and H2 = R x2:
// W_rc = H1_rc + i H2_rc, W_cr = conj(H1_rc) + i conj(H2_rc) (n-tile 7: pairs of diagonal elements).
// 8 blocks per warp pass: 16 k-steps x 8 n-tiles x 2 products = 256 DMMA.
// TMAB: component ci of block (xb, yb) is sub-block position (x, y) = (xb | xr, yb | yc) of logical
// tile t (T.hsd[ci] = t * boxes per tile, T.hsa[ci] = xr << 4 | yc), transposed for adjoint tiles
// (stored orientation); it sits in the 8 x 8 box (x >> 3, y >> 3) of the tile (base T.cdir[slot],
// swizzle phase T.tsk[slot]) at (x & 7) * 8 + ((y & 7) ^ (((x & 7) + phi) & 7)).
template <int NC, bool TMAB = false>
__device__ __forceinline__ void hform3(const Geo& G, const Tabs& T, const uint8_t* hin, const uint8_t* hout,
                                       const double* rfr, uint64_t am, double2* sb, uint32_t warp) {
    const uint32_t lane = threadIdx.x & 31u, gq = lane >> 2, cq = lane & 3u;
    const uint32_t lbt = G.logNxb + G.logNyb, npass = ((G.grp4 ? 4u : 1u) << lbt) >> 3;
    const uint32_t logNy = G.logNyb, ymask = G.nyb - 1;
    const uint8_t* myin = hin + 16 * cq;
    auto addr = [&](uint32_t ci, uint32_t adj, uint32_t base, uint32_t baseA, uint32_t xbv, uint32_t ybv) -> uint32_t {
        if constexpr (TMAB) {
            const uint32_t xy = T.hsa[ci], xd = xbv | (xy >> 4), yd = ybv | (xy & 15u);
            const uint32_t x = adj ? yd : xd, y = adj ? xd : yd;
            const uint32_t sl = T.hsd[ci] + ((x >> 3) << (G.logS0 - 3)) + (y >> 3);
            return T.cdir[sl] + (x & 7u) * 8u + ((y & 7u) ^ (((x & 7u) + T.tsk[sl]) & 7u));
        } else {
            return adj ? baseA + T.cadj[ci] : base + T.cdir[ci];
        }
    };
    for (uint32_t p = warp; p < npass; p += NC / 32) {
        const uint32_t b = 8 * p + gq, bq = b & ((1u << lbt) - 1);
        const uint32_t xbv = T.xb[bq >> logNy], ybv = T.yb[bq & ymask];
        const uint32_t slot = (b >> lbt) * G.TS;
        const uint32_t base = slot + xbv * G.PD + (xbv >> 3) * G.s8 + ybv;
        const uint32_t baseA = slot + ybv * G.PD + (ybv >> 3) * G.s8 + xbv;
        double x1[16], x2[16];
#pragma unroll
        for (uint32_t j = 0; j < 8; ++j) {
            double2 v[2];
#pragma unroll
            for (uint32_t e = 0; e < 2; ++e) {
                const uint32_t ci = myin[2 * j + e], adj = (uint32_t)(am >> T.ttr[ci]) & 1u;
                v[e] = sb[addr(ci, adj, base, baseA, xbv, ybv)];
                v[e].y = flip_sign(v[e].y, adj << 31);
            }
            if (j < 7) {  // mirrored pair (r, c), (c, r)
                x1[2 * j] = v[0].x + v[1].x;
                x2[2 * j] = v[0].y + v[1].y;
                x1[2 * j + 1] = v[0].y - v[1].y;
                x2[2 * j + 1] = v[1].x - v[0].x;
            } else {      // two diagonal elements
                x1[14] = v[0].x;
                x2[14] = v[0].y;
                x1[15] = v[1].x;
                x2[15] = v[1].y;
            }
        }
        auto store = [&](uint32_t nt, double h1a, double h1b, double h2a, double h2b) {
            const uint32_t e0 = hout[2 * (4 * nt + cq)], e1 = hout[2 * (4 * nt + cq) + 1];
            double2 w0, w1;
            if (nt < 7) {
                w0 = make_double2(h1a - h2b, h1b + h2a);
                w1 = make_double2(h1a + h2b, h2a - h1b);
            } else {
                w0 = make_double2(h1a, h2a);
                w1 = make_double2(h1b, h2b);
            }
            const uint32_t a0 = (uint32_t)(am >> T.ttr[e0]) & 1u, a1 = (uint32_t)(am >> T.ttr[e1]) & 1u;
            sb[addr(e0, a0, base, baseA, xbv, ybv)] = make_double2(w0.x, flip_sign(w0.y, a0 << 31));
            sb[addr(e1, a1, base, baseA, xbv, ybv)] = make_double2(w1.x, flip_sign(w1.y, a1 << 31));
        };
        // two n-tiles at a time: four independent accumulator chains per warp keep the FP64 tensor
        // pipe fed (two chains left it waiting on the DMMA latency); R's fragments come from shared
        // memory (ks stride 256 doubles)
#ifndef HFORM_NTB
#define HFORM_NTB 2  // 4 (eight chains) measured 5-9% slower: profiles/r02/k3_ntb_ab.txt
#endif
        constexpr uint32_t NTB = HFORM_NTB;  // n-tiles per batch: 2 x NTB accumulator chains per warp
#pragma unroll 1
        for (uint32_t nt = 0; nt < 8; nt += NTB) {
            double acc[NTB][4];
#pragma unroll
            for (uint32_t u = 0; u < NTB; ++u)
                acc[u][0] = acc[u][1] = acc[u][2] = acc[u][3] = 0.0;
            const uint32_t f = smem_u32(rfr + nt * 32 + lane);
            // (volatile: program order bounds the live fragment registers to NTB)
#pragma unroll
            for (uint32_t ks = 0; ks < 16; ++ks) {
                double r[NTB];
#pragma unroll
                for (uint32_t u = 0; u < NTB; ++u)
                    asm volatile("ld.shared.f64 %0, [%1];" : "=d"(r[u]) : "r"(f + ks * 2048u + u * 256u));
                // (m16n8k4 with x1 / x2 as rows g / g + 8 against the shared fragment is the same
                // math in half the instructions, and measured 4-5% slower: profiles/r02/k3_m16n8k4_ab.txt)
#pragma unroll
                for (uint32_t u = 0; u < NTB; ++u) {
                    dmma_acc_v(acc[u][0], acc[u][1], x1[ks], r[u]);
                    dmma_acc_v(acc[u][2], acc[u][3], x2[ks], r[u]);
                }
            }
#pragma unroll
            for (uint32_t u = 0; u < NTB; ++u)
                store(nt + u, acc[u][0], acc[u][1], acc[u][2], acc[u][3]);
        }
    }
}

__device__ unsigned long long g_phase_cycles[8];  // diagnostics: gather phase cycles per group
template <int K, int MODE, int NS, int NC>
__global__ void __launch_bounds__(NC, 1) gather_kernel(const Geo G, const Coef<NS> cf, double2* __restrict__ st) {
    constexpr uint32_t NH = NC / 2;  // threads per group
    constexpr uint32_t S = 3;        // stages (plan_gather)
    extern __shared__ __align__(128) double2 ring[];
    __shared__ uint64_t gt[S][64];
    __shared__ uint64_t am[S][1];
    __shared__ __align__(8) uint64_t full[S];
    __shared__ Tabs T;
    const uint32_t tid = threadIdx.x, grp = tid / NH, gtid = tid % NH;
    if (tid < 32) {
        T.xdep[tid] = G.xdep[tid];
        T.xb[tid] = G.xb_tab[tid];
        T.yb[tid] = G.yb_tab[tid];
        if (tid < 8) {
            T.xs_in[tid] = G.xs_in[tid];
            T.y_in[tid] = G.y_in[tid];
        }
    }
    if (tid < 64) {
        T.cdir[tid] = G.cdir[tid];
        T.cadj[tid] = G.cadj[tid];
        T.ttr[tid] = G.ttr[tid];
        T.tsk[tid] = G.tsk[tid];
    }
    if (tid == 0)
        for (uint32_t q = 0; q < S; ++q)
            mbar_init(&full[q], 2 * NH);
    const uint64_t nItems = G.nG_items;
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint32_t NT = 1u << G.logNT, NGm = (1u << G.logNG) - 1;
    const uint32_t logT = 2 * G.logS0, P = G.S0 + 1;
    // NH is a multiple of S0^2: every element this thread moves sits at the same sub-block
    // position (i, jj) in stored order, in tiles tt = gtid / S0^2 + k * NH / S0^2
    // positions moved by this thread: npos = max(1, S0^2 / NH) sub-block positions
    // r = (gtid mod S0^2) + q * NH, each in tiles tt = tt0 + k * ttstep
    const uint32_t T2 = 1u << logT;
    const uint32_t npos = T2 > NH ? T2 / NH : 1u;
    const uint32_t tt0 = T2 > NH ? 0u : gtid >> logT, ttstep = T2 > NH ? 1u : NH >> logT;
    const uint32_t nsbm = (1u << (2 * G.log_nsb_side)) - 1;
    const uint32_t barid = 1 + grp;
    auto gbar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NH) : "memory"); };

    auto item_of = [&](uint64_t j) { return sweep_item(G, nItems, j); };
    // global offsets (within a tile) of this thread's q-th sub-block position, direct / adjoint,
    // and its logical staging slot (direct / adjoint placement)
    auto offsets = [&](uint64_t item, uint32_t q, uint32_t& od, uint32_t& oa, uint32_t& sm_d, uint32_t& sm_a) {
        const uint32_t r = (gtid & (T2 - 1)) + q * NH, i0 = r >> G.logS0, j0 = r & (G.S0 - 1);
        const uint32_t sb = (uint32_t)(item & nsbm);
        const uint32_t x0 = G.sdep[sb >> G.log_nsb_side], y0 = G.sdep[sb & ((1u << G.log_nsb_side) - 1)];
        od = ((x0 | T.xdep[i0]) << G.logM) + (y0 | T.xdep[j0]);
        oa = ((y0 | T.xdep[i0]) << G.logM) + (x0 | T.xdep[j0]);
        sm_d = i0 * P + j0;
        sm_a = j0 * P + i0;
    };
    // this group loads item j into stage j % S (tile table, adjoint mask, copies, arrivals)
    auto load = [&](uint64_t j) {
        const uint32_t s = (uint32_t)(j % S);
        const uint64_t u = item_of(j) >> (2 * G.log_nsb_side);
        if (gtid < NT) {
            uint64_t tbi, tbj;
            unit_decode(G, u, true, tbi, tbj);
            const uint64_t tr = ins_bits(tbi, gtid >> G.logNG, G.gr_pos, G.g);
            const uint64_t tc = ins_bits(tbj, gtid & NGm, G.gr_pos, G.g);
            uint64_t ent = tile_entry(G, tr, tc);
            if (MODE == M_MONO && !((G.active >> gtid) & 1ull))
                ent |= F_SKIP;
            gt[s][gtid] = ent;
        }
        gbar();
        if (gtid < 32) {
            unsigned long long m = 0;
            for (uint32_t t = gtid; t < NT; t += 32)
                m |= (unsigned long long)((gt[s][t] & F_ADJ) != 0) << t;
            for (int o = 16; o; o >>= 1)
                m |= __shfl_xor_sync(0xffffffffu, m, o);
            if (gtid == 0)
                am[s][0] = m;
        }
        const uint32_t base = smem_u32(ring) + s * G.stage_elems * 16u;
        for (uint32_t q = 0; q < npos; ++q) {
            uint32_t od, oa, sm_d, sm_a;
            offsets(item_of(j), q, od, oa, sm_d, sm_a);
            for (uint32_t tt = tt0; tt < NT && !(G.dbg & 2u); tt += ttstep) {
                const uint64_t ent = gt[s][tt];
                if (ent & F_SKIP)
                    continue;
                const bool adj = (ent & F_ADJ) != 0;
                const uint64_t g = ((ent & F_MASK) << (2 * G.logM)) + (adj ? oa : od);
                cp_async16(base + (tt * G.TS + T.tsk[tt] + (adj ? sm_a : sm_d)) * 16u,
                           tile_base(G, ent, st) + g);
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        mbar_arrive(&full[s]);
    };
    __syncthreads();
    DmmaFrag fr;
    if constexpr (K == 3 && MODE == M_DIRECT)
        fr = dmma_frag<3>(G, T, cf);
    for (uint64_t j = 0; j < S && j < nlocal; ++j)  // item j is loaded by group (j + 1) & 1
        if (((j + 1) & 1) == grp)
            load(j);
    const bool prof = (G.dbg & 16u) && gtid == 0;  // phase timing (diagnostics): wait / transform / write-back / load
    long long ph[4] = {0, 0, 0, 0};
    for (uint64_t i = grp; i < nlocal; i += 2) {
        const uint32_t s = (uint32_t)(i % S);
        long long t0 = prof ? clock64() : 0;
        mbar_wait(&full[s], (uint32_t)((i / S) & 1));
        long long t1 = prof ? clock64() : 0;
        double2* sb = ring + (size_t)s * G.stage_elems;
        if (!(G.dbg & 1u)) {
            if constexpr (K == 3 && MODE == M_DIRECT)
                dmma_direct3<NH>(G, T, fr, am[s][0], sb, gtid >> 5);
            else
                pipe_compute<K, MODE, NS, NH>(G, T, cf, am[s], 1, sb, 0, (int)gtid, barid);
        }
        gbar();
        long long t2 = prof ? clock64() : 0;
        // write back along stored rows (adjoint components are already in stored, conjugated form)
        for (uint32_t q = 0; q < npos; ++q) {
            uint32_t od, oa, sm_d, sm_a;
            offsets(item_of(i), q, od, oa, sm_d, sm_a);
            for (uint32_t tt = tt0; tt < NT && !(G.dbg & 4u); tt += ttstep) {
                const uint64_t ent = gt[s][tt];
                if (ent & (F_SKIP | F_NOSTORE))
                    continue;
                const bool adj = (ent & F_ADJ) != 0;
                G.out[((ent & F_MASK) << (2 * G.logM)) + (adj ? oa : od)] = sb[tt * G.TS + T.tsk[tt] + (adj ? sm_a : sm_d)];
            }
        }
        gbar();
        long long t3 = prof ? clock64() : 0;
        if (i + S < nlocal && (G.dbg & DBG_POISON)) {  // diagnostics: NaN until the copies of item i + S land
            poison_stage(sb, G.stage_elems, gtid, NH);
            gbar();
        }
        if (i + S < nlocal)
            load(i + S);
        if (prof) {
            const long long t4 = clock64();
            ph[0] += t1 - t0;
            ph[1] += t2 - t1;
            ph[2] += t3 - t2;
            ph[3] += t4 - t3;
        }
    }
    if (prof)
        for (int q = 0; q < 4; ++q)
            atomicAdd(&g_phase_cycles[grp * 4 + q], (unsigned long long)ph[q]);
    cp_async_wait<0>();
}

// Warp-specialised gather for the k = 3 tensor-core transform: 8 transform warps and 16 copy warps
// (768 threads).  The copy warps write back item i as soon as the transform warps release its stage
// (`done`), then load item i + 3 into it (`full`, cp.async tracked by the mbarrier); the transform
// warps only wait for data and run DMMA.  The 16 copy warps keep twice the memory-instruction
// parallelism of a ping-pong group, and the transform never waits for its own write-back or loads.
// (Register-staged loads in place of cp.async were 1.6x slower here.)
// One k = 1 step of a grid program on the staged logical tiles (MODE == M_PROG in gather_ws_kernel):
// quads of logical tiles (R, C), (R, C | e), (R | e, C), (R | e, C | e) at every staged position,
// e = 2^l for the step's grid bit l; adjoint tiles are staged transposed and conjugated on the fly.
template <uint32_t NCW, int NS, bool TMAB = false>
__device__ __forceinline__ void grid_prog_step(const Geo& G, const Tabs& T, const Coef<NS>& cf, uint32_t p,
                                               uint32_t p1, uint64_t am, double2* sb, uint32_t tid) {
    // steps [p, p1) act on one grid qubit: its chain runs on each quad in registers
    // TMA boxes: tiles in stored orientation (adjoint ones transposed), 8 x 8 boxes; for grid
    // programs every box has phase 0 and box `slot` sits at slot * 64 (plan_gather), so the
    // address is pure arithmetic (no table lookups)
    const uint32_t nbx = G.S0 >> 3, lbpt = 2 * (G.logS0 - 3);
    const uint32_t g = G.g, NG = 1u << g, e = 1u << cf.pbit[p], lo = e - 1;
    const uint32_t S0 = G.S0, P = S0 + 1, npos = S0 * S0, lp = 2 * G.logS0;
    const uint32_t nq = (NG / 2) * (NG / 2) * npos;
    for (uint32_t q = tid; q < nq; q += NCW) {
        const uint32_t tq = q >> lp, pos = q & (npos - 1), i = pos >> G.logS0, j = pos & (S0 - 1);
        const uint32_t rr = tq >> (g - 1), cc = tq & ((NG >> 1) - 1);
        const uint32_t R0 = ((rr & ~lo) << 1) | (rr & lo), C0 = ((cc & ~lo) << 1) | (cc & lo);
        const uint32_t t0 = R0 * NG + C0, t1 = R0 * NG + (C0 | e), t2 = (R0 | e) * NG + C0, t3 = t2 + e;
        const uint32_t f0 = (uint32_t)((am >> t0) & 1ull) << 31, f1 = (uint32_t)((am >> t1) & 1ull) << 31;
        const uint32_t f2 = (uint32_t)((am >> t2) & 1ull) << 31, f3 = (uint32_t)((am >> t3) & 1ull) << 31;
        uint32_t a0, a1, a2, a3;
        if constexpr (TMAB) {
            // one position, four tiles: the direct and the transposed in-tile offsets once (the
            // swizzle term (x ^ y) & 7 is symmetric), the tile's slot base and orientation per tile
            const uint32_t sw = (i ^ j) & 7u;
            const uint32_t ad = (((i >> 3) * nbx + (j >> 3)) << 6) + (i & 7u) * 8u + sw;
            const uint32_t aa = (((j >> 3) * nbx + (i >> 3)) << 6) + (j & 7u) * 8u + sw;
            a0 = (t0 << (lbpt + 6)) + (f0 ? aa : ad);
            a1 = (t1 << (lbpt + 6)) + (f1 ? aa : ad);
            a2 = (t2 << (lbpt + 6)) + (f2 ? aa : ad);
            a3 = (t3 << (lbpt + 6)) + (f3 ? aa : ad);
        } else {
            const uint32_t off = i * P + j;
            a0 = t0 * G.TS + T.tsk[t0] + off;
            a1 = t1 * G.TS + T.tsk[t1] + off;
            a2 = t2 * G.TS + T.tsk[t2] + off;
            a3 = t3 * G.TS + T.tsk[t3] + off;
        }
        double2 v0 = sb[a0], v1 = sb[a1], v2 = sb[a2], v3 = sb[a3];
        v0.y = flip_sign(v0.y, f0);
        v1.y = flip_sign(v1.y, f1);
        v2.y = flip_sign(v2.y, f2);
        v3.y = flip_sign(v3.y, f3);
        for (uint32_t pp = p; pp < p1; ++pp)
            prog_quad(cf.pkind[pp], cf.s + 16 * pp, v0, v1, v2, v3);
        v0.y = flip_sign(v0.y, f0);
        v1.y = flip_sign(v1.y, f1);
        v2.y = flip_sign(v2.y, f2);
        v3.y = flip_sign(v3.y, f3);
        sb[a0] = v0;
        sb[a1] = v1;
        sb[a2] = v2;
        sb[a3] = v3;
    }
}

// grid_prog_step for TMA boxes when an item holds exactly two quads per transform thread and qubit
// (3 grid qubits: 16 tile quads x 64 positions; 2 grid qubits: 4 x 256; NCW = 512).  A thread's
// position -- hence its direct / transposed in-box offsets `ad` / `aa` -- is the same for every
// item, qubit and quad, and the two tile quads of each pass are the same for every item: both are
// computed once per kernel (gather_ws_kernel), per item only the adjoint flags are looked up.  Both
// quads are loaded before either chain runs (the compiler cannot hoist shared loads over shared
// stores itself), and the adjoint flag rides in bit 31 of each address.
template <int NS, bool PLAIN>
__device__ __forceinline__ void grid_prog_step2_(const Geo& G, const Coef<NS>& cf, uint32_t p, uint32_t p1, uint64_t am,
                                                 double2* sb, uint32_t t0ab, uint32_t ad, uint32_t dlt) {
    // t0ab: the (0, 0) logical tile of this thread's two quads for this pass (bits 0-7, 8-15);
    // ad: direct in-box offset of its position, dlt: transposed minus direct offset
    const uint32_t g = G.g, sh = 2 * G.logS0, l = cf.pbit[p];  // box slots per tile << 6 == S0^2
    const uint32_t o1 = 1u << l, o2 = o1 << g, o3 = o1 + o2;
    uint32_t a[8];
#pragma unroll
    for (uint32_t h = 0; h < 2; ++h) {
        const uint32_t t0 = (t0ab >> (8 * h)) & 0xffu;
        const uint32_t base = (t0 << sh) + ad;
        if constexpr (PLAIN) {  // every tile of the unit in stored orientation: no transposed offsets, no flips
            a[4 * h + 0] = base;
            a[4 * h + 1] = base + (o1 << sh);
            a[4 * h + 2] = base + (o2 << sh);
            a[4 * h + 3] = base + (o3 << sh);
        } else {
            const uint64_t amt = am >> t0;  // the quad's adjoint flags at bit offsets 0, o1, o2, o3 (<= 36)
            const uint32_t f0 = (uint32_t)amt & 1u, f1 = (uint32_t)(amt >> o1) & 1u, f2 = (uint32_t)(amt >> o2) & 1u,
                           f3 = (uint32_t)(amt >> o3) & 1u;
            a[4 * h + 0] = (base + f0 * dlt) | (f0 << 31);
            a[4 * h + 1] = (base + (o1 << sh) + f1 * dlt) | (f1 << 31);
            a[4 * h + 2] = (base + (o2 << sh) + f2 * dlt) | (f2 << 31);
            a[4 * h + 3] = (base + (o3 << sh) + f3 * dlt) | (f3 << 31);
        }
    }
    double2 va[4], vb[4];
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
        va[c] = sb[a[c] & 0x7fffffffu];
        vb[c] = sb[a[4 + c] & 0x7fffffffu];
    }
    if constexpr (!PLAIN) {
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) {
            va[c].y = flip_sign(va[c].y, a[c] & 0x80000000u);
            vb[c].y = flip_sign(vb[c].y, a[4 + c] & 0x80000000u);
        }
    }
    for (uint32_t pp = p; pp < p1; ++pp)
        prog_quad2(cf.pkind[pp], cf.s + 16 * pp, va, vb);
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
        if constexpr (!PLAIN) {
            va[c].y = flip_sign(va[c].y, a[c] & 0x80000000u);
            vb[c].y = flip_sign(vb[c].y, a[4 + c] & 0x80000000u);
        }
        sb[a[c] & 0x7fffffffu] = va[c];
        sb[a[4 + c] & 0x7fffffffu] = vb[c];
    }
}
template <int NS>
__device__ __forceinline__ void grid_prog_step2(const Geo& G, const Coef<NS>& cf, uint32_t p, uint32_t p1, uint64_t am,
                                                double2* sb, uint32_t t0ab, uint32_t ad, uint32_t dlt) {
    if (am == 0)  // off-diagonal units away from the diagonal: every logical tile is a stored tile
        grid_prog_step2_<NS, true>(G, cf, p, p1, am, sb, t0ab, ad, dlt);
    else
        grid_prog_step2_<NS, false>(G, cf, p, p1, am, sb, t0ab, ad, dlt);
}

// Two passes of a grid program in one shared-memory round trip (as pipe_compute's paired in-tile
// passes): lanes l and l ^ 16 hold, at one staged position, the four quads of the first qubit (local
// index la) that make up one 4 x 4 block of logical tiles over the qubits (la, lb) -- this lane the
// two with tile-row bit lb = its role.  After the first chains role 0 keeps the halves with row bit
// la = 0 and gets the partner's, role 1 those with row bit la = 1: two quads of the second qubit per
// lane.  tA / tB: the (0, 0) tiles of the lane's two quads in the first / second pass.
template <int NS, bool PLAIN>
__device__ __forceinline__ void grid_prog_pair2_(const Geo& G, const Coef<NS>& cf, uint32_t p, uint32_t p1, uint32_t p2,
                                                 uint64_t am, double2* sb, uint32_t tA, uint32_t tB, uint32_t ad,
                                                 uint32_t dlt, bool r1) {
    const uint32_t g = G.g, sh = 2 * G.logS0;
    auto addrs = [&](uint32_t t0ab, uint32_t l, uint32_t (&a)[8]) {
        const uint32_t o1 = 1u << l, o2 = o1 << g, o3 = o1 + o2;
#pragma unroll
        for (uint32_t h = 0; h < 2; ++h) {
            const uint32_t t0 = (t0ab >> (8 * h)) & 0xffu;
            const uint32_t base = (t0 << sh) + ad;
            if constexpr (PLAIN) {  // every tile of the unit in stored orientation: no transposed offsets, no flips
                a[4 * h + 0] = base;
                a[4 * h + 1] = base + (o1 << sh);
                a[4 * h + 2] = base + (o2 << sh);
                a[4 * h + 3] = base + (o3 << sh);
            } else {
                const uint64_t amt = am >> t0;
                const uint32_t f0 = (uint32_t)amt & 1u, f1 = (uint32_t)(amt >> o1) & 1u, f2 = (uint32_t)(amt >> o2) & 1u,
                               f3 = (uint32_t)(amt >> o3) & 1u;
                a[4 * h + 0] = (base + f0 * dlt) | (f0 << 31);
                a[4 * h + 1] = (base + (o1 << sh) + f1 * dlt) | (f1 << 31);
                a[4 * h + 2] = (base + (o2 << sh) + f2 * dlt) | (f2 << 31);
                a[4 * h + 3] = (base + (o3 << sh) + f3 * dlt) | (f3 << 31);
            }
        }
    };
    uint32_t a[8];
    addrs(tA, cf.pbit[p], a);
    double2 va[4], vb[4];
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
        va[c] = sb[a[c] & 0x7fffffffu];
        vb[c] = sb[a[4 + c] & 0x7fffffffu];
    }
    if constexpr (!PLAIN) {
#pragma unroll
        for (uint32_t c = 0; c < 4; ++c) {
            va[c].y = flip_sign(va[c].y, a[c] & 0x80000000u);
            vb[c].y = flip_sign(vb[c].y, a[4 + c] & 0x80000000u);
        }
    }
    for (uint32_t pp = p; pp < p1; ++pp)
        prog_quad2(cf.pkind[pp], cf.s + 16 * pp, va, vb);
    auto xch = [&](double2& e0, double2& e2) {  // role 0 sends e2 and keeps e0, role 1 the other way round
        double2 snd = r1 ? e0 : e2;
        snd.x = __shfl_xor_sync(0xffffffffu, snd.x, 16);
        snd.y = __shfl_xor_sync(0xffffffffu, snd.y, 16);
        if (r1)
            e0 = snd;
        else
            e2 = snd;
    };
    xch(va[0], va[2]);
    xch(vb[0], vb[2]);
    xch(va[1], va[3]);
    xch(vb[1], vb[3]);
    double2 wa[4] = {va[0], vb[0], va[2], vb[2]}, wb[4] = {va[1], vb[1], va[3], vb[3]};
    for (uint32_t pp = p1; pp < p2; ++pp)
        prog_quad2(cf.pkind[pp], cf.s + 16 * pp, wa, wb);
    addrs(tB, cf.pbit[p1], a);
#pragma unroll
    for (uint32_t c = 0; c < 4; ++c) {
        if constexpr (!PLAIN) {
            wa[c].y = flip_sign(wa[c].y, a[c] & 0x80000000u);
            wb[c].y = flip_sign(wb[c].y, a[4 + c] & 0x80000000u);
        }
        sb[a[c] & 0x7fffffffu] = wa[c];
        sb[a[4 + c] & 0x7fffffffu] = wb[c];
    }
}
template <int NS>
__device__ __forceinline__ void grid_prog_pair2(const Geo& G, const Coef<NS>& cf, uint32_t p, uint32_t p1, uint32_t p2,
                                                uint64_t am, double2* sb, uint32_t tA, uint32_t tB, uint32_t ad,
                                                uint32_t dlt, bool r1) {
    if (am == 0)  // off-diagonal units away from the diagonal: every logical tile is a stored tile
        grid_prog_pair2_<NS, true>(G, cf, p, p1, p2, am, sb, tA, tB, ad, dlt, r1);
    else
        grid_prog_pair2_<NS, false>(G, cf, p, p1, p2, am, sb, tA, tB, ad, dlt, r1);
}

// BULK (G.bulk): sub-block rows are contiguous runs of S0 >= 16 elements; every tile is staged in its
// stored orientation (pitch S0 + 1) by one cp.async.bulk per row (256 / 512 B, completing on the
// stage's `full` mbarrier) and written back by one bulk store per row -- no per-element copy
// instructions.  Adjoint components are addressed through cadj (transposed offsets); the bank
// groups are the same as in the logical layout since the pitch is 1 mod 8.
// TMAB (G.tma, with BULK): items of 8 x 8 sub-block boxes (g = 3, or g = 2 with its in-tile target
// at bit 4: 128-B rows, too short for row copies) move as 2-D tensor-map copies (one 1 KiB box per
// tile and box position), SWIZZLE_128B, each box at a 128-B phase of its own (host search) so the
// DMMA lane patterns spread over the bank groups; same two-copy-group schedule as BULK.
// KSUM: the k = 2 Kraus-sum variant (own instantiation, so the unitary kernels keep their registers)
// SF (MODE == M_SF2): the S-form transform; 8 transform warps and 8 copy warps (512 threads, 128
// registers: the per-lane S fragments stay in registers).  With 16-row sub-blocks (two grid targets)
// the copy side issues 512 bulk row copies per item: 2 copy warps streamed 4.2 TB/s, 8 copy warps
// 6.2 TB/s (n = 16, copies alone); transform alone 8.8 ms (profiles/r02_kraus_sform.txt).
// NARROW (bulk staging): 8 transform warps and 8 copy warps (512 threads, 128 registers) instead of
// 16 + 8 (768 threads, 80 registers)
template <int K, int NS, int MODE = M_DIRECT, bool BULK = false, bool TMAB = false, bool KSUM = false,
          bool NARROW = false>
__global__ void __launch_bounds__((MODE == M_SF2 || MODE == M_SF3 || NARROW) ? 512 : 768, 1)
    gather_ws_kernel(const Geo G, const Coef<NS> cf, double2* __restrict__ st, const __grid_constant__ CUtensorMap tin,
                     const __grid_constant__ CUtensorMap tout) {
    // bulk rows need few copy instructions: 16 transform warps and 8 copy warps (else 8 and 16)
    constexpr bool SF = MODE == M_SF2, SF3 = MODE == M_SF3;
    static_assert(!(SF || SF3) || BULK, "the S-form transforms run on bulk-row staging");
    static_assert(!NARROW || BULK, "the narrow layout is for bulk staging");
    // SF3: two ring stages (the 64 KiB transfer matrix takes the third's shared memory; the op is
    // bound by the FP64 pipe, twice the copy time, so two stages still hide the copies)
    constexpr uint32_t NCW = (SF || SF3 || NARROW) ? 256 : BULK ? 512 : 256, NMW = (SF || SF3) ? 256 : BULK ? 256 : 512,
                       S = SF3 ? 2 : 3;
    // tile tables by item % TSL, built S items ahead (BULK: by two copy groups that may be one item
    // apart, hence two more slots)
    constexpr uint32_t TSL = BULK ? S + 3 : S + 1;
    extern __shared__ __align__(128) double2 ring_raw[];
    // TMA boxes: stage bases 1 KiB aligned (the swizzle phase follows absolute address bits 7-9)
    double2* const ring = TMAB ? ring_raw + ((1024u - (smem_u32(ring_raw) & 1023u)) & 1023u) / 16u : ring_raw;
    __shared__ uint64_t gt[TSL][64];
    __shared__ uint64_t am[TSL][1];
    __shared__ uint32_t mir[TSL];     // BULK: the item has mirrored tiles (diagonal unit, a > b)
    __shared__ __align__(8) uint64_t full[S], done[S];
    __shared__ Tabs T;
    const uint32_t tid = threadIdx.x;
    if (tid < 32) {
        T.xdep[tid] = G.xdep[tid];
        T.xb[tid] = G.xb_tab[tid];
        T.yb[tid] = G.yb_tab[tid];
        if (tid < 8) {
            T.xs_in[tid] = G.xs_in[tid];
            T.y_in[tid] = G.y_in[tid];
        }
    }
    if (tid < 64) {
        T.cdir[tid] = G.cdir[tid];
        T.cadj[tid] = G.cadj[tid];
        T.ttr[tid] = G.ttr[tid];
        T.tsk[tid] = G.tsk[tid];
        if constexpr (MODE == M_SF3 && TMAB) {
            T.hsd[tid] = G.hsd[tid];
            T.hsa[tid] = G.hsa[tid];
        }
    }
    if (tid == 0)
        for (uint32_t q = 0; q < S; ++q) {
            mbar_init(&full[q], BULK ? NMW : 2 * NMW);  // BULK: one copy group (NMW / 2) loads an item
            mbar_init(&done[q], NCW);
        }
    const uint64_t nItems = G.nG_items;
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item_of = [&](uint64_t j) { return sweep_item(G, nItems, j); };
    __syncthreads();
    // register rebalancing between the warp groups (768-thread layouts compile at 80 registers):
    // the copy warps (2 warp groups) release 16 per thread to 64, the DMMA transform warps (4 warp
    // groups) take 8 more to 88 -- setmaxnreg.inc waits until the CTA's own released registers
    // cover it, so the exchange must balance within the CTA (an unbalanced 96 / 64 never returns)
#ifdef HS_NO_REBAL
    constexpr bool REBAL = false;
#else
    constexpr bool REBAL = !(SF || SF3 || NARROW) && BULK && (MODE == M_DIRECT || (MODE == M_PROG && TMAB));
#endif
    if (tid < NCW) {
        if constexpr (REBAL)
            asm volatile("setmaxnreg.inc.sync.aligned.u32 88;" ::: "memory");
        // ---- transform warps
        DmmaFrag fr;
        if constexpr (MODE == M_DIRECT)
            fr = dmma_frag<K, NS, BULK, TMAB>(G, T, cf);
        SfFrag sf;
        if constexpr (SF)
            sf = sform2_frag(G, T, cf);
        double* sfr = nullptr;
        __shared__ uint8_t hin[64], hout[64];
        if constexpr (SF3) {  // R's fragments into shared memory, after the ring; the element tables
            sfr = reinterpret_cast<double*>(ring + (size_t)S * G.stage_elems);
            for (uint32_t i = tid; i < 4096u; i += NCW)
                sfr[i] = G.sf3[i];
            if (tid < 64) {
                hin[tid] = G.hf_in[tid];
                hout[tid] = G.hf_out[tid];
            }
            asm volatile("bar.sync 2, %0;" ::"n"(NCW) : "memory");  // transform warps only
        }
        double* kf = nullptr;
        if constexpr (KSUM) {
            // Kraus sum: every operator's per-lane fragment values, [a][8][lane] (8 KiB)
            __shared__ double kfrag[4 * 8 * 32];
            kf = kfrag;
            if (cf.nk > 1 && tid < 32) {
                const uint32_t gq = tid >> 2, cq = tid & 3;
                for (uint32_t a = 0; a < cf.nk; ++a)
                    for (int j = 0; j < 2; ++j) {
                        const uint32_t c8 = 2 * cq + j;
                        double2 l;
                        if constexpr (K == 3)
                            l = cf.s[64 * a + gq * 8 + c8];
                        else
                            l = (gq >> 2) == (c8 >> 2) ? cf.s[16 * a + (gq & 3) * 4 + (c8 & 3)] : make_double2(0.0, 0.0);
                        kfrag[a * 256 + (0 + j) * 32 + tid] = l.x;
                        kfrag[a * 256 + (2 + j) * 32 + tid] = l.y;
                        kfrag[a * 256 + (4 + j) * 32 + tid] = l.x + l.y;
                        kfrag[a * 256 + (6 + j) * 32 + tid] = l.x - l.y;
                    }
            }
            asm volatile("bar.sync 2, %0;" ::"n"(NCW) : "memory");  // transform warps only
        }
        // grid programs on TMA boxes: this thread's position and its in-box offsets (direct / transposed;
        // the swizzle term (x ^ y) & 7 is symmetric), fixed for the whole kernel (grid_prog_step2)
        uint32_t pg_ad = 0, pg_dlt = 0, pg_t[3] = {0, 0, 0}, pg_end[3] = {0, 0, 0}, pg_tA = 0, pg_tB = 0, pg_half = 0;
        bool pg_two = false, pg_pair = false;
        if constexpr (MODE == M_PROG && TMAB) {
            // Paired passes (grid_prog_pair2; bit 15: off): lane bits 0-3 and the low warp bits give the
            // position, lane bit 4 the role, the other warp bits the 4 x 4 tile block (3 grid qubits: 4 per
            // position); the same bits select the two quads of an unpaired pass.
            const uint32_t nbx = G.S0 >> 3, lp = 2 * G.logS0;
            pg_pair = !(G.dbg & 32768u) && (lp == 6 || lp == 8) && NCW == 512;
            const uint32_t wlo = (tid >> 5) & ((1u << (lp - 4)) - 1);
            const uint32_t pos = pg_pair ? (tid & 15u) | (wlo << 4) : tid & ((1u << lp) - 1);
            const uint32_t role = (tid >> 4) & 1u, beta = (tid >> 5) >> (lp - 4);
            const uint32_t tq0 = pg_pair ? (beta << 1) | role : tid >> lp;
            pg_half = (pos >> (lp - 1)) & 1u;
            const uint32_t pi = pos >> G.logS0, pj = pos & (G.S0 - 1);
            const uint32_t sw = (pi ^ pj) & 7u;
            pg_ad = (((pi >> 3) * nbx + (pj >> 3)) << 6) + (pi & 7u) * 8u + sw;
            pg_dlt = (((pj >> 3) * nbx + (pi >> 3)) << 6) + (pj & 7u) * 8u + sw - pg_ad;
            // passes (one per qubit: its steps are consecutive), at most three; per pass the (0, 0)
            // tiles of the thread's two quads
            uint32_t p = 0;
#pragma unroll
            for (int np = 0; np < 3; ++np)
                if (p < cf.nsteps) {
                    uint32_t p1 = p + 1;
                    while (p1 < cf.nsteps && cf.pbit[p1] == cf.pbit[p])
                        ++p1;
                    const uint32_t lo = (1u << cf.pbit[p]) - 1, hm = (1u << (G.g - 1)) - 1;
                    uint32_t t0ab = 0;
#pragma unroll
                    for (uint32_t h = 0; h < 2; ++h) {
                        const uint32_t tq = tq0 + h * (NCW >> lp);
                        const uint32_t rr = tq >> (G.g - 1), cc = tq & hm;
                        const uint32_t R0 = ((rr & ~lo) << 1) | (rr & lo), C0 = ((cc & ~lo) << 1) | (cc & lo);
                        t0ab |= ((R0 << G.g) | C0) << (8 * h);
                    }
                    pg_t[np] = t0ab;
                    pg_end[np] = p1;
                    p = p1;
                }
            // bit 11: the one-quad loop
            pg_two = p >= cf.nsteps && ((1u << (2 * G.g - 2)) << lp) == 2 * NCW && !(G.dbg & 2048u);
            pg_pair = pg_pair && pg_two && pg_end[1] && (G.g == 2 || G.g == 3);
            if (pg_pair) {
                const uint32_t la = cf.pbit[0], lb = cf.pbit[pg_end[0]], g = G.g;
                uint32_t R0 = 0, C0 = 0;
                if (g == 3) {  // the block: the row / column bit of the third qubit
                    const uint32_t f = 3u - la - lb;
                    R0 = (beta >> 1) << f;
                    C0 = (beta & 1u) << f;
                }
                const uint32_t a0 = ((R0 | (role << lb)) << g) | C0, b0 = ((R0 | (role << la)) << g) | C0;
                pg_tA = a0 | ((a0 + (1u << lb)) << 8);
                pg_tB = b0 | ((b0 + (1u << la)) << 8);
            }
        }
        for (uint64_t i = 0; i < nlocal; ++i) {
            const uint32_t s = (uint32_t)(i % S);
            mbar_wait(&full[s], (uint32_t)((i / S) & 1));
            double2* sb = ring + (size_t)s * G.stage_elems;
            if constexpr (SF) {
                if (!(G.dbg & 1u))
                    sform2<NCW>(G, T, sf, am[i % TSL][0], sb, tid >> 5);
            } else if constexpr (SF3) {
                if (!(G.dbg & 1u))
                    hform3<NCW, TMAB>(G, T, hin, hout, sfr, am[i % TSL][0], sb, tid >> 5);
            } else if constexpr (MODE == M_DIRECT) {
                if constexpr (KSUM) {
                    if (!(G.dbg & 1u))
                        dmma_direct3<NCW, K, BULK, TMAB, true, NARROW>(G, T, fr, am[i % TSL][0], sb, tid >> 5, kf, cf.nk);
                } else if (!(G.dbg & 1u)) {
                    dmma_direct3<NCW, K, BULK, TMAB, false, NARROW>(G, T, fr, am[i % TSL][0], sb, tid >> 5);
                }
            } else {
                if (TMAB && pg_two) {
                    // Steps never couple staged positions, and a thread keeps its position: the warps
                    // holding the lower and the upper half of the positions synchronise separately
                    // between passes (named barriers 5 / 6) and drift apart, one half's shared-memory
                    // phase over the other's FP64 chains; after the last pass the stage's `done`
                    // mbarrier is the only synchronisation.  Bit 13: one barrier over all transform
                    // warps after every pass.
                    const uint32_t half = pg_half;
                    uint32_t p = 0;
                    if (pg_pair) {
                        grid_prog_pair2<NS>(G, cf, 0, pg_end[0], pg_end[1], am[i % TSL][0], sb, pg_tA, pg_tB, pg_ad, pg_dlt,
                                            (tid & 16u) != 0);
                        p = pg_end[1];
                        if (p < cf.nsteps) {
                            asm volatile("bar.sync %0, %1;" ::"r"(5 + half), "n"(NCW / 2) : "memory");
                            grid_prog_step2<NS>(G, cf, p, pg_end[2], am[i % TSL][0], sb, pg_t[2], pg_ad, pg_dlt);
                            p = pg_end[2];
                        }
                    }
#pragma unroll
                    for (int ps = 0; ps < 3; ++ps) {
                        if (p < cf.nsteps) {
                            grid_prog_step2<NS>(G, cf, p, pg_end[ps], am[i % TSL][0], sb, pg_t[ps], pg_ad, pg_dlt);
                            p = pg_end[ps];
                            if (G.dbg & 8192u)
                                asm volatile("bar.sync 2, %0;" ::"n"(NCW) : "memory");  // transform warps only
                            else if (p < cf.nsteps)
                                asm volatile("bar.sync %0, %1;" ::"r"(5 + half), "n"(NCW / 2) : "memory");
                        }
                    }
                } else {
                    for (uint32_t p = 0; p < cf.nsteps;) {  // one pass per qubit (its steps are consecutive)
                        uint32_t p1 = p + 1;
                        while (p1 < cf.nsteps && cf.pbit[p1] == cf.pbit[p])
                            ++p1;
                        grid_prog_step<NCW, NS, TMAB>(G, T, cf, p, p1, am[i % TSL][0], sb, tid);
                        asm volatile("bar.sync 2, %0;" ::"n"(NCW) : "memory");  // transform warps only
                        p = p1;
                    }
                }
            }
            if constexpr (BULK)
                fence_async_smem();  // the bulk stores (async proxy) read what these threads wrote
            mbar_arrive(&done[s]);
        }
        return;
    }
    // ---- copy warps
    if constexpr (REBAL)
        asm volatile("setmaxnreg.dec.sync.aligned.u32 64;" ::: "memory");
    const uint32_t mtid = tid - NCW;
    const uint32_t NT = 1u << G.logNT, NGm = (1u << G.logNG) - 1;
    const uint32_t logT = 2 * G.logS0, P = G.S0 + 1;
    const uint32_t T2 = 1u << logT;
    const uint32_t npos = T2 > NMW ? T2 / NMW : 1u;
    const uint32_t tt0 = T2 > NMW ? 0u : mtid >> logT, ttstep = T2 > NMW ? 1u : NMW >> logT;
    const uint32_t nsbm = (1u << (2 * G.log_nsb_side)) - 1;
    const bool fast = npos == 1 && (NT << logT) == 8 * NMW;  // every thread moves 8 tiles at one position
    const bool fast2 = npos == 2 && NT == 4;                  // or 4 tiles at two positions (whole-tile units)
    auto mbar_sync = [&]() { asm volatile("bar.sync 1, %0;" ::"n"(NMW) : "memory"); };
    auto offsets = [&](uint64_t item, uint32_t q, uint32_t& od, uint32_t& oa, uint32_t& sm_d, uint32_t& sm_a) {
        const uint32_t r = (mtid & (T2 - 1)) + q * NMW, i0 = r >> G.logS0, j0 = r & (G.S0 - 1);
        const uint32_t sb = (uint32_t)(item & nsbm);
        const uint32_t x0 = G.sdep[sb >> G.log_nsb_side], y0 = G.sdep[sb & ((1u << G.log_nsb_side) - 1)];
        od = ((x0 | T.xdep[i0]) << G.logM) + (y0 | T.xdep[j0]);
        oa = ((y0 | T.xdep[i0]) << G.logM) + (x0 | T.xdep[j0]);
        sm_d = i0 * P + j0;
        sm_a = j0 * P + i0;
    };
    // tile table and adjoint mask of item j, by the first two copy warps (one logical tile per
    // lane) into slot j % TSL, which no stage in flight uses
    auto tables = [&](uint64_t j, uint32_t t) {  // threads t < 64 (two warps): one logical tile per lane (NT <= 64)
        const uint32_t ts = (uint32_t)(j % TSL);
        uint64_t tbi, tbj;
        if (!G.grp4)
            unit_decode(G, item_of(j) >> (2 * G.log_nsb_side), !G.ws_diag, tbi, tbj);
        bool adj = false;
        if (G.grp4) {  // 4 consecutive local stored tiles, all direct (in-tile operation)
            if (t < NT) {
                const uint64_t idx = 4 * (item_of(j) >> (2 * G.log_nsb_side)) + t;
                gt[ts][t] = idx < G.nloc_tiles ? idx : (F_SKIP | F_NOSTORE);
                if (BULK && t == 0)
                    mir[ts] = 0;
            }
        } else if (t < NT) {
            const uint64_t tr = ins_bits(tbi, t >> G.logNG, G.gr_pos, G.g);
            const uint64_t tc = ins_bits(tbj, t & NGm, G.gr_pos, G.g);
            uint64_t ent = tile_entry(G, tr, tc);
            if (tbi == tbj) {
                // Diagonal unit: logical (R, C), R < C, aliases stored (C, R) of the same unit, so
                // sub-block items (a, b) and (b, a) read what the other writes.  Only a >= b runs:
                // a == b stores R >= C (the block is its own mirror); a > b stores every tile, R < C
                // through the adjoint write-back and R == C also at the mirrored position.
                const uint32_t sb = (uint32_t)(item_of(j) & nsbm);
                const uint32_t a = sb >> G.log_nsb_side, b = sb & ((1u << G.log_nsb_side) - 1);
                const uint32_t R = t >> G.logNG, C = t & NGm;
                if (a < b)
                    ent |= F_SKIP | F_NOSTORE;
                else if (a == b && R < C)
                    ent |= F_NOSTORE;
                else if (a > b && R == C && !(ent & F_NOSTORE))
                    ent |= F_MIRROR;
            }
            gt[ts][t] = ent;
            adj = (ent & F_ADJ) != 0;
            if (BULK && t == 0) {
                const uint32_t sb = (uint32_t)(item_of(j) & nsbm);
                mir[ts] = tbi == tbj && (sb >> G.log_nsb_side) > (sb & ((1u << G.log_nsb_side) - 1));
            }
        }
        const unsigned bal = __ballot_sync(0xffffffffu, adj);
        if ((t & 31) == 0)
            reinterpret_cast<uint32_t*>(&am[ts][0])[t >> 5] = bal;  // little endian: tiles 0-31, 32-63
        if (NMW / 2 == 32 && t == 0)  // one-warp copy groups (NT <= 32): tiles 32-63 absent
            reinterpret_cast<uint32_t*>(&am[ts][0])[1] = 0u;
    };
    // cp.async of item j into stage j % S (its table is visible: a copy-warp barrier separates them)
    auto issue = [&](uint64_t j) {
        const uint32_t s = (uint32_t)(j % S), ts = (uint32_t)(j % TSL);
        const uint32_t base = smem_u32(ring) + s * G.stage_elems * 16u;
        auto one = [&](uint32_t tt, uint32_t od, uint32_t oa, uint32_t sm_d, uint32_t sm_a) {
            const uint64_t ent = gt[ts][tt];
            if (ent & F_SKIP)
                return;
            const bool adj = (ent & F_ADJ) != 0;
            const uint64_t g = ((ent & F_MASK) << (2 * G.logM)) + (adj ? oa : od);
            cp_async16(base + (tt * G.TS + T.tsk[tt] + (adj ? sm_a : sm_d)) * 16u, tile_base(G, ent, st) + g);
        };
        if (G.dbg & 2u) {
        } else if (fast) {  // 8 tiles at one position: unrolled, table reads hoisted
            uint32_t od, oa, sm_d, sm_a;
            offsets(item_of(j), 0, od, oa, sm_d, sm_a);
#pragma unroll
            for (uint32_t e = 0; e < 8; ++e)
                one(tt0 + e * ttstep, od, oa, sm_d, sm_a);
        } else if (fast2) {
#pragma unroll
            for (uint32_t q = 0; q < 2; ++q) {
                uint32_t od, oa, sm_d, sm_a;
                offsets(item_of(j), q, od, oa, sm_d, sm_a);
#pragma unroll
                for (uint32_t tt = 0; tt < 4; ++tt)
                    one(tt, od, oa, sm_d, sm_a);
            }
        } else {
            for (uint32_t q = 0; q < npos; ++q) {
                uint32_t od, oa, sm_d, sm_a;
                offsets(item_of(j), q, od, oa, sm_d, sm_a);
                for (uint32_t tt = tt0; tt < NT; tt += ttstep)
                    one(tt, od, oa, sm_d, sm_a);
            }
        }
        asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        mbar_arrive(&full[s]);
    };
    const bool prof = (G.dbg & 16u) && mtid == 0;
    long long ph[4] = {0, 0, 0, 0};
    if constexpr (BULK) {
        // Two copy groups of NMW / 2 threads: group (i & 1) writes item i back (one bulk store per
        // row), waits until its stores have read the stage, and loads item i + S into it.  The other
        // group's stores of item i + 1 queue behind, so the bulk-copy engine always has work (one
        // group would leave it idle from the end of its stores to the issue of its loads).
        constexpr uint32_t NGT = NMW / 2;
        const uint32_t cg = mtid / NGT, gtid = mtid % NGT;
        auto gsync = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(3 + cg), "n"(NGT) : "memory"); };
        // runs: item = NT tiles x S0 rows x rps runs of 2^logRun elements (contiguous in-tile columns)
        const uint32_t lrr = G.logS0 - G.logRun, rps = 1u << lrr, lrt = G.logS0 + lrr;
        const uint32_t nruns = NT << lrt, rbytes = 16u << G.logRun;
        // TMA boxes: nbx x nbx boxes of 8 x 8 per tile (slot t * bpt + bx * nbx + by: base T.cdir, phase T.tsk)
        const uint32_t nbx = G.S0 >> 3, lnbx = G.logS0 - 3, lbpt = 2 * lnbx, bpt = 1u << lbpt;
        // in-tile offset of run c (sub-block column c) of sub-block row r: stored row x0|xdep[r]
        // (direct) or y0|xdep[r] (adjoint, stored orientation)
        auto run_off = [&](bool adj, uint32_t x0, uint32_t y0, uint32_t r, uint32_t c) -> uint64_t {
            return adj ? ((uint64_t)(y0 | T.xdep[r]) << G.logM) + (x0 | T.xdep[c])
                       : ((uint64_t)(x0 | T.xdep[r]) << G.logM) + (y0 | T.xdep[c]);
        };
        auto rows_of = [&](uint64_t j, uint32_t& x0, uint32_t& y0) {
            const uint32_t sb = (uint32_t)(item_of(j) & nsbm);
            x0 = G.sdep[sb >> G.log_nsb_side];
            y0 = G.sdep[sb & ((1u << G.log_nsb_side) - 1)];
        };
        auto bissue = [&](uint64_t j) {  // item j into stage j % S: one bulk copy per stored row
            const uint32_t s = (uint32_t)(j % S), ts = (uint32_t)(j % TSL);
            const uint32_t base = smem_u32(ring) + s * G.stage_elems * 16u;
            uint32_t x0, y0;
            rows_of(j, x0, y0);
            if constexpr (TMAB) {
                for (uint32_t q = gtid; !(G.dbg & 2u) && q < (NT << lbpt); q += NGT) {
                    const uint32_t t = q >> lbpt, bx = (q & (bpt - 1)) >> lnbx, by = q & (nbx - 1);
                    const uint64_t ent = gt[ts][t];
                    if (!(ent & F_SKIP)) {
                        const bool adj = (ent & F_ADJ) != 0;
                        const uint32_t r0 = (adj ? y0 : x0) | T.xdep[8 * bx], c0 = (adj ? x0 : y0) | T.xdep[8 * by];
                        mbar_expect(&full[s], 1024u);
                        tma_load_2d(base + T.cdir[q] * 16u, &tin, 2 * c0, (uint32_t)((ent & F_MASK) << G.logM) + r0, &full[s]);
                    }
                }
            } else {
                for (uint32_t q = gtid; !(G.dbg & 2u) && q < nruns; q += NGT) {
                    const uint32_t t = q >> lrt, r = (q >> lrr) & (G.S0 - 1), c = (q & (rps - 1)) << G.logRun;
                    const uint64_t ent = gt[ts][t];
                    if (!(ent & F_SKIP)) {
                        const bool adj = (ent & F_ADJ) != 0;
                        const uint64_t g = ((ent & F_MASK) << (2 * G.logM)) + run_off(adj, x0, y0, r, c);
                        mbar_expect(&full[s], rbytes);
                        bulk_g2s(base + (t * G.TS + T.tsk[t] + r * G.PD + (r >> 3) * G.s8 + c) * 16u, tile_base(G, ent, st) + g, rbytes,
                                 &full[s]);
                    }
                }
            }
            mbar_arrive(&full[s]);
            mbar_arrive(&full[s]);
        };
        for (uint64_t j = 0; j < S && j < nlocal; ++j)  // item j is loaded by group (j + 1) & 1
            if (((j + 1) & 1) == cg) {
                if (gtid < 64)
                    tables(j, gtid);
                gsync();
                bissue(j);
            }
        for (uint64_t i = cg; i < nlocal; i += 2) {
            const uint32_t s = (uint32_t)(i % S), ts = (uint32_t)(i % TSL);
            mbar_wait(&done[s], (uint32_t)((i / S) & 1));
            const bool more = i + S < nlocal;
            if (more && gtid < 64)
                tables(i + S, gtid);
            const double2* sb = ring + (size_t)s * G.stage_elems;
            if (!(G.dbg & 4u)) {
                uint32_t x0, y0;
                rows_of(i, x0, y0);
                if constexpr (TMAB) {
                    for (uint32_t q = gtid; q < (NT << lbpt); q += NGT) {
                        const uint32_t t = q >> lbpt, bx = (q & (bpt - 1)) >> lnbx, by = q & (nbx - 1);
                        const uint64_t ent = gt[ts][t];
                        if (!(ent & F_NOSTORE)) {
                            const bool adj = (ent & F_ADJ) != 0;
                            const uint32_t r0 = (adj ? y0 : x0) | T.xdep[8 * bx], c0 = (adj ? x0 : y0) | T.xdep[8 * by];
                            tma_store_2d(&tout, 2 * c0, (uint32_t)((ent & F_MASK) << G.logM) + r0, smem_u32(sb + T.cdir[q]));
                            bulk_commit();
                        }
                    }
                } else {
                    for (uint32_t q = gtid; q < nruns; q += NGT) {
                        const uint32_t t = q >> lrt, r = (q >> lrr) & (G.S0 - 1), c = (q & (rps - 1)) << G.logRun;
                        const uint64_t ent = gt[ts][t];
                        if (!(ent & F_NOSTORE)) {
                            const bool adj = (ent & F_ADJ) != 0;
                            const uint64_t g = ((ent & F_MASK) << (2 * G.logM)) + run_off(adj, x0, y0, r, c);
                            bulk_s2g(G.out + g, smem_u32(sb + t * G.TS + T.tsk[t] + r * G.PD + (r >> 3) * G.s8 + c), rbytes);
                            bulk_commit();
                        }
                    }
                }
                if (mir[ts]) {  // diagonal unit, a > b: the R == C tiles also at the mirrored position
                    for (uint32_t p = gtid; p < (NT << logT); p += NGT) {
                        const uint32_t tt = p >> logT, rr = p & (T2 - 1), i0 = rr >> G.logS0, j0 = rr & (G.S0 - 1);
                        const uint64_t ent = gt[ts][tt];
                        if (ent & F_MIRROR) {  // stored (y0|i0, x0|j0) = conj(logical (x0|j0, y0|i0))
                            uint32_t a;
                            if constexpr (TMAB) {
                                const uint32_t sl = (tt << lbpt) + (j0 >> 3) * nbx + (i0 >> 3);
                                a = T.cdir[sl] + (j0 & 7u) * 8u + ((i0 & 7u) ^ (((j0 & 7u) + T.tsk[sl]) & 7u));
                            } else {
                                a = tt * G.TS + T.tsk[tt] + j0 * P + (j0 >> 3) * G.s8 + i0;
                            }
                            const double2 w = sb[a];
                            G.out[((ent & F_MASK) << (2 * G.logM)) + ((uint64_t)(y0 | T.xdep[i0]) << G.logM) +
                                  (x0 | T.xdep[j0])] = make_double2(w.x, -w.y);
                        }
                    }
                }
                bulk_wait_read0();  // this thread's rows have left shared memory
            }
            gsync();  // the group's stores have read stage s; the table of item i + S is visible
            if (more && (G.dbg & DBG_POISON)) {  // diagnostics: NaN until the loads of item i + S land
                poison_stage(ring + (size_t)s * G.stage_elems, G.stage_elems, gtid, NGT);
                gsync();
            }
            if (more)
                bissue(i + S);
        }
        bulk_wait_all();
        return;
    }
    if (mtid < 64)
        for (uint64_t j = 0; j < S && j < nlocal; ++j)
            tables(j, mtid);
    mbar_sync();
    for (uint64_t j = 0; j < S && j < nlocal; ++j)
        issue(j);
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = (uint32_t)(i % S), ts = (uint32_t)(i % TSL);
        const long long t0 = prof ? clock64() : 0;
        mbar_wait(&done[s], (uint32_t)((i / S) & 1));
        const long long t1 = prof ? clock64() : 0;
        const bool more = i + S < nlocal;
        if (more && mtid < 64)
            tables(i + S, mtid);
        const double2* sb = ring + (size_t)s * G.stage_elems;
        auto wb = [&](uint32_t tt, uint32_t od, uint32_t oa, uint32_t sm_d, uint32_t sm_a) {
            const uint64_t ent = gt[ts][tt];
            if (ent & F_NOSTORE)
                return;
            const bool adj = (ent & F_ADJ) != 0;
            double2* o = G.out + ((ent & F_MASK) << (2 * G.logM));
            const double2* v = sb + tt * G.TS + T.tsk[tt];
            o[adj ? oa : od] = v[adj ? sm_a : sm_d];
            if (ent & F_MIRROR) {
                const double2 w = v[sm_a];
                o[oa] = make_double2(w.x, -w.y);
            }
        };
        if (G.dbg & 4u) {
        } else if (fast) {
            uint32_t od, oa, sm_d, sm_a;
            offsets(item_of(i), 0, od, oa, sm_d, sm_a);
#pragma unroll
            for (uint32_t e = 0; e < 8; ++e)
                wb(tt0 + e * ttstep, od, oa, sm_d, sm_a);
        } else if (fast2) {
#pragma unroll
            for (uint32_t q = 0; q < 2; ++q) {
                uint32_t od, oa, sm_d, sm_a;
                offsets(item_of(i), q, od, oa, sm_d, sm_a);
#pragma unroll
                for (uint32_t tt = 0; tt < 4; ++tt)
                    wb(tt, od, oa, sm_d, sm_a);
            }
        } else {
            for (uint32_t q = 0; q < npos; ++q) {
                uint32_t od, oa, sm_d, sm_a;
                offsets(item_of(i), q, od, oa, sm_d, sm_a);
                for (uint32_t tt = tt0; tt < NT; tt += ttstep)
                    wb(tt, od, oa, sm_d, sm_a);
            }
        }
        mbar_sync();  // every write-back read of stage s is done; the next table is visible
        const long long t2 = prof ? clock64() : 0;
        if (more && (G.dbg & DBG_POISON)) {  // diagnostics: NaN until the copies of item i + S land
            poison_stage(ring + (size_t)s * G.stage_elems, G.stage_elems, mtid, NMW);
            mbar_sync();
        }
        if (more)
            issue(i + S);
        if (prof) {
            const long long t3 = clock64();
            ph[0] += t1 - t0;
            ph[2] += t2 - t1;
            ph[3] += t3 - t2;
        }
    }
    if (prof)
        for (int q = 0; q < 4; ++q)
            atomicAdd(&g_phase_cycles[q], (unsigned long long)ph[q]);
    cp_async_wait<0>();
}

}  // namespace
