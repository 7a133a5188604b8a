// engine.cu -- B200 (sm_100a) conjugation engine behind the C-ABI of include/hs_cuda.h.
//
// Hot path (BASELINE.json north_star): rho -> sum_a L_a B L_a^dagger on every coupled
// 2^k x 2^k block B of a hermitian operator held in the reference's tiled lower-triangle
// layout (include/hermsim/storage.hpp:60-96).  The reference walks the blocks with CPU loops
// (quad_kernels.hpp:85-217, kernels.cpp:198-444, native.cpp); here one pass over HBM:
//
//   * A "unit" is the set of logical tiles one grid base pair couples: 2^g x 2^g tiles for the
//     g targets that are tile-grid bits (g = 0: one stored tile).  Logical tile (R, C) is the
//     stored tile (tr[R], tc[C]) when tr[R] >= tc[C] and otherwise the conjugate transpose of
//     the stored tile (tc[C], tr[R]) -- Algorithm 3's subcases A/B generalised to k <= 3
//     (SURVEY 8a').
//   * Path U: off-diagonal units (tbi > tbj), and every tile when g == 0.  A CTA stages a slab of
//     a unit (all its logical tiles, a set of in-tile rows closed under the in-tile target bits)
//     into shared memory in LOGICAL layout -- direct tiles row-wise, adjoint tiles read along
//     stored rows (sector-aligned column chunks) and transposed + conjugated on the way in --
//     applies the block transform in shared memory, and writes everything back.  Every stored
//     element belongs to exactly one slab, so slabs are independent CTAs.
//   * Path D: diagonal units (tbi == tbj, g >= 1), where logical (R, C) and (C, R) alias one
//     stored tile.  Blocks are visited on the lower wedge of in-tile base pairs and hermitian
//     mirrors are written explicitly (cross_tile_diag, quad_kernels.hpp:158-176, and the
//     diagonal branch of tiled_two_cross, kernels.cpp:281-297, generalised; this also carries
//     the corrected tiled_two_mixed mirror indices).
//   * Block transforms: transfer matrix S (k = 1, 2; kernels.cpp:27-77), real Hadamard quad
//     (native.cpp:332-339), direct two-stage U B U^dagger (k = 2, 3), monomial U = P D covering
//     Pauli X/Y, diagonal phases and permutations (native.cpp:99-549) with untouched logical
//     tiles skipped entirely, and a Kraus sum for k = 3.
//
// All data is complex128 (double2).  No tensor cores: the path is HBM-bound.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hs_cuda.h"

namespace {

constexpr int NTHR = 256;          // threads per CTA
constexpr uint32_t CAP = 2048;     // target complex elements staged per CTA item (32 KiB)
constexpr uint32_t CAPD = 2048;    // same for diagonal-unit items
constexpr uint32_t CAP_WHOLE = 4096;  // units up to 64 KiB are staged as whole stored tiles
constexpr uint32_t MAX_TT = 256;   // max logical tiles per item (tile table in smem)
constexpr uint64_t F_ADJ = 1ull << 63, F_SKIP = 1ull << 62, F_BAD = 1ull << 61, F_NOSTORE = 1ull << 60,
                   F_REMOTE = 1ull << 59, F_MASK = (1ull << 56) - 1;

enum Mode : int { M_S1 = 0, M_HAD = 1, M_S2 = 2, M_DIRECT = 3, M_MONO = 4, M_KRAUS = 5, M_PROG = 6 };

thread_local std::string g_err;
thread_local bool g_plan_subcases = true;  // hs_set_plan_subcases
std::atomic<uint64_t> g_launches{0};

int set_err(int code, const std::string& msg) {
    g_err = msg;
    return code;
}

#define CUDA_TRY(expr)                                                                          \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess)                                                                  \
            return set_err(HS_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));  \
    } while (0)

// ----------------------------------------------------------------------------- geometry
struct Geo {
    // storage
    uint32_t m, M, Mp, logM;
    uint64_t G;
    // operation
    uint32_t k, kin, g, D;
    uint32_t gr_pos[3];   // grid target bits (a - m), ascending
    uint32_t in_mask;     // in-tile target bits
    uint64_t nb;          // grid bases G >> g
    // path U
    uint64_t nU_units, nU_items;
    uint32_t offdiag;     // 1: units are grid base pairs tbi > tbj; 0: units are stored tiles
    uint32_t U, logU, SR, logSR, slabs, logSlabs, logNT, logNG, E;
    uint32_t nxb, logNxb, nyb, logNyb;
    uint32_t Epad;        // shared elements of a U item
    uint8_t xdep[32];     // xs -> in-tile row offset
    uint8_t sdep[32];     // slab -> in-tile row base
    uint8_t xb_tab[32];   // row-base index -> xs base
    uint8_t yb_tab[32];   // column-base index -> y base
    uint8_t xs_in[8], y_in[8];
    uint8_t xs_rin[32], xs_base[32], y_cin[32], y_base[32];
    uint16_t comp_off[64];
    uint64_t active;      // logical tiles (R * NG + C) that must be staged (monomial skip)
    // path D
    uint64_t nD_units, nD_items;
    uint32_t nbase, BPI, itemsD;
    uint64_t nblkD;
    // pipelined path U (pipe_kernel)
    uint32_t TS;          // shared elements reserved per logical tile slab (SR * M + max(SR, M))
    uint32_t SRp;         // pitch of an adjoint tile kept in stored orientation (SR + 1)
    uint32_t nruns;       // maximal runs of consecutive in-tile rows inside a slab
    uint8_t run_xs[32], run_len[32];
    uint32_t stages;      // shared-memory ring depth
    uint32_t stage_elems; // elements per stage buffer
    uint16_t cdir[64], cadj[64];  // component offsets from the unit base (direct / adjoint orientation)
    uint8_t ttr[64];              // logical tile (R * NG + C) of each component
    uint32_t A;                   // logical tiles staged per unit (monomials skip untouched ones)
    uint8_t slot[64];             // logical tile -> staging slot within its unit
    uint32_t diag_map;            // transform walks 8x8 position blocks diagonally
    uint32_t pipe_diag;           // pipeline also owns the diagonal units (whole-tile items)
    uint32_t groups;              // > 0: an item is (unit, tile group) of a tile permutation
    uint64_t gmask[16];           // logical tiles of each group
    uint32_t PD;                  // row pitch of a direct logical tile in shared memory
    uint32_t logical;             // adjoint tiles staged transposed (logical layout, gather kernel)
    uint8_t tsk[64];              // gather: per-logical-tile skew of the staging slot (bank spread for DMMA)
    // gather kernel (square sub-blocks of S0 x S0 positions, g >= 2)
    uint32_t S0, logS0, nsb_side, log_nsb_side;
    uint64_t nG_items;
    // sharding (XOR blocks over the top Plog tile-index bits; Plog == 0: the reference layout)
    uint32_t Plog, shard, logB;   // 2^Plog shards, this shard, 2^logB tile rows per block
    uint32_t cross, cmask;        // top targets: `cross` of them, shard bits cb[]; cmask: the shard bits whose
    uint32_t cb[3];               // remote tiles the op reads (all top targets, or only the moving ones)
    uint32_t xmask, nx, xb[3];    // exchange-slot layout (recv_mask): slot = pext(own ^ shard, xmask) - 1
    double2* out;                 // where stores go: the state itself, or (peer mode) the next buffer
    uint32_t q, Pulog, logBu;     // local units: group q over 2^Pulog blocks of 2^logBu grid bases
    const double2* rbase[7];      // remote tiles of group slot j: exchange buffer slot j, or the peer's payload
    uint64_t nU_strict, nU_loose; // local off-diagonal units / units including diagonal ones
    uint32_t dbg;                 // diagnostics (HS_DEBUG_FLAGS): gather bit 0 skips the transform, bit 1 the loads, bit 2 the stores
    uint32_t ws_diag;             // gather_ws: units include the diagonal base pairs (grid programs)
    uint32_t rev;                 // sweep the items in reverse order (alternates per launch: L2 reuse)
};

// Per-CTA copies of the small index tables of Geo (shared memory).
struct Tabs {
    uint8_t xdep[32], xb[32], yb[32], xs_rin[32], xs_base[32], y_cin[32], y_base[32], xs_in[8], y_in[8];
    uint16_t cdir[64], cadj[64];  // component offsets (copied from Geo: indexed per thread)
    uint8_t ttr[64];
    uint8_t tsk[64];
    uint8_t slt[64];  // pipe kernel, monomials: staging slot -> logical tile (compacted active tiles)
};

template <int NS>
struct Coef {
    double2 s[NS];
    uint8_t pinv[8];
    uint64_t fone;   // monomial: bit (rho*D+gamma) set when the factor is exactly 1
    // monomial, in place: non-trivial cycles of the component map c -> src(c); out[cyc[j]] =
    // f[cyc[j]] * in[cyc[j+1]] within each cycle [cyc_off[i], cyc_off[i+1])
    uint8_t cyc[64];
    uint8_t cyc_off[66];
    uint32_t ncyc;
    // tile permutations (every target a grid bit): cycles grouped into <= 4-tile item groups;
    // group g owns cycles [gcyc_off[g], gcyc_off[g + 1])
    uint8_t gcyc_off[17];
    // fused program (M_PROG): nsteps single-qubit steps on in-tile bits, step p uses s[16p .. 16p+15]
    uint8_t pbit[16], pkind[16];
    uint32_t nsteps;
    // k = 1 transfer matrix that couples only (00, 11) and (01, 10) (depolarising, amplitude
    // damping, dephasing, ...): w = S v reads only class-consistent components
    uint32_t xpat;
    // monomial that is diagonal (phases only): element-wise scaling fast path; ibit = in-tile
    // target bits (ascending), nib of them
    uint32_t diag, nib;
    uint8_t ibit[3];
    uint32_t ngroups;  // tile permutations: number of item groups
};

uint32_t pdep(uint32_t v, uint32_t mask) {
    uint32_t r = 0;
    for (uint32_t b = 0, i = 0; b < 32; ++b)
        if (mask >> b & 1u) {
            if (v >> i & 1u)
                r |= 1u << b;
            ++i;
        }
    return r;
}
uint32_t pext(uint32_t v, uint32_t mask) {
    uint32_t r = 0;
    for (uint32_t b = 0, i = 0; b < 32; ++b)
        if (mask >> b & 1u) {
            if (v >> b & 1u)
                r |= 1u << i;
            ++i;
        }
    return r;
}
uint32_t ilog2(uint64_t v) {
    uint32_t r = 0;
    while ((1ull << r) < v)
        ++r;
    return r;
}

// ------------------------------------------------------------------------ device helpers
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
__device__ __forceinline__ double2 cfma(double2 a, double2 b, double2 c) {  // c + a*b
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(-a.y, b.y, c.x);
    c.y = fma(a.x, b.y, c.y);
    c.y = fma(a.y, b.x, c.y);
    return c;
}
__device__ __forceinline__ double2 cfmaconj(double2 a, double2 b, double2 c) {  // c + a*conj(b)
    c.x = fma(a.x, b.x, c.x);
    c.x = fma(a.y, b.y, c.x);
    c.y = fma(a.y, b.x, c.y);
    c.y = fma(-a.x, b.y, c.y);
    return c;
}
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }
__device__ __forceinline__ double2 ldg2(const double2* p) { return *p; }

__device__ __forceinline__ uint64_t tri(uint64_t t) { return t * (t + 1) / 2; }

// insert_bits (bit_index.hpp:40-51) on grid indices
__device__ __forceinline__ uint64_t ins_bits(uint64_t s, uint32_t a, const uint32_t* pos, uint32_t k) {
    for (uint32_t l = 0; l < k; ++l) {
        const uint32_t p = pos[l];
        const uint64_t right = s & ((1ull << p) - 1);
        s = ((((s >> p) << 1) | ((a >> l) & 1u)) << p) | right;
    }
    return s;
}

// u -> (i > j) with u = i(i-1)/2 + j
__device__ __forceinline__ void tri_strict(uint64_t u, uint64_t& i, uint64_t& j) {
    uint64_t r = (uint64_t)((1.0 + sqrt(1.0 + 8.0 * (double)u)) * 0.5);
    while (r * (r - 1) / 2 > u)
        --r;
    while ((r + 1) * r / 2 <= u)
        ++r;
    i = r;
    j = u - r * (r - 1) / 2;
}
// u -> (i >= j) with u = i(i+1)/2 + j
__device__ __forceinline__ void tri_loose(uint64_t u, uint64_t& i, uint64_t& j) {
    uint64_t r = (uint64_t)((sqrt(1.0 + 8.0 * (double)u) - 1.0) * 0.5);
    while (r * (r + 1) / 2 > u)
        --r;
    while ((r + 1) * (r + 2) / 2 <= u)
        ++r;
    i = r;
    j = u - r * (r + 1) / 2;
}

// ----------------------------------------------------------------------- shard addressing
// XOR blocks: stored tile (ti >= tj) belongs to shard (ti >> logB) ^ (tj >> logB).  Shard 0
// stores the 2^Plog diagonal blocks (triangular, B(B+1)/2 tiles each), shard s != 0 the 2^(Plog-1)
// rectangular blocks (a, a ^ s) with a > a ^ s (B x B tiles, row-major), ordered by a with bit
// msb(s) removed.  With Plog == 0 this is exactly the reference's triangle (storage.hpp:78-83).
__device__ __forceinline__ uint32_t msb32(uint32_t v) { return 31u - __clz(v); }
__device__ __forceinline__ uint32_t del_bit(uint32_t a, uint32_t h) {
    return ((a >> (h + 1)) << h) | (a & ((1u << h) - 1));
}
__device__ __forceinline__ uint32_t ins_one(uint32_t v, uint32_t h) {
    return ((v >> h) << (h + 1)) | (1u << h) | (v & ((1u << h) - 1));
}
__device__ __forceinline__ uint32_t shard_of(uint32_t Plog, uint32_t logB, uint64_t tr, uint64_t tc) {
    return Plog ? (uint32_t)((tr >> logB) ^ (tc >> logB)) : 0u;
}
__device__ __forceinline__ uint64_t shard_index(uint32_t Plog, uint32_t logB, uint64_t tr, uint64_t tc, uint32_t s) {
    if (!Plog)
        return tri(tr) + tc;
    const uint32_t a = (uint32_t)(tr >> logB);
    const uint64_t Bm = (1ull << logB) - 1, r = tr & Bm, c = tc & Bm;
    if (s == 0)
        return (uint64_t)a * ((Bm + 1) * (Bm + 2) / 2) + tri(r) + c;
    return ((uint64_t)del_bit(a, msb32(s)) << (2 * logB)) + (r << logB) + c;
}
// local tile index -> (ti, tj) in shard s
__device__ __forceinline__ void shard_decode(uint32_t Plog, uint32_t logB, uint32_t s, uint64_t t, uint64_t& ti,
                                             uint64_t& tj) {
    if (!Plog) {
        tri_loose(t, ti, tj);
        return;
    }
    const uint64_t B = 1ull << logB;
    if (s == 0) {
        const uint64_t per = B * (B + 1) / 2, a = t / per;
        uint64_t r, c;
        tri_loose(t - a * per, r, c);
        ti = a * B + r;
        tj = a * B + c;
    } else {
        const uint32_t a = ins_one((uint32_t)(t >> (2 * logB)), msb32(s)), b = a ^ s;
        const uint64_t v = t & (B * B - 1);
        ti = (uint64_t)a * B + (v >> logB);
        tj = (uint64_t)b * B + (v & (B - 1));
    }
}
// base pointer of the payload an entry's tile lives in (own state or the group slot's source)
__device__ __forceinline__ const double2* tile_base(const Geo& G, uint64_t ent, const double2* st) {
    return (ent & F_REMOTE) ? G.rbase[(ent >> 56) & 7u] : st;
}
// (stored-tile index | F_ADJ | F_REMOTE) of logical tile (tr, tc) for this operation's shard
__device__ __forceinline__ uint64_t tile_entry(const Geo& G, uint64_t tr, uint64_t tc) {
    const bool adj = tr < tc;
    const uint64_t hi = adj ? tc : tr, lo = adj ? tr : tc;
    const uint32_t own = shard_of(G.Plog, G.logB, hi, lo);
    uint64_t ent = shard_index(G.Plog, G.logB, hi, lo, own);
    if (adj)
        ent |= F_ADJ;
    if (own != G.shard) {
        const uint32_t d = own ^ G.shard;
        if (d & ~G.cmask)  // a shard the op never reads from (stationary top target): not staged
            return ent | F_REMOTE | F_NOSTORE | F_SKIP;
        uint32_t slot = 0;
        for (uint32_t i = 0; i < G.nx; ++i)
            slot |= ((d >> G.xb[i]) & 1u) << i;
        ent |= F_REMOTE | F_NOSTORE | ((uint64_t)(slot - 1) << 56);  // bits 56-58: the slot
    }
    return ent;
}
// Item j of this CTA (persistent kernels: items blockIdx + j * gridDim).  Consecutive operations
// sweep the state in opposite directions, so the lines the previous operation wrote last (still in
// the 126 MB L2) are read first: an L2-sized state (n = 12: 135 MB) is then largely served from L2.
__device__ __forceinline__ uint64_t sweep_item(const Geo& G, uint64_t n_items, uint64_t j) {
    const uint64_t it = blockIdx.x + j * gridDim.x;
    return G.rev ? n_items - 1 - it : it;
}
// local unit u -> grid base pair (tbi, tbj); strict: off-diagonal units only
__device__ __forceinline__ void unit_decode(const Geo& G, uint64_t u, bool strict, uint64_t& tbi, uint64_t& tbj) {
    if (!G.Pulog) {
        if (strict)
            tri_strict(u, tbi, tbj);
        else
            tri_loose(u, tbi, tbj);
        return;
    }
    const uint64_t Bu = 1ull << G.logBu;
    if (G.q == 0) {
        const uint64_t per = strict ? Bu * (Bu - 1) / 2 : Bu * (Bu + 1) / 2, a = u / per;
        uint64_t r, c;
        if (strict)
            tri_strict(u - a * per, r, c);
        else
            tri_loose(u - a * per, r, c);
        tbi = a * Bu + r;
        tbj = a * Bu + c;
    } else {
        const uint32_t a = ins_one((uint32_t)(u >> (2 * G.logBu)), msb32(G.q)), b = a ^ G.q;
        const uint64_t v = u & (Bu * Bu - 1);
        tbi = (uint64_t)a * Bu + (v >> G.logBu);
        tbj = (uint64_t)b * Bu + (v & (Bu - 1));
    }
}

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
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
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
// (01, 10) (depolarising, amplitude damping and their compositions).
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
    } else if (kind == 2) {
        w0 = cmul(S[0], v0);
        w1 = cmul(S[5], v1);
        w2 = cmul(S[10], v2);
        w3 = cmul(S[15], v3);
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
template <int K, int MODE, int NS, int NC = NCONS>
__device__ __forceinline__ void pipe_compute(const Geo& G, const Tabs& T, const Coef<NS>& cf, const uint64_t* am,
                                             uint32_t nvalid_units, double2* sb, uint32_t grp = 0, int tidv = -1,
                                             uint32_t barid = 1) {
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
        const uint32_t lq = G.logM - 1, nq = nvalid_units << (2 * lq), M = G.M;
        for (uint32_t p = 0; p < cf.nsteps; ++p) {
            const uint32_t a = cf.pbit[p], sa = 1u << a, lo = sa - 1, kind = cf.pkind[p];
            const double2* S = cf.s + 16 * p;
            for (uint32_t q = tid; q < nq; q += NC) {
                const uint32_t u = q >> (2 * lq), r = q & ((1u << (2 * lq)) - 1);
                const uint32_t qx = r >> lq, qy = r & ((1u << lq) - 1);
                const uint32_t x = ((qx & ~lo) << 1) | (qx & lo), y = ((qy & ~lo) << 1) | (qy & lo);
                const uint32_t b0 = u * G.A * G.TS + x * M + y;
                const uint32_t b1 = b0 + sa, b2 = b0 + sa * M, b3 = b2 + sa;
                double2 v0 = sb[b0], v1 = sb[b1], v2 = sb[b2], v3 = sb[b3];
                prog_quad(kind, S, v0, v1, v2, v3);
                sb[b0] = v0;
                sb[b1] = v1;
                sb[b2] = v2;
                sb[b3] = v3;
            }
            if (p + 1 < cf.nsteps)
                asm volatile("bar.sync %0, %1;" ::"r"(barid), "n"(NC) : "memory");  // consumer warps only
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
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = (uint32_t)(i % S);
        double2* sb = ring + (size_t)s * G.stage_elems;
        const uint64_t item = sweep_item(G, nItems, i);
        const uint32_t grp = G.groups ? (uint32_t)(item % G.groups) : 0;
        const uint64_t u0 = G.groups ? item / G.groups : (item >> G.logSlabs) << G.logU;
        const uint32_t nvalid = G.nU_units - u0 < G.U ? (uint32_t)(G.nU_units - u0) : G.U;
        mbar_wait(&full[s], (uint32_t)((i / S) & 1));
        pipe_compute<K, MODE, NS>(G, T, cf, am[s], nvalid, sb, grp);
        fence_async_smem();
        __syncwarp();
        if (lane == 0)
            mbar_arrive(&done[s]);
    }
}


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
// conjugation flag applied as a sign-bit flip on the integer pipe (a DADD negation would compete
// with the DMMA for the FP64 pipe)
__device__ __forceinline__ double flip_sign(double x, uint32_t m) {
    return __hiloint2double(__double2hiint(x) ^ (int)m, __double2loint(x));
}
// per-lane constant fragments of the transform (loaded once per kernel: the lane-dependent
// coefficient index would serialise the constant-cache reads if repeated per item)
struct DmmaFrag {
    double lr[2], li[2], nli[2];
    double ls[2], ld[2];      // Lr + Li (stage 1, 3M) and Pr + Pi = Lr - Li (stage 2, 3M)
    uint32_t old[2], ost[2];  // staging offsets of the loaded / stored components (from the block base)
    uint32_t tld[2], tst[2];  // their logical tiles (adjoint mask bits)
};
// k = 3: the 8 x 8 block itself.  k = 2: four 4 x 4 blocks (2X + R1, 2Y + C1) as the quadrants of
// one 8 x 8 matrix M, transformed by I2 (x) L: (I2 (x) L) M (I2 (x) L)^dagger applies L . L^dagger to
// every quadrant, so one tensor-core transform serves four k = 2 blocks (kin = 0: quadrant
// offsets are R1 * PD + C1, folded into the component offsets).
template <int K, int NS>
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
        f.nli[j] = -l.y;
        f.ls[j] = l.x + l.y;
        f.ld[j] = l.x - l.y;
        if constexpr (K == 3) {
            const uint32_t il = c8 * 8 + gq, is = gq * 8 + c8;
            f.old[j] = T.cdir[il];
            f.ost[j] = T.cdir[is];
            f.tld[j] = T.ttr[il];
            f.tst[j] = T.ttr[is];
        } else {
            // load component (row c8, column gq), store component (row gq, column c8) of M
            const uint32_t il = (c8 & 3) * 4 + (gq & 3), is = (gq & 3) * 4 + (c8 & 3);
            f.old[j] = T.cdir[il] + (c8 >> 2) * G.PD + (gq >> 2);
            f.ost[j] = T.cdir[is] + (gq >> 2) * G.PD + (c8 >> 2);
            f.tld[j] = T.ttr[il];
            f.tst[j] = T.ttr[is];
        }
    }
    return f;
}
template <int NC, int K = 3>
__device__ __forceinline__ void dmma_direct3(const Geo& G, const Tabs& T, const DmmaFrag& f, uint64_t am,
                                             double2* sb, uint32_t warp) {
    constexpr uint32_t sh = K == 3 ? 0u : 1u;  // k = 2: 8 x 8 matrices of 2 x 2 blocks
    const uint32_t cld0 = (uint32_t)((am >> f.tld[0]) & 1ull) << 31, cld1 = (uint32_t)((am >> f.tld[1]) & 1ull) << 31;
    const uint32_t cst0 = (uint32_t)((am >> f.tst[0]) & 1ull) << 31, cst1 = (uint32_t)((am >> f.tst[1]) & 1ull) << 31;
    const uint32_t logNy = G.logNyb - sh, nblk = (G.nxb >> sh) << logNy, ymask = (G.nyb >> sh) - 1;
    // two blocks per pass: independent accumulator chains keep the FP64 tensor pipe fed (small
    // tiles, m < 5, have fewer blocks than warps: the second block of a pass may be absent and is
    // then computed on a copy of the first and not stored)
    for (uint32_t b = warp; b < nblk; b += 2 * (NC / 32)) {
        uint32_t base[2];
        double2 v0[2], v1[2];
        const bool two = b + NC / 32 < nblk;
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            const uint32_t bq = (q && two) ? b + NC / 32 : b;
            base[q] = T.xb[(bq >> logNy) << sh] * G.PD + T.yb[(bq & ymask) << sh];
            v0[q] = sb[base[q] + f.old[0]];
            v1[q] = sb[base[q] + f.old[1]];
            v0[q].y = flip_sign(v0[q].y, cld0);
            v1[q].y = flip_sign(v1[q].y, cld1);
        }
        // 3M form (Gauss): three real products per complex product.  Stage 1: Y = L B with
        // T1 = Lr Br, T2 = Li Bi, T3 = (Lr + Li)(Br + Bi); Yr = T1 - T2, Yi = T3 - T1 - T2
        double yr0[2], yr1[2], yi0[2], yi1[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            double t1a = 0.0, t1b = 0.0, t2a = 0.0, t2b = 0.0, t3a = 0.0, t3b = 0.0;
            const double s0 = v0[q].x + v0[q].y, s1 = v1[q].x + v1[q].y;
            dmma_acc(t1a, t1b, f.lr[0], v0[q].x);
            dmma_acc(t2a, t2b, f.li[0], v0[q].y);
            dmma_acc(t3a, t3b, f.ls[0], s0);
            dmma_acc(t1a, t1b, f.lr[1], v1[q].x);
            dmma_acc(t2a, t2b, f.li[1], v1[q].y);
            dmma_acc(t3a, t3b, f.ls[1], s1);
            yr0[q] = t1a - t2a;
            yr1[q] = t1b - t2b;
            yi0[q] = t3a - t1a - t2a;
            yi1[q] = t3b - t1b - t2b;
        }
        // stage 2: Z = Y P, P = L^dagger (B fragment of chunk j: P[2c + j][g] = conj(L[g][2c + j]));
        // U1 = Yr Pr, U2 = Yi Pi, U3 = (Yr + Yi)(Pr + Pi); Zr = U1 - U2, Zi = U3 - U1 - U2
        double zr0[2], zr1[2], zi0[2], zi1[2];
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            double u1a = 0.0, u1b = 0.0, u2a = 0.0, u2b = 0.0, u3a = 0.0, u3b = 0.0;
            const double s0 = yr0[q] + yi0[q], s1 = yr1[q] + yi1[q];
            dmma_acc(u1a, u1b, yr0[q], f.lr[0]);
            dmma_acc(u2a, u2b, yi0[q], f.nli[0]);
            dmma_acc(u3a, u3b, s0, f.ld[0]);
            dmma_acc(u1a, u1b, yr1[q], f.lr[1]);
            dmma_acc(u2a, u2b, yi1[q], f.nli[1]);
            dmma_acc(u3a, u3b, s1, f.ld[1]);
            zr0[q] = u1a - u2a;
            zr1[q] = u1b - u2b;
            zi0[q] = u3a - u1a - u2a;
            zi1[q] = u3b - u1b - u2b;
        }
#pragma unroll
        for (int q = 0; q < 2; ++q) {
            if (q && !two)
                break;
            sb[base[q] + f.ost[0]] = make_double2(zr0[q], flip_sign(zi0[q], cst0));
            sb[base[q] + f.ost[1]] = make_double2(zr1[q], flip_sign(zi1[q], cst1));
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
template <uint32_t NCW, int NS>
__device__ __forceinline__ void grid_prog_step(const Geo& G, const Tabs& T, const Coef<NS>& cf, uint32_t p,
                                               uint64_t am, double2* sb, uint32_t tid) {
    const uint32_t g = G.g, NG = 1u << g, e = 1u << cf.pbit[p], lo = e - 1;
    const uint32_t S0 = G.S0, P = S0 + 1, npos = S0 * S0, lp = 2 * G.logS0;
    const uint32_t nq = (NG / 2) * (NG / 2) * npos;
    const double2* S = cf.s + 16 * p;
    const uint32_t kind = cf.pkind[p];
    for (uint32_t q = tid; q < nq; q += NCW) {
        const uint32_t tq = q >> lp, pos = q & (npos - 1), i = pos >> G.logS0, j = pos & (S0 - 1);
        const uint32_t rr = tq >> (g - 1), cc = tq & ((NG >> 1) - 1);
        const uint32_t R0 = ((rr & ~lo) << 1) | (rr & lo), C0 = ((cc & ~lo) << 1) | (cc & lo);
        const uint32_t t0 = R0 * NG + C0, t1 = R0 * NG + (C0 | e), t2 = (R0 | e) * NG + C0, t3 = t2 + e;
        const uint32_t off = i * P + j;
        const uint32_t a0 = t0 * G.TS + T.tsk[t0] + off, a1 = t1 * G.TS + T.tsk[t1] + off;
        const uint32_t a2 = t2 * G.TS + T.tsk[t2] + off, a3 = t3 * G.TS + T.tsk[t3] + off;
        const uint32_t f0 = (uint32_t)((am >> t0) & 1ull) << 31, f1 = (uint32_t)((am >> t1) & 1ull) << 31;
        const uint32_t f2 = (uint32_t)((am >> t2) & 1ull) << 31, f3 = (uint32_t)((am >> t3) & 1ull) << 31;
        double2 v0 = sb[a0], v1 = sb[a1], v2 = sb[a2], v3 = sb[a3];
        v0.y = flip_sign(v0.y, f0);
        v1.y = flip_sign(v1.y, f1);
        v2.y = flip_sign(v2.y, f2);
        v3.y = flip_sign(v3.y, f3);
        prog_quad(kind, S, v0, v1, v2, v3);
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

template <int K, int NS, int MODE = M_DIRECT>
__global__ void __launch_bounds__(768, 1) gather_ws_kernel(const Geo G, const Coef<NS> cf, double2* __restrict__ st) {
    constexpr uint32_t NCW = 256, NMW = 512, S = 3;
    extern __shared__ __align__(128) double2 ring[];
    __shared__ uint64_t gt[S + 1][64];  // tile tables by item % (S + 1): built one item ahead
    __shared__ uint64_t am[S + 1][1];
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
    }
    if (tid == 0)
        for (uint32_t q = 0; q < S; ++q) {
            mbar_init(&full[q], 2 * NMW);
            mbar_init(&done[q], NCW);
        }
    const uint64_t nItems = G.nG_items;
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item_of = [&](uint64_t j) { return sweep_item(G, nItems, j); };
    __syncthreads();
    if (tid < NCW) {
        // ---- transform warps
        DmmaFrag fr;
        if constexpr (MODE == M_DIRECT)
            fr = dmma_frag<K>(G, T, cf);
        for (uint64_t i = 0; i < nlocal; ++i) {
            const uint32_t s = (uint32_t)(i % S);
            mbar_wait(&full[s], (uint32_t)((i / S) & 1));
            double2* sb = ring + (size_t)s * G.stage_elems;
            if constexpr (MODE == M_DIRECT) {
                if (!(G.dbg & 1u))
                    dmma_direct3<NCW, K>(G, T, fr, am[i % (S + 1)][0], sb, tid >> 5);
            } else {
                for (uint32_t p = 0; p < cf.nsteps; ++p) {
                    grid_prog_step<NCW>(G, T, cf, p, am[i % (S + 1)][0], sb, tid);
                    asm volatile("bar.sync 2, %0;" ::"n"(NCW) : "memory");  // transform warps only
                }
            }
            mbar_arrive(&done[s]);
        }
        return;
    }
    // ---- copy warps
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
    // lane) into slot j % (S + 1), which no stage in flight uses
    auto tables = [&](uint64_t j) {  // copy warps 0 and 1: one logical tile per lane (NT <= 64)
        const uint32_t ts = (uint32_t)(j % (S + 1));
        uint64_t tbi, tbj;
        unit_decode(G, item_of(j) >> (2 * G.log_nsb_side), !G.ws_diag, tbi, tbj);
        const uint32_t t = mtid;
        bool adj = false;
        if (t < NT) {
            const uint64_t tr = ins_bits(tbi, t >> G.logNG, G.gr_pos, G.g);
            const uint64_t tc = ins_bits(tbj, t & NGm, G.gr_pos, G.g);
            uint64_t ent = tile_entry(G, tr, tc);
            if (tbi == tbj && (t >> G.logNG) < (t & NGm))
                ent |= F_NOSTORE;  // aliases stored (C, R) of the same diagonal unit: read-only copy
            gt[ts][t] = ent;
            adj = (ent & F_ADJ) != 0;
        }
        const unsigned bal = __ballot_sync(0xffffffffu, adj);
        if ((mtid & 31) == 0)
            reinterpret_cast<uint32_t*>(&am[ts][0])[mtid >> 5] = bal;  // little endian: tiles 0-31, 32-63
    };
    // cp.async of item j into stage j % S (its table is visible: a copy-warp barrier separates them)
    auto issue = [&](uint64_t j) {
        const uint32_t s = (uint32_t)(j % S), ts = (uint32_t)(j % (S + 1));
        const uint32_t base = smem_u32(ring) + s * G.stage_elems * 16u;
        auto one = [&](uint32_t tt, uint32_t od, uint32_t oa, uint32_t sm_d, uint32_t sm_a) {
            const uint64_t ent = gt[ts][tt];
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
    if (mtid < 64)
        for (uint64_t j = 0; j < S && j < nlocal; ++j)
            tables(j);
    mbar_sync();
    for (uint64_t j = 0; j < S && j < nlocal; ++j)
        issue(j);
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = (uint32_t)(i % S), ts = (uint32_t)(i % (S + 1));
        const long long t0 = prof ? clock64() : 0;
        mbar_wait(&done[s], (uint32_t)((i / S) & 1));
        const long long t1 = prof ? clock64() : 0;
        const bool more = i + S < nlocal;
        if (more && mtid < 64)
            tables(i + S);
        const double2* sb = ring + (size_t)s * G.stage_elems;
        auto wb = [&](uint32_t tt, uint32_t od, uint32_t oa, uint32_t sm_d, uint32_t sm_a) {
            const uint64_t ent = gt[ts][tt];
            if (ent & F_NOSTORE)
                return;
            const bool adj = (ent & F_ADJ) != 0;
            G.out[((ent & F_MASK) << (2 * G.logM)) + (adj ? oa : od)] = sb[tt * G.TS + T.tsk[tt] + (adj ? sm_a : sm_d)];
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

}  // namespace

// =============================================================================== host side
struct hs_state {
    int n, m, device;
    uint64_t N, M, G, count;
    double2* d = nullptr;
    cudaStream_t stream = nullptr;
    bool own_stream = false;
    double* red = nullptr;  // reduction scratch: 2 * RED_BLOCKS partials + result
    double2* kraus = nullptr;  // device buffer for k = 3 Kraus operators
    size_t kraus_cap = 0;
    // sharding (XOR blocks): 2^Plog shards of 2^logB tile rows per block; this is shard `shard`
    uint32_t Plog = 0, logB = 0, shard = 0;
    double2* recv = nullptr;  // group members' payloads for cross-shard operations (slots)
    uint64_t recv_count = 0;  // elements per slot (the largest shard)
    uint64_t sweeps = 0;      // launches so far (alternating sweep direction)
    uint32_t recv_slots = 0;  // allocated slots
    uint32_t recv_mask = 0;   // shard-bit mask of the last exchange (which slots hold whom)
    void* comm = nullptr;     // ncclComm_t
    // peer mode: cross-shard operations read the group members' payloads in place (peer memory over
    // NVLink, or the same device) and write this shard's result out of place into the other buffer
    bool peer_mode = false;
    double2* buf[2] = {nullptr, nullptr};     // this shard's two payload buffers (buf[flip] is current)
    uint32_t flip = 0;
    const double2* peer_buf[64][2] = {};       // peers' buffers, valid on this device
};

namespace {

// NCCL, loaded on first use (the engine itself does not depend on it): whichever libnccl.so.2 the
// process already has (PyTorch's bundled one) or the system library.
struct NcclApi {
    bool tried = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi& nccl() {
    static NcclApi api;
    if (!api.tried) {
        api.tried = true;
        void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (lib) {
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(lib, "ncclGetUniqueId");
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(lib, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(lib, "ncclCommDestroy");
            api.Send = (decltype(api.Send))dlsym(lib, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(lib, "ncclRecv");
            api.GroupStart = (decltype(api.GroupStart))dlsym(lib, "ncclGroupStart");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(lib, "ncclGroupEnd");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(lib, "ncclGetErrorString");
        }
    }
    return api;
}

uint64_t shard_count_of(const hs_state* h, uint32_t shard) {
    const uint64_t B = 1ull << h->logB, P = 1ull << h->Plog;
    const uint64_t tiles = shard == 0 ? P * (B * (B + 1) / 2) : (P / 2) * B * B;
    return tiles * h->M * h->M;
}

struct DeviceGuard {
    int prev = -1;
    explicit DeviceGuard(int dev) {
        cudaGetDevice(&prev);
        if (prev != dev)
            cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        int cur;
        cudaGetDevice(&cur);
        if (prev >= 0 && cur != prev)
            cudaSetDevice(prev);
    }
};

int check_targets(const hs_state* h, int k, const uint32_t* t) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (k < 1 || k > 3 || !t)
        return set_err(HS_ERR_INVALID, "locality must be 1..3");
    for (int i = 0; i < k; ++i) {
        if (t[i] >= (uint32_t)h->n)
            return set_err(HS_ERR_RANGE, "target qubit out of range");
        if (i > 0 && t[i - 1] >= t[i])
            return set_err(HS_ERR_INVALID, "bound targets must be strictly ascending");
    }
    return HS_OK;
}

// Builds the launch geometry of one k-local operation on state h.
void plan_geo(const hs_state* h, int k, const uint32_t* t, Geo& G, uint32_t extra_buffers) {
    std::memset(&G, 0, sizeof(G));
    G.m = h->m;
    G.M = 1u << h->m;
    G.logM = h->m;
    G.Mp = G.M >= 8 ? G.M + 1 : G.M;
    G.G = h->G;
    G.k = k;
    G.D = 1u << k;
    uint32_t in_mask = 0;
    uint32_t g = 0;
    for (int l = 0; l < k; ++l) {
        if (t[l] < (uint32_t)h->m)
            in_mask |= 1u << t[l];
        else
            G.gr_pos[g++] = t[l] - h->m;
    }
    G.in_mask = in_mask;
    G.g = g;
    G.kin = k - g;
    G.logNG = g;
    G.logNT = 2 * g;
    const uint32_t NT = 1u << (2 * g);
    G.nb = G.G >> g;
    // sharding: which units this shard works on (local unit enumeration, see unit_decode)
    G.Plog = h->Plog;
    G.shard = h->shard;
    G.logB = h->logB;
    G.out = h->d;
    G.cross = 0;
    G.cmask = 0;
    G.cb[0] = G.cb[1] = G.cb[2] = 0;
    G.xmask = G.nx = 0;
    G.xb[0] = G.xb[1] = G.xb[2] = 0;
    G.Pulog = h->Plog;
    G.q = h->shard;
    if (h->Plog && g) {
        const uint32_t gbits = ilog2(G.G), top0 = gbits - h->Plog;
        for (uint32_t l = 0; l < g; ++l)  // gr_pos ascending
            if (G.gr_pos[l] >= top0) {
                G.cb[G.cross++] = G.gr_pos[l] - top0;
                G.cmask |= 1u << (G.gr_pos[l] - top0);
            }
        // the group's units: the shard index with the cross bits deleted (highest first)
        G.Pulog = h->Plog - G.cross;
        uint32_t q = h->shard;
        for (int i = (int)G.cross - 1; i >= 0; --i)
            q = ((q >> (G.cb[i] + 1)) << G.cb[i]) | (q & ((1u << G.cb[i]) - 1));
        G.q = q;
    }
    G.logBu = ilog2(G.nb) - G.Pulog;
    {
        const uint64_t Bu = 1ull << G.logBu, Pu = 1ull << G.Pulog;
        if (G.Pulog == 0) {
            G.nU_strict = G.nb * (G.nb - 1) / 2;
            G.nU_loose = G.nb * (G.nb + 1) / 2;
        } else if (G.q == 0) {
            G.nU_strict = Pu * (Bu * (Bu - 1) / 2);
            G.nU_loose = Pu * (Bu * (Bu + 1) / 2);
        } else {
            G.nU_strict = G.nU_loose = (Pu / 2) * Bu * Bu;
        }
    }
    if (g == 0) {
        G.offdiag = 0;
        G.nU_units = h->count >> (2 * h->m);  // local tiles
        G.nD_units = 0;
    } else {
        G.offdiag = 1;
        G.nU_units = G.nU_strict;
        G.nD_units = G.q == 0 ? G.nb : 0;
    }
    const uint32_t M = G.M;
    const uint64_t unit_elems = (uint64_t)NT * M * M;
    uint32_t cmask;
    if (unit_elems <= CAP_WHOLE) {  // whole stored tiles per item (one 16 KiB bulk copy each)
        G.SR = M;
        G.slabs = 1;
        uint32_t U = (uint32_t)(CAP_WHOLE / unit_elems);
        if ((uint64_t)U * NT > MAX_TT)
            U = std::max<uint32_t>(1, MAX_TT / NT);
        G.U = U;
        cmask = M - 1;
    } else {
        G.U = 1;
        const uint32_t base = in_mask | (M >= 2 ? 1u : 0u);
        uint32_t SR = (uint32_t)(CAP / ((uint64_t)NT * M));
        SR = std::max<uint32_t>(SR, 1u << __builtin_popcount(base));
        SR = std::min<uint32_t>(SR, M);
        cmask = base;
        for (uint32_t b = 0; b < h->m && (uint32_t)__builtin_popcount(cmask) < ilog2(SR); ++b)
            cmask |= 1u << b;
        G.SR = SR;
        G.slabs = M / SR;
    }
    G.logU = ilog2(G.U);
    G.logSR = ilog2(G.SR);
    G.logSlabs = ilog2(G.slabs);
    G.E = G.U * NT * G.SR * M;
    G.Epad = G.U * NT * G.SR * G.Mp;
    for (uint32_t xs = 0; xs < G.SR; ++xs)
        G.xdep[xs] = (uint8_t)pdep(xs, cmask);
    for (uint32_t s = 0; s < G.slabs; ++s)
        G.sdep[s] = (uint8_t)pdep(s, (M - 1) & ~cmask);
    G.nU_items = ((G.nU_units + G.U - 1) / G.U) * G.slabs;
    // in-tile target bits as seen in slab-row (xs) coordinates
    uint32_t xs_tmask = 0;
    for (uint32_t b = 0; b < 32; ++b)
        if (in_mask >> b & 1u)
            xs_tmask |= 1u << __builtin_popcount(cmask & ((1u << b) - 1));
    G.nxb = G.SR >> G.kin;
    G.nyb = M >> G.kin;
    G.logNxb = ilog2(G.nxb);
    G.logNyb = ilog2(G.nyb);
    for (uint32_t i = 0; i < G.nxb; ++i)
        G.xb_tab[i] = (uint8_t)pdep(i, (G.SR - 1) & ~xs_tmask);
    for (uint32_t i = 0; i < G.nyb; ++i)
        G.yb_tab[i] = (uint8_t)pdep(i, (M - 1) & ~in_mask);
    for (uint32_t r = 0; r < (1u << G.kin); ++r) {
        G.xs_in[r] = (uint8_t)pdep(r, xs_tmask);
        G.y_in[r] = (uint8_t)pdep(r, in_mask);
    }
    for (uint32_t xs = 0; xs < G.SR; ++xs) {
        G.xs_rin[xs] = (uint8_t)pext(xs, xs_tmask);
        G.xs_base[xs] = (uint8_t)(xs & ~xs_tmask);
    }
    for (uint32_t y = 0; y < M; ++y) {
        G.y_cin[y] = (uint8_t)pext(y, in_mask);
        G.y_base[y] = (uint8_t)(y & ~in_mask);
    }
    const uint32_t D = G.D, kinm = (1u << G.kin) - 1, NG = 1u << g;
    for (uint32_t rho = 0; rho < D; ++rho)
        for (uint32_t gam = 0; gam < D; ++gam) {
            const uint32_t R = rho >> G.kin, C = gam >> G.kin;
            G.comp_off[rho * D + gam] =
                (uint16_t)(((R * NG + C) * G.SR + G.xs_in[rho & kinm]) * G.Mp + G.y_in[gam & kinm]);
        }
    G.active = NT >= 64 ? ~0ull : ((1ull << NT) - 1);
    // path D
    G.nbase = M >> G.kin;
    G.nblkD = (uint64_t)G.nbase * (G.nbase + 1) / 2;
    G.BPI = std::max<uint32_t>(1, CAPD / (D * D));
    G.itemsD = (uint32_t)((G.nblkD + G.BPI - 1) / G.BPI);
    G.nD_items = G.nD_units * G.itemsD;
    // pipelined path U
    // whole tiles keep their stored orientation unpadded (the diagonal lane mapping of the
    // transform keeps both orientations bank-conflict free); slabs pad adjoint rows by one
    G.SRp = G.SR == M ? M : G.SR + 1;
    G.TS = G.SR * M + (G.SRp == G.SR ? 0 : M);
    G.diag_map = (G.nxb >= 8 && G.nyb >= 8) ? 1 : 0;
    G.PD = M;
    G.logical = 0;
    G.nruns = 0;
    for (uint32_t xs = 0; xs < G.SR; ++xs) {
        if (xs == 0 || G.xdep[xs] != G.xdep[xs - 1] + 1) {
            G.run_xs[G.nruns] = (uint8_t)xs;
            G.run_len[G.nruns] = 0;
            ++G.nruns;
        }
        ++G.run_len[G.nruns - 1];
    }
    for (uint32_t rho = 0; rho < D; ++rho)
        for (uint32_t gam = 0; gam < D; ++gam) {
            const uint32_t R = rho >> G.kin, C = gam >> G.kin, i = rho * D + gam;
            const uint32_t xs = G.xs_in[rho & kinm], y = G.y_in[gam & kinm];
            G.ttr[i] = (uint8_t)(R * NG + C);
            G.cdir[i] = (uint16_t)((R * NG + C) * G.TS + xs * M + y);
            G.cadj[i] = (uint16_t)((R * NG + C) * G.TS + y * G.SRp + xs);
        }
    G.A = NT;
    for (uint32_t t = 0; t < 64; ++t)
        G.slot[t] = (uint8_t)t;
    G.stage_elems = ((G.U << G.logNT) * G.TS + 7) & ~7u;
    const uint32_t budget = 200u * 1024u / 16u;  // elements of shared memory for the ring
    G.stages = std::min<uint32_t>(MAX_STAGES, budget / G.stage_elems);
    (void)extra_buffers;
}

// Tile permutations (all targets are grid bits, kin == 0): every component is a whole logical tile,
// so each unit splits into independent groups of <= 4 tiles closed under the permutation's cycles
// (G.gmask, host-built).  Whole stored tiles are staged (one 16 KiB bulk copy each); a tile's slot is
// its rank within its group, so one component-offset table serves every group.
void plan_grouped(Geo& G) {
    const uint32_t M = G.M, NT = 1u << G.logNT;
    G.SR = M;
    G.logSR = G.logM;
    G.slabs = 1;
    G.logSlabs = 0;
    G.U = 1;
    G.logU = 0;
    for (uint32_t i = 0; i < 32; ++i) {
        G.xdep[i] = (uint8_t)(i < M ? i : 0);
        G.xb_tab[i] = G.yb_tab[i] = (uint8_t)(i < M ? i : 0);
    }
    G.sdep[0] = 0;
    G.nruns = 1;
    G.run_xs[0] = 0;
    G.run_len[0] = (uint8_t)M;
    G.nxb = G.nyb = M;
    G.logNxb = G.logNyb = G.logM;
    for (uint32_t r = 0; r < 8; ++r)
        G.xs_in[r] = G.y_in[r] = 0;
    G.SRp = M;
    G.PD = M;
    G.logical = 0;
    G.TS = M * M;
    uint32_t A = 1;
    for (uint32_t gi = 0; gi < G.groups; ++gi) {
        uint32_t r = 0;
        for (uint32_t t = 0; t < NT; ++t)
            if ((G.gmask[gi] >> t) & 1ull)
                G.slot[t] = (uint8_t)r++;
        A = std::max(A, r);
    }
    G.A = A;
    const uint32_t D = G.D, NG = 1u << G.g;
    for (uint32_t rho = 0; rho < D; ++rho)
        for (uint32_t gam = 0; gam < D; ++gam) {
            const uint32_t i = rho * D + gam;
            G.ttr[i] = (uint8_t)(rho * NG + gam);
            G.cdir[i] = G.cadj[i] = (uint16_t)(G.slot[G.ttr[i]] * G.TS);
        }
    G.diag_map = (M >= 8) ? 1 : 0;
    // diagonal units alias logical (R, C) and (C, R) across groups: they stay on the wedge path
    G.pipe_diag = 0;
    G.nU_units = G.nU_strict;
    G.nU_items = G.nU_units * G.groups;
    G.stage_elems = (A * G.TS + 7) & ~7u;
    const uint32_t budget = 200u * 1024u / 16u;
    G.stages = std::min<uint32_t>(MAX_STAGES, budget / G.stage_elems);
}

// Monomials leave whole logical tiles untouched (a phase on a grid qubit: half of them): stage only
// the active ones, packed, and put more units in an item so each item still moves ~64 KiB.
void compact_pipe(Geo& G) {
    const uint32_t NT = 1u << G.logNT;
    const uint64_t all = NT >= 64 ? ~0ull : ((1ull << NT) - 1);
    if ((G.active & all) == all || G.SR != G.M)
        return;
    uint32_t A = 0;
    for (uint32_t t = 0; t < NT; ++t)
        G.slot[t] = (G.active >> t) & 1ull ? (uint8_t)A++ : 0;
    if (A == 0)
        return;
    G.A = A;
    const uint32_t kinm = (1u << G.kin) - 1, D = G.D;
    for (uint32_t rho = 0; rho < D; ++rho)
        for (uint32_t gam = 0; gam < D; ++gam) {
            const uint32_t i = rho * D + gam, sl = G.slot[G.ttr[i]];
            const uint32_t xs = G.xs_in[rho & kinm], y = G.y_in[gam & kinm];
            G.cdir[i] = (uint16_t)(sl * G.TS + xs * G.M + y);
            G.cadj[i] = (uint16_t)(sl * G.TS + y * G.SRp + xs);
        }
    const uint64_t unit_elems = (uint64_t)A * G.M * G.M;
    uint32_t U = 1;
    while ((uint64_t)(2 * U) * unit_elems <= CAP_WHOLE && (2 * U) * NT <= MAX_TT && 2 * U <= MAX_UA)
        U *= 2;
    G.U = U;
    G.logU = ilog2(U);
    G.nU_items = (G.nU_units + U - 1) / U;
    G.nxb = G.M >> G.kin;  // unchanged block structure; only the unit count per item moves
    G.stage_elems = ((uint32_t)(U * unit_elems) + 7) & ~7u;
    const uint32_t budget = 200u * 1024u / 16u;
    G.stages = std::min<uint32_t>(MAX_STAGES, budget / G.stage_elems);
}

size_t smem_bytes(const Geo& G, int buffers) {
    const size_t u = (size_t)G.Epad * buffers, d = (size_t)G.BPI * G.D * G.D * buffers;
    return (std::max(u, d) + (buffers == 3 ? 64 : 0)) * sizeof(double2);
}


// Geometry of the gather kernel for an operation whose units do not fit whole (g >= 2).
void plan_gather(Geo& G, bool dmma = false) {
    const uint32_t M = G.M, g = G.g, NT = 1u << (2 * g), NG = 1u << g, kin = G.kin;
    const uint32_t in_mask = G.in_mask;
    uint32_t S0 = 1;
    while (NT * (2 * S0) * (2 * S0) <= 4096 && 2 * S0 <= M)
        S0 *= 2;
    S0 = std::max<uint32_t>(S0, 1u << __builtin_popcount(in_mask));
    S0 = std::min<uint32_t>(S0, M);
    uint32_t cmask = in_mask;
    for (uint32_t b = 0; b < G.m && (uint32_t)__builtin_popcount(cmask) < ilog2(S0); ++b)
        cmask |= 1u << b;
    G.S0 = S0;
    G.logS0 = ilog2(S0);
    G.nsb_side = M / S0;
    G.log_nsb_side = ilog2(G.nsb_side);
    for (uint32_t i = 0; i < 32; ++i)
        G.xdep[i] = i < S0 ? (uint8_t)pdep(i, cmask) : 0;
    for (uint32_t b = 0; b < 32; ++b)
        G.sdep[b] = b < G.nsb_side ? (uint8_t)pdep(b, (M - 1) & ~cmask) : 0;
    uint32_t xs_tmask = 0;
    for (uint32_t b = 0; b < 32; ++b)
        if (in_mask >> b & 1u)
            xs_tmask |= 1u << __builtin_popcount(cmask & ((1u << b) - 1));
    G.SR = S0;
    G.logSR = G.logS0;
    G.nxb = G.nyb = S0 >> kin;
    G.logNxb = G.logNyb = ilog2(G.nxb);
    for (uint32_t i = 0; i < 32; ++i)
        G.xb_tab[i] = G.yb_tab[i] = i < G.nxb ? (uint8_t)pdep(i, (S0 - 1) & ~xs_tmask) : 0;
    for (uint32_t r = 0; r < 8; ++r)
        G.xs_in[r] = G.y_in[r] = r < (1u << kin) ? (uint8_t)pdep(r, xs_tmask) : 0;
    G.PD = S0 + 1;
    G.SRp = S0 + 1;
    G.logical = 1;
    G.TS = S0 * (S0 + 1);
    const uint32_t D = G.D, kinm = (1u << kin) - 1;
    for (uint32_t t = 0; t < 64; ++t)
        G.tsk[t] = 0;
    auto tables = [&]() {
        for (uint32_t rho = 0; rho < D; ++rho)
            for (uint32_t gam = 0; gam < D; ++gam) {
                const uint32_t R = rho >> kin, C = gam >> kin, i = rho * D + gam, t = R * NG + C;
                G.ttr[i] = (uint8_t)t;
                G.cdir[i] = G.cadj[i] =
                    (uint16_t)(t * G.TS + G.tsk[t] + G.xs_in[rho & kinm] * G.PD + G.y_in[gam & kinm]);
            }
    };
    tables();
    uint32_t extra = 0;
    if (dmma && D == 8) {
        // the DMMA transform's lane patterns (load B[2c+j][g], store Z[g][2c+j]) hit 16-byte bank
        // groups (addr mod 8) by component offset: pick a tile pitch and per-tile-row skew that
        // spread every quarter-warp over 8 groups
        const uint32_t TS0 = G.TS;
        uint32_t best = ~0u, bestE = 0, bestS = 0;
        for (uint32_t e = 0; e < 8; ++e)
            for (uint32_t sk = 0; sk < 8; ++sk) {
                G.TS = TS0 + e;
                for (uint32_t t = 0; t < NT; ++t)
                    G.tsk[t] = (uint8_t)((sk * (t >> g)) & 7u);
                tables();
                uint32_t cost = 0;
                for (int pat = 0; pat < 2; ++pat)
                    for (uint32_t j = 0; j < 2; ++j)
                        for (uint32_t ph = 0; ph < 4; ++ph) {
                            uint32_t cnt[8] = {0}, mx = 0;
                            for (uint32_t l = 8 * ph; l < 8 * ph + 8; ++l) {
                                const uint32_t gq = l >> 2, cq = l & 3;
                                const uint32_t i = pat ? gq * 8 + 2 * cq + j : (2 * cq + j) * 8 + gq;
                                mx = std::max(mx, ++cnt[G.cdir[i] & 7u]);
                            }
                            cost += mx;
                        }
                cost = cost * 64 + e + sk;  // ties: the smallest footprint
                if (cost < best) {
                    best = cost;
                    bestE = e;
                    bestS = sk;
                }
            }
        G.TS = TS0 + bestE;
        for (uint32_t t = 0; t < NT; ++t)
            G.tsk[t] = (uint8_t)((bestS * (t >> g)) & 7u);
        tables();
        extra = 7;
    }
    G.diag_map = (G.nxb >= 8 && G.nyb >= 8) ? 1 : 0;
    G.U = 1;
    G.logU = 0;
    G.stage_elems = (NT * G.TS + extra + 7) & ~7u;
    G.stages = 3;
    G.nG_items = G.nU_strict << (2 * G.log_nsb_side);
}

int sm_count(int device) {
    static int cache[64] = {0};
    if (device < 0 || device >= 64)
        return 148;
    if (!cache[device]) {
        int v = 0;
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device) != cudaSuccess || v <= 0)
            v = 148;
        cache[device] = v;
    }
    return cache[device];
}

template <int K, int MODE, int NS>
int launch_impl(hs_state* h, const Geo& G0, const Coef<NS>& cf, const KrausArgs& ka, int buffers) {
    const bool peer = G0.cmask && h->peer_mode;
    if (peer) {
        for (uint32_t d = 1; d < 32; ++d)
            if (!(d & ~G0.cmask) && !h->peer_buf[h->shard ^ d][h->flip])
                return set_err(HS_ERR_INVALID, "peer mode: a group member's buffers are not registered");
    } else if (G0.cmask && (!h->recv || (G0.cmask & ~h->recv_mask) ||
                            h->recv_slots < (1u << __builtin_popcount(h->recv_mask)) - 1))
        return set_err(HS_ERR_INVALID, "cross-shard operation: exchange with the group's shards first");
    Geo G = G0;
    if (peer) {
        // read the group members' current payloads where they lie, write ours into the other
        // buffer (the members read our current one concurrently); slots follow the op's own mask
        G.xmask = G.cmask;
        G.nx = 0;
        for (uint32_t b = 0; b < 32 && G.nx < 3; ++b)
            if (G.xmask >> b & 1u)
                G.xb[G.nx++] = b;
        for (uint32_t j = 0; j < 7; ++j)
            G.rbase[j] = nullptr;
        for (uint32_t d = 1; d < 32; ++d) {
            if (d & ~G.cmask)
                continue;
            uint32_t slot = 0, i = 0;
            for (uint32_t b = 0; b < 32; ++b)
                if (G.cmask >> b & 1u)
                    slot |= ((d >> b) & 1u) << i++;
            G.rbase[slot - 1] = h->peer_buf[h->shard ^ d][h->flip];
        }
        G.out = h->buf[h->flip ^ 1];
        if (MODE == M_MONO || MODE == M_KRAUS)  // tiles a monomial leaves untouched must carry over
            CUDA_TRY(cudaMemcpyAsync(G.out, h->d, h->count * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream));
    } else if (G.cmask) {  // exchange-slot layout of the last exchange (it may cover more bits than needed)
        G.xmask = h->recv_mask;
        G.nx = 0;
        for (uint32_t b = 0; b < 32 && G.nx < 3; ++b)
            if (G.xmask >> b & 1u)
                G.xb[G.nx++] = b;
        for (uint32_t j = 0; j < 7; ++j)
            G.rbase[j] = j < h->recv_slots ? h->recv + (uint64_t)j * h->recv_count : nullptr;
    }
    G.rev = (uint32_t)(h->sweeps++ & 1u);
    G.dbg = 0;
    if (MODE == M_MONO && G.groups) {
        // tile permutation on >= 2 grid bits: whole-tile pipeline, items = (unit, cycle group);
        // diagonal units through the slab kernel's wedge path
        cudaError_t e;
        if (G.nD_items) {
            Geo Gs = G;
            Gs.nU_items = 0;
            Gs.Epad = 0;
            const size_t smem = smem_bytes(Gs, buffers);
            auto kd = conj_kernel<K, MODE, NS>;
            e = cudaFuncSetAttribute(kd, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
            kd<<<(unsigned)G.nD_items, NTHR, smem, h->stream>>>(Gs, cf, ka, h->d);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("conj_kernel launch: ") + cudaGetErrorString(e));
        }
        plan_grouped(G);
        const size_t smem = (size_t)G.stages * G.stage_elems * sizeof(double2);
        auto kern = pipe_kernel<K, MODE, NS>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(pipe): ") + cudaGetErrorString(e));
        if (G.nU_items) {
            const uint64_t grid = std::min<uint64_t>(G.nU_items, (uint64_t)sm_count(h->device));
            kern<<<(unsigned)grid, NTHR_PIPE, smem, h->stream>>>(G, cf, h->d);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("pipe_kernel launch: ") + cudaGetErrorString(e));
        }
        return HS_OK;
    }
    if (MODE != M_KRAUS && ((G.g >= 2 && G.slabs > 1) || (K == 3 && MODE == M_DIRECT && G.g == 1))) {
        // units of 16 / 64 stored tiles (and k = 3 unitaries on one grid bit, whose 4-tile units
        // are whole gather items for the FP64 tensor transform): sub-block gather kernel for the
        // off-diagonal units, the slab kernel's wedge path for the diagonal ones
        cudaError_t e;
        if (G.nD_items && MODE != M_PROG) {  // grid programs: diagonal units inside the gather
            Geo Gs = G;
            Gs.nU_items = 0;
            Gs.Epad = 0;
            const size_t smem = smem_bytes(Gs, buffers);
            auto kern = conj_kernel<K, MODE, NS>;
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
            kern<<<(unsigned)G.nD_items, NTHR, smem, h->stream>>>(Gs, cf, ka, h->d);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("conj_kernel launch: ") + cudaGetErrorString(e));
        }
        Geo Gg = G;
        constexpr bool dmma = K == 3 && MODE == M_DIRECT;
        plan_gather(Gg, dmma);
        {
            static const char* dbg = getenv("HS_DEBUG_FLAGS");
            Gg.dbg = dbg ? (uint32_t)atoi(dbg) : 0u;
        }
        if constexpr (MODE == M_PROG) {
            // grid program: every unit including the diagonal ones (logical (R, C), R < C, of a
            // diagonal unit is a read-only staged copy of stored (C, R), never written back)
            Gg.ws_diag = 1;
            Gg.nG_items = Gg.nU_loose << (2 * Gg.log_nsb_side);
            const size_t smem = (size_t)Gg.stages * Gg.stage_elems * sizeof(double2);
            auto kw = gather_ws_kernel<K, NS, M_PROG>;
            e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(gather_ws): ") + cudaGetErrorString(e));
            const uint64_t grid = std::min<uint64_t>(Gg.nG_items, (uint64_t)sm_count(h->device));
            kw<<<(unsigned)grid, 768, smem, h->stream>>>(Gg, cf, h->d);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("gather_ws_kernel launch: ") + cudaGetErrorString(e));
            return HS_OK;
        }
        if (Gg.nG_items) {
            const size_t smem = (size_t)Gg.stages * Gg.stage_elems * sizeof(double2);
            // tensor-core transform in the warp-specialised kernel (bit 5: the ping-pong kernel instead);
            // k = 2 pairs blocks two by two in each direction
            if constexpr (K == 3 ? dmma : (K == 2 && MODE == M_DIRECT)) {
                if (!(Gg.dbg & 32u) && (K == 3 || (Gg.nxb >= 2 && Gg.nyb >= 2 && Gg.kin == 0))) {
                    auto kw = gather_ws_kernel<K, NS>;
                    e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
                    if (e != cudaSuccess)
                        return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(gather_ws): ") + cudaGetErrorString(e));
                    const uint64_t grid = std::min<uint64_t>(Gg.nG_items, (uint64_t)sm_count(h->device));
                    kw<<<(unsigned)grid, 768, smem, h->stream>>>(Gg, cf, h->d);
                    g_launches.fetch_add(1, std::memory_order_relaxed);
                    e = cudaGetLastError();
                    if (e != cudaSuccess)
                        return set_err(HS_ERR_CUDA, std::string("gather_ws_kernel launch: ") + cudaGetErrorString(e));
                    return HS_OK;
                }
            }
            constexpr int NC = 512;  // two groups of 256 (a multiple of the S0^2 positions of an item)
            auto kern = gather_kernel<K, MODE, NS, NC>;
            e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(gather): ") + cudaGetErrorString(e));
            const uint64_t grid = std::min<uint64_t>(Gg.nG_items, (uint64_t)sm_count(h->device));
            kern<<<(unsigned)grid, NC, smem, h->stream>>>(Gg, cf, h->d);
            g_launches.fetch_add(1, std::memory_order_relaxed);
            e = cudaGetLastError();
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("gather_kernel launch: ") + cudaGetErrorString(e));
        }
        return HS_OK;
    }
    const bool pipe = MODE != M_KRAUS && G.stages >= 3 && (G.nU_items > 0 || G.nD_items > 0);
    if (pipe && G.g >= 1 && G.slabs == 1) {
        // whole-unit items: the pipeline handles the diagonal base pairs as well
        G.pipe_diag = 1;
        G.nU_units = G.nU_loose;
        G.nU_items = (G.nU_units + G.U - 1) / G.U;
        G.nD_items = 0;
    }
    if (pipe)
        compact_pipe(G);
    cudaError_t e;
    // slab kernel: diagonal units (path D) and, when the pipeline does not apply, path U too
    const uint64_t nU_slab = pipe ? 0 : G.nU_items;
    const uint64_t items = G.nD_items + nU_slab;
    if (items) {
        Geo Gs = G;
        Gs.nU_items = nU_slab;
        if (!nU_slab)
            Gs.Epad = 0;  // diagonal units only: size shared memory for path D alone
        const size_t smem = smem_bytes(Gs, buffers);
        auto kern = conj_kernel<K, MODE, NS>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute: ") + cudaGetErrorString(e));
        const uint64_t gx = std::min<uint64_t>(items, 1u << 30);
        const uint64_t gy = (items + gx - 1) / gx;
        kern<<<dim3((unsigned)gx, (unsigned)gy), NTHR, smem, h->stream>>>(Gs, cf, ka, h->d);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("conj_kernel launch: ") + cudaGetErrorString(e));
    }
    if (pipe && G.nU_items > 0) {
        const size_t smem = (size_t)G.stages * G.stage_elems * sizeof(double2);
        auto kern = pipe_kernel<K, MODE, NS>;
        e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(pipe): ") + cudaGetErrorString(e));
        const uint64_t grid = std::min<uint64_t>(G.nU_items, (uint64_t)sm_count(h->device));
        kern<<<(unsigned)grid, NTHR_PIPE, smem, h->stream>>>(G, cf, h->d);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("pipe_kernel launch: ") + cudaGetErrorString(e));
    }
    return HS_OK;
}

// One operation's kernels.  Peer mode: the result went to the other buffer, which becomes current.
template <int K, int MODE, int NS>
int launch(hs_state* h, const Geo& G0, const Coef<NS>& cf, const KrausArgs& ka, int buffers) {
    const int rc = launch_impl<K, MODE, NS>(h, G0, cf, ka, buffers);
    if (rc == HS_OK && G0.cmask && h->peer_mode) {
        h->flip ^= 1u;
        h->d = h->buf[h->flip];
    }
    return rc;
}

// Subcase counters (SubcaseCounters, kernels.hpp:29-41) for the cross/mixed engines: A = unit
// whose logical tiles are all stored directly, B = some logical tile is an adjoint, C =
// diagonal base pair.  Counted on the host by the closed form (k = 1) or by enumeration.
void count_subcases(const hs_state* h, const Geo& G, uint64_t* sub) {
    sub[0] = sub[1] = sub[2] = 0;
    if (G.g == 0)
        return;
    const uint64_t nb = G.nb;
    sub[2] = nb;
    if (G.k == 1) {  // B = (G/2)(2^a' - 1)/2
        const uint64_t P = nb * (nb + 1) / 2;
        const uint64_t B = nb * ((1ull << G.gr_pos[0]) - 1) / 2;
        sub[1] = B;
        sub[0] = P - B - nb;
        return;
    }
    // generic: a unit is "adjoint" when some logical tile lies in the upper triangle
    auto ins = [&](uint64_t s, uint32_t a) {
        for (uint32_t l = 0; l < G.g; ++l) {
            const uint32_t p = G.gr_pos[l];
            const uint64_t right = s & ((1ull << p) - 1);
            s = ((((s >> p) << 1) | ((a >> l) & 1u)) << p) | right;
        }
        return s;
    };
    const uint32_t NG = 1u << G.g;
    uint64_t a = 0, b = 0;
    for (uint64_t tbi = 1; tbi < nb; ++tbi) {
        // the max column index of a unit is tc[NG-1], the min row index tr[0]
        const uint64_t tr0 = ins(tbi, 0);
        for (uint64_t tbj = 0; tbj < tbi; ++tbj) {
            if (tr0 >= ins(tbj, NG - 1))
                ++a;
            else
                ++b;
        }
    }
    if (G.k == 2 && G.g == 1) {
        // tiled_two_mixed counts per (ti, tj) the single t01 tile test (kernels.cpp:379-387)
        sub[0] = a;
        sub[1] = b;
        return;
    }
    sub[0] = a;
    sub[1] = b;
}

int finish_plan(hs_state* h, const Geo& G, int k, const uint32_t* t, int path, hs_plan* plan, uint64_t touched) {
    if (!plan)
        return HS_OK;
    std::memset(plan, 0, sizeof(*plan));
    plan->path = path;
    plan->k = k;
    for (int i = 0; i < k; ++i)
        plan->targets[i] = t[i];
    plan->grid_bits = (int)G.g;
    plan->launches = (G.nD_items + G.nU_items) ? 1 : 0;
    // a cross-shard op also reads the 2^cross - 1 exchanged payloads of its group (about one shard each)
    plan->touched_bytes = G.cmask ? touched / 2 * ((1ull << __builtin_popcount(G.cmask)) + 1) : touched;
    if (g_plan_subcases)
        count_subcases(h, G, plan->subcases);
    return HS_OK;
}

uint64_t state_bytes(const hs_state* h) { return h->count * sizeof(double2); }

int generic_path(const Geo& G) {
    if (G.g == 0)
        return HS_PATH_TILED_INTRA;
    if (G.g == G.k)
        return HS_PATH_TILED_CROSS;
    return HS_PATH_TILED_MIXED;
}

}  // namespace

// ================================================================================ C-ABI
extern "C" {

const char* hs_last_error(void) { return g_err.c_str(); }
int hs_set_plan_subcases(int enable) {
    g_plan_subcases = enable != 0;
    return HS_OK;
}
const char* hs_version(void) { return "hermsim_b200 0.1 (sm_100a)"; }
uint64_t hs_launch_count(void) { return g_launches.load(); }

int hs_device_count(int* out) {
    if (!out)
        return set_err(HS_ERR_INVALID, "null out");
    CUDA_TRY(cudaGetDeviceCount(out));
    return HS_OK;
}

int hs_state_create_sharded(int n, int m, int device, int nshards, int shard, hs_state** out) {
    if (!out)
        return set_err(HS_ERR_INVALID, "null out");
    *out = nullptr;
    if (n < 1 || n > 30)
        return set_err(HS_ERR_INVALID, "qubit count must be in [1, 30]");
    if (m < 0 || m > n + 2)
        return set_err(HS_ERR_INVALID, "tile exponent must be in [0, n + 2]");
    if (m > 5)
        return set_err(HS_ERR_UNSUPPORTED, "this build supports tile exponents m <= 5");
    const uint64_t Gt = (1ull << n) >= (1ull << m) ? (1ull << n) >> m : 1;
    if (nshards < 1 || (nshards & (nshards - 1)) || (uint64_t)nshards > Gt)
        return set_err(HS_ERR_INVALID, "shard count must be a power of two <= tiles per grid row");
    if (shard < 0 || shard >= nshards)
        return set_err(HS_ERR_RANGE, "shard index out of range");
    int ndev = 0;
    CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev)
        return set_err(HS_ERR_RANGE, "device index out of range");
    DeviceGuard dg(device);
    auto* h = new hs_state();
    h->n = n;
    h->m = m;
    h->device = device;
    h->N = 1ull << n;
    h->M = 1ull << m;
    h->G = h->N >= h->M ? h->N / h->M : 1;
    h->Plog = ilog2((uint64_t)nshards);
    h->shard = (uint32_t)shard;
    h->logB = ilog2(h->G) - h->Plog;
    {
        const uint64_t B = 1ull << h->logB, P = (uint64_t)nshards;
        const uint64_t tiles = shard == 0 ? P * (B * (B + 1) / 2) : (P / 2) * B * B;
        h->count = tiles * h->M * h->M;
    }
    cudaError_t e = cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete h;
        return set_err(HS_ERR_CUDA, cudaGetErrorString(e));
    }
    h->own_stream = true;
    e = cudaMalloc(&h->d, h->count * sizeof(double2));
    if (e != cudaSuccess) {
        cudaStreamDestroy(h->stream);
        delete h;
        cudaGetLastError();
        return set_err(HS_ERR_NOMEM, std::string("cudaMalloc state: ") + cudaGetErrorString(e));
    }
    e = cudaMalloc(&h->red, (2 * RED_BLOCKS + 8) * sizeof(double));
    if (e == cudaSuccess)
        e = cudaMemsetAsync(h->d, 0, h->count * sizeof(double2), h->stream);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(h->stream);
    if (e != cudaSuccess) {
        cudaFree(h->d);
        cudaFree(h->red);
        cudaStreamDestroy(h->stream);
        delete h;
        return set_err(HS_ERR_CUDA, cudaGetErrorString(e));
    }
    *out = h;
    return HS_OK;
}

int hs_state_create(int n, int m, int device, hs_state** out) {
    return hs_state_create_sharded(n, m, device, 1, 0, out);
}

int hs_state_free(hs_state* h) {
    if (!h)
        return HS_OK;
    DeviceGuard dg(h->device);
    cudaStreamSynchronize(h->stream);
    if (h->peer_mode) {
        cudaFree(h->buf[0]);
        cudaFree(h->buf[1]);
    } else {
        cudaFree(h->d);
    }
    cudaFree(h->red);
    cudaFree(h->kraus);
    cudaFree(h->recv);
    if (h->comm && nccl().CommDestroy)
        nccl().CommDestroy((ncclComm_t)h->comm);
    if (h->own_stream)
        cudaStreamDestroy(h->stream);
    delete h;
    return HS_OK;
}

int hs_state_info(const hs_state* h, int* n, int* m, uint64_t* count, uint64_t* grid) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (n)
        *n = h->n;
    if (m)
        *m = h->m;
    if (count)
        *count = h->count;
    if (grid)
        *grid = h->G;
    return HS_OK;
}

int hs_state_shard_info(const hs_state* h, int* nshards, int* shard, uint64_t* block_rows) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (nshards)
        *nshards = 1 << h->Plog;
    if (shard)
        *shard = (int)h->shard;
    if (block_rows)
        *block_rows = 1ull << h->logB;
    return HS_OK;
}

namespace {
// the op's cross-shard mask: shard bit c set when a target is the c-th top qubit
int op_group_mask(const hs_state* h, int k, const uint32_t* targets, uint32_t* mask) {
    if (!h || !targets || !mask || k < 1 || k > 3)
        return set_err(HS_ERR_INVALID, "bad arguments");
    *mask = 0;
    for (int i = 0; i < k; ++i)
        if (targets[i] >= (uint32_t)h->n)
            return set_err(HS_ERR_RANGE, "target qubit out of range");
    if (!h->Plog)
        return HS_OK;
    const uint32_t gbits = ilog2(h->G), top0 = h->m + gbits - h->Plog;  // qubit index of the lowest top bit
    for (int i = 0; i < k; ++i)
        if (targets[i] >= top0)
            *mask |= 1u << (targets[i] - top0);
    return HS_OK;
}
// slot of group member `shard ^ d` in the exchange buffer (the bits of d under mask, packed, minus 1)
uint32_t group_slot(uint32_t d, uint32_t mask) {
    uint32_t slot = 0, i = 0;
    for (uint32_t b = 0; b < 32; ++b)
        if (mask >> b & 1u)
            slot |= ((d >> b) & 1u) << i++;
    return slot - 1;
}
}  // namespace

int hs_op_group(const hs_state* h, int k, const uint32_t* targets, uint32_t* mask) {
    return op_group_mask(h, k, targets, mask);
}

int hs_op_partner(const hs_state* h, int k, const uint32_t* targets, int* partner) {
    if (!partner)
        return set_err(HS_ERR_INVALID, "bad arguments");
    *partner = -1;
    uint32_t mask = 0;
    int rc = op_group_mask(h, k, targets, &mask);
    if (rc)
        return rc;
    if (mask & (mask - 1))
        return set_err(HS_ERR_UNSUPPORTED, "operation couples more than one cross-shard qubit: use hs_op_group");
    if (mask)
        *partner = (int)(h->shard ^ mask);
    return HS_OK;
}

int hs_state_recv_reserve(hs_state* h, int slots) {
    if (!h || slots < 1 || slots > 7)
        return set_err(HS_ERR_INVALID, "bad arguments");
    if (h->recv && h->recv_slots >= (uint32_t)slots)
        return HS_OK;
    DeviceGuard dg(h->device);
    if (h->recv) {
        cudaStreamSynchronize(h->stream);
        cudaFree(h->recv);
        h->recv = nullptr;
        h->recv_slots = 0;
        h->recv_mask = 0;
    }
    const uint64_t cnt = shard_count_of(h, 0);  // the largest shard
    cudaError_t e = cudaMalloc(&h->recv, (uint64_t)slots * cnt * sizeof(double2));
    if (e != cudaSuccess) {
        cudaGetLastError();
        h->recv = nullptr;
        return set_err(HS_ERR_NOMEM, std::string("cudaMalloc exchange buffer: ") + cudaGetErrorString(e));
    }
    h->recv_count = cnt;
    h->recv_slots = (uint32_t)slots;
    return HS_OK;
}

int hs_state_recv_alloc(hs_state* h) { return hs_state_recv_reserve(h, 1); }

// In-process / single-node exchange: slot of `peer` (group `mask`) <- peer payload (device or peer
// copy, stream-ordered).  Call once per other member of the group before the operation.
int hs_state_exchange_group_from(hs_state* h, const hs_state* peer, uint32_t mask) {
    if (!h || !peer)
        return set_err(HS_ERR_INVALID, "null state");
    if (peer->Plog != h->Plog || peer->n != h->n || peer->m != h->m)
        return set_err(HS_ERR_INVALID, "peer is not a shard of the same operator");
    const uint32_t d = peer->shard ^ h->shard;
    if (!d || (d & ~mask) || mask >> h->Plog)
        return set_err(HS_ERR_INVALID, "peer is not another member of the group");
    const int nbits = __builtin_popcount(mask);
    int rc = hs_state_recv_reserve(h, (1 << nbits) - 1);
    if (rc)
        return rc;
    DeviceGuard dg(h->device);
    double2* dst = h->recv + (uint64_t)group_slot(d, mask) * h->recv_count;
    CUDA_TRY(cudaStreamSynchronize(peer->stream));
    if (peer->device == h->device)
        CUDA_TRY(cudaMemcpyAsync(dst, peer->d, peer->count * sizeof(double2), cudaMemcpyDeviceToDevice, h->stream));
    else
        CUDA_TRY(cudaMemcpyPeerAsync(dst, h->device, peer->d, peer->device, peer->count * sizeof(double2), h->stream));
    h->recv_mask = mask;
    return HS_OK;
}

int hs_state_exchange_from(hs_state* h, const hs_state* peer) {
    if (!h || !peer)
        return set_err(HS_ERR_INVALID, "null state");
    return hs_state_exchange_group_from(h, peer, peer->shard ^ h->shard);
}

int hs_nccl_unique_id(void* id128) {
    if (!id128)
        return set_err(HS_ERR_INVALID, "null out");
    NcclApi& api = nccl();
    if (!api.GetUniqueId)
        return set_err(HS_ERR_UNSUPPORTED, "libnccl.so.2 not available");
    ncclUniqueId id;
    const ncclResult_t r = api.GetUniqueId(&id);
    if (r != ncclSuccess)
        return set_err(HS_ERR_CUDA, std::string("ncclGetUniqueId: ") + api.GetErrorString(r));
    std::memcpy(id128, &id, sizeof(id));
    return HS_OK;
}

int hs_state_comm_init(hs_state* h, const void* id128, int nranks, int rank) {
    if (!h || !id128)
        return set_err(HS_ERR_INVALID, "null argument");
    if (nranks != (1 << h->Plog) || rank != (int)h->shard)
        return set_err(HS_ERR_INVALID, "communicator ranks must be the shards (rank == shard)");
    NcclApi& api = nccl();
    if (!api.CommInitRank)
        return set_err(HS_ERR_UNSUPPORTED, "libnccl.so.2 not available");
    DeviceGuard dg(h->device);
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    ncclComm_t comm;
    const ncclResult_t r = api.CommInitRank(&comm, nranks, id, rank);
    if (r != ncclSuccess)
        return set_err(HS_ERR_CUDA, std::string("ncclCommInitRank: ") + api.GetErrorString(r));
    h->comm = comm;
    return HS_OK;
}

// NCCL exchange over NVLink within the op's group (shards s ^ span(mask)): send the whole local shard
// to every other member and receive theirs into the exchange slots; one grouped call, stream-ordered.
// One top target = a pairwise butterfly step.
int hs_state_exchange_group(hs_state* h, uint32_t mask) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (!h->comm)
        return set_err(HS_ERR_INVALID, "no communicator: call hs_state_comm_init");
    if (!mask || mask >> h->Plog || __builtin_popcount(mask) > 3)
        return set_err(HS_ERR_RANGE, "bad group mask");
    const int nbits = __builtin_popcount(mask);
    int rc = hs_state_recv_reserve(h, (1 << nbits) - 1);
    if (rc)
        return rc;
    NcclApi& api = nccl();
    DeviceGuard dg(h->device);
    ncclComm_t comm = (ncclComm_t)h->comm;
    ncclResult_t r = api.GroupStart();
    for (uint32_t d = 1; d < (1u << h->Plog) && r == ncclSuccess; ++d) {
        if (d & ~mask)
            continue;
        const int peer = (int)(h->shard ^ d);
        const uint64_t pc = shard_count_of(h, (uint32_t)peer);
        r = api.Send(h->d, h->count * 2, ncclDouble, peer, comm, h->stream);
        if (r == ncclSuccess)
            r = api.Recv(h->recv + (uint64_t)group_slot(d, mask) * h->recv_count, pc * 2, ncclDouble, peer, comm,
                         h->stream);
    }
    const ncclResult_t r2 = api.GroupEnd();
    if (r != ncclSuccess || r2 != ncclSuccess)
        return set_err(HS_ERR_CUDA, std::string("NCCL exchange: ") + api.GetErrorString(r != ncclSuccess ? r : r2));
    h->recv_mask = mask;
    return HS_OK;
}

int hs_state_exchange(hs_state* h, int partner) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (partner < 0 || partner >= (1 << h->Plog) || partner == (int)h->shard)
        return set_err(HS_ERR_RANGE, "bad partner shard");
    return hs_state_exchange_group(h, (uint32_t)partner ^ h->shard);
}

int hs_state_upload_range(hs_state* h, const double* host, uint64_t offset, uint64_t count) {
    if (!h || (!host && count))
        return set_err(HS_ERR_INVALID, "null argument");
    if (offset > h->count || count > h->count - offset)
        return set_err(HS_ERR_RANGE, "upload range exceeds the payload");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaMemcpyAsync(h->d + offset, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return HS_OK;
}

int hs_state_download_range(const hs_state* h, double* host, uint64_t offset, uint64_t count) {
    if (!h || (!host && count))
        return set_err(HS_ERR_INVALID, "null argument");
    if (offset > h->count || count > h->count - offset)
        return set_err(HS_ERR_RANGE, "download range exceeds the payload");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaMemcpyAsync(host, h->d + offset, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return HS_OK;
}

int hs_state_upload(hs_state* h, const double* host, uint64_t count) {
    if (h && count != h->count)
        return set_err(HS_ERR_INVALID, "payload length mismatch");
    return hs_state_upload_range(h, host, 0, count);
}

int hs_state_download(const hs_state* h, double* host, uint64_t count) {
    if (h && count != h->count)
        return set_err(HS_ERR_INVALID, "payload length mismatch");
    return hs_state_download_range(h, host, 0, count);
}

int hs_state_upload_async(hs_state* h, const double* host, uint64_t count) {
    if (!h || !host || count != h->count)
        return set_err(HS_ERR_INVALID, "bad upload arguments");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaMemcpyAsync(h->d, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
    return HS_OK;
}

int hs_state_download_async(const hs_state* h, double* host, uint64_t count) {
    if (!h || !host || count != h->count)
        return set_err(HS_ERR_INVALID, "bad download arguments");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaMemcpyAsync(host, h->d, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    return HS_OK;
}

int hs_state_copy(hs_state* dst, const hs_state* src) {
    if (!dst || !src)
        return set_err(HS_ERR_INVALID, "null state");
    if (dst->count != src->count || dst->m != src->m || dst->n != src->n)
        return set_err(HS_ERR_INVALID, "state shapes differ");
    DeviceGuard dg(dst->device);
    CUDA_TRY(cudaStreamSynchronize(src->stream));
    CUDA_TRY(cudaMemcpyAsync(dst->d, src->d, dst->count * sizeof(double2), cudaMemcpyDefault, dst->stream));
    CUDA_TRY(cudaStreamSynchronize(dst->stream));
    return HS_OK;
}

int hs_state_zero(hs_state* h) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaMemsetAsync(h->d, 0, h->count * sizeof(double2), h->stream));
    return HS_OK;
}

int hs_state_synchronize(const hs_state* h) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return HS_OK;
}

int hs_state_set_stream(hs_state* h, void* stream) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    if (h->own_stream)
        cudaStreamDestroy(h->stream);
    if (stream) {
        h->stream = (cudaStream_t)stream;
        h->own_stream = false;
    } else {
        CUDA_TRY(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
        h->own_stream = true;
    }
    return HS_OK;
}

void* hs_state_stream(const hs_state* h) { return h ? (void*)h->stream : nullptr; }
void* hs_state_device_ptr(hs_state* h) { return h ? (void*)h->d : nullptr; }

int hs_host_alloc(uint64_t bytes, void** out) {
    if (!out)
        return set_err(HS_ERR_INVALID, "null out");
    CUDA_TRY(cudaHostAlloc(out, bytes, cudaHostAllocPortable));
    return HS_OK;
}
int hs_host_free(void* p) {
    CUDA_TRY(cudaFreeHost(p));
    return HS_OK;
}

// ------------------------------------------------------------------------ apply entry points
int hs_apply_transfer(hs_state* h, int k, const double* s, const uint32_t* t, hs_plan* plan) {
    int rc = check_targets(h, k, t);
    if (rc)
        return rc;
    if (!s)
        return set_err(HS_ERR_INVALID, "null transfer matrix");
    if (k == 3)
        return set_err(HS_ERR_UNSUPPORTED, "k = 3 transfer matrices: use hs_apply_kraus / hs_apply_unitary");
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, k, t, G, 1);
    KrausArgs ka{nullptr, 0};
    if (k == 1) {
        Coef<16> cf{};
        std::memcpy(cf.s, s, sizeof(cf.s));
        // (00, 11) and (01, 10) are the two shard classes of a cross-shard quad (T00, T11 on one
        // shard, T01, T10 on the partner): a transfer matrix without couplings between
        // them needs no exchange, and the quad reads only class-consistent components
        bool xp = true;
        for (int r = 0; r < 4; ++r)
            for (int c = 0; c < 4; ++c)
                if (((r == 0 || r == 3) != (c == 0 || c == 3)) && (s[2 * (4 * r + c)] != 0.0 || s[2 * (4 * r + c) + 1] != 0.0))
                    xp = false;
        cf.xpat = xp ? 1u : 0u;
        if (xp)
            G.cmask = 0;
        rc = launch<1, M_S1, 16>(h, G, cf, ka, 1);
    } else {
        auto* cf = new Coef<256>();
        std::memcpy(cf->s, s, sizeof(cf->s));
        rc = launch<2, M_S2, 256>(h, G, *cf, ka, 1);
        delete cf;
    }
    if (rc)
        return rc;
    return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
}

// Fused program of nsteps (<= 8) single-qubit steps on in-tile qubits (< m), one HBM pass
// (SURVEY 8f "op fusion": a run of consecutive in-tile single-qubit operations).  kinds[p]: 0 row-
// stacked 4 x 4 transfer matrix s[16p..16p+15] (interleaved complex), 1 Hadamard, 2 diagonal
// transfer (s diagonal used).  Equivalent to applying the steps one by one (hs_apply_transfer).
int hs_apply_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s, hs_plan* plan) {
    if (!h || nsteps < 1 || nsteps > 16 || !kinds || !bits || !s)
        return set_err(HS_ERR_INVALID, "bad program");
    const uint32_t edge = std::min<uint32_t>((uint32_t)h->m, (uint32_t)h->n);
    for (int p = 0; p < nsteps; ++p) {
        if (bits[p] >= edge)
            return set_err(HS_ERR_RANGE, "program steps act on in-tile qubits (< m) only");
        if (kinds[p] < 0 || kinds[p] > 3)
            return set_err(HS_ERR_INVALID, "bad program step kind");
    }
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, 1, bits, G, 1);
    KrausArgs ka{nullptr, 0};
    auto* cf = new Coef<256>();
    std::memcpy(cf->s, s, (size_t)nsteps * 16 * sizeof(double2));
    for (int p = 0; p < nsteps; ++p) {
        cf->pbit[p] = (uint8_t)bits[p];
        cf->pkind[p] = (uint8_t)kinds[p];
    }
    cf->nsteps = (uint32_t)nsteps;
    int rc = launch<1, M_PROG, 256>(h, G, *cf, ka, 1);
    delete cf;
    if (rc)
        return rc;
    return finish_plan(h, G, 1, bits, HS_PATH_TILED_INTRA, plan, 2 * state_bytes(h));
}

// Fused grid program: one k = 1 step on each of nsteps (<= 3) distinct grid qubits
// (>= m), applied in ONE pass: the units of the g = nsteps grid bits are gathered (warp-specialised
// gather) and the steps run one after another on the staged logical tiles.  kinds / s as for
// hs_apply_program.  Single-GPU states only (a cross-shard step would need its own exchange).
int hs_apply_grid_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s,
                          hs_plan* plan) {
    if (!h || nsteps < 2 || nsteps > 3 || !kinds || !bits || !s)
        return set_err(HS_ERR_INVALID, "bad grid program (2 or 3 steps; one step: hs_apply_transfer)");
    if (h->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "grid programs run on single-GPU states");
    uint32_t t[3];
    for (int p = 0; p < nsteps; ++p) {
        if (bits[p] < (uint32_t)h->m || bits[p] >= (uint32_t)h->n)
            return set_err(HS_ERR_RANGE, "grid program steps act on grid qubits (>= m) only");
        if (kinds[p] < 0 || kinds[p] > 3)
            return set_err(HS_ERR_INVALID, "bad program step kind");
        for (int q = 0; q < p; ++q)
            if (bits[q] == bits[p])
                return set_err(HS_ERR_INVALID, "grid program: one step per qubit");
        t[p] = bits[p];
    }
    std::sort(t, t + nsteps);
    if (h->m != 5 || ((uint64_t)1 << (2 * nsteps)) * 1024 < 4096)
        return set_err(HS_ERR_UNSUPPORTED, "grid programs need 32 x 32 tiles");
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, nsteps, t, G, 1);
    auto* cf = new Coef<64>();
    for (int p = 0; p < nsteps; ++p) {
        std::memcpy(cf->s + 16 * p, s + 32 * p, 16 * sizeof(double2));
        uint32_t l = 0;
        while (t[l] != bits[p])
            ++l;
        cf->pbit[p] = (uint8_t)l;  // local grid bit of the step
        cf->pkind[p] = (uint8_t)kinds[p];
    }
    cf->nsteps = (uint32_t)nsteps;
    int rc = launch<3, M_PROG, 64>(h, G, *cf, KrausArgs{nullptr, 0}, 1);
    delete cf;
    if (rc)
        return rc;
    return finish_plan(h, G, nsteps, t, HS_PATH_TILED_CROSS, plan, 2 * state_bytes(h));
}

int hs_apply_unitary(hs_state* h, int k, const double* u, const uint32_t* t, hs_plan* plan) {
    int rc = check_targets(h, k, t);
    if (rc)
        return rc;
    if (!u)
        return set_err(HS_ERR_INVALID, "null unitary");
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, k, t, G, 1);
    KrausArgs ka{nullptr, 0};
    const double2* U = reinterpret_cast<const double2*>(u);
    if (k == 1) {
        // S = conj(U) (x) U, row-stacked (kernels.cpp:27-37 of channel.cpp:24-34)
        Coef<16> cf{};
        for (int a = 0; a < 2; ++a)
            for (int ap = 0; ap < 2; ++ap)
                for (int mu = 0; mu < 2; ++mu)
                    for (int nu = 0; nu < 2; ++nu) {
                        // row-stacked (a*2+ap, mu*2+nu) = col-stacked (a + 2ap, mu + 2nu)
                        //  = conj(U[ap][nu]) * U[a][mu]
                        const double2 x = U[ap * 2 + nu], y = U[a * 2 + mu];
                        cf.s[(a * 2 + ap) * 4 + mu * 2 + nu] =
                            make_double2(x.x * y.x + x.y * y.y, x.x * y.y - x.y * y.x);
                    }
        rc = launch<1, M_S1, 16>(h, G, cf, ka, 1);
    } else if (k == 2) {
        Coef<64> cf{};
        std::memcpy(cf.s, u, 16 * sizeof(double2));
        rc = launch<2, M_DIRECT, 64>(h, G, cf, ka, 1);
    } else {
        Coef<64> cf{};
        std::memcpy(cf.s, u, 64 * sizeof(double2));
        rc = launch<3, M_DIRECT, 64>(h, G, cf, ka, 1);
    }
    if (rc)
        return rc;
    return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
}

int hs_apply_kraus(hs_state* h, int k, int nops, const double* ops, const uint32_t* t, hs_plan* plan) {
    int rc = check_targets(h, k, t);
    if (rc)
        return rc;
    const int d = 1 << k;
    if (nops < 1 || nops > d * d || !ops)
        return set_err(HS_ERR_INVALID, "Kraus set: needs 1 .. 4^k operators");
    if (nops == 1 && k >= 2)
        return hs_apply_unitary(h, k, ops, t, plan);
    const double2* L = reinterpret_cast<const double2*>(ops);
    if (k <= 2) {
        // S = sum_a conj(L_a) (x) L_a, row-stacked
        const int dd = d * d;
        std::vector<double2> srow(dd * dd, make_double2(0.0, 0.0));
        for (int a = 0; a < nops; ++a)
            for (int r = 0; r < d; ++r)
                for (int rp = 0; rp < d; ++rp)
                    for (int c = 0; c < d; ++c)
                        for (int cp = 0; cp < d; ++cp) {
                            // out[r][rp] (block row r, col rp) += L[r][c] B[c][cp] conj(L[rp][cp])
                            const double2 x = L[a * dd + r * d + c], y = L[a * dd + rp * d + cp];
                            double2& o = srow[(r * d + rp) * dd + c * d + cp];
                            o.x += x.x * y.x + x.y * y.y;
                            o.y += x.y * y.x - x.x * y.y;
                        }
        return hs_apply_transfer(h, k, reinterpret_cast<const double*>(srow.data()), t, plan);
    }
    DeviceGuard dg(h->device);
    const size_t bytes = (size_t)nops * d * d * sizeof(double2);
    if (h->kraus_cap < bytes) {
        cudaFree(h->kraus);
        h->kraus = nullptr;
        h->kraus_cap = 0;
        CUDA_TRY(cudaMalloc(&h->kraus, bytes));
        h->kraus_cap = bytes;
    }
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(h->stream, &cs));
        if (cs != cudaStreamCaptureStatusNone)  // the upload of the Kraus set would read host memory at replay
            return set_err(HS_ERR_UNSUPPORTED, "k = 3 Kraus channels with several operators cannot be captured in a graph");
    }
    CUDA_TRY(cudaMemcpyAsync(h->kraus, ops, bytes, cudaMemcpyHostToDevice, h->stream));
    Geo G;
    plan_geo(h, k, t, G, 3);
    Coef<16> cf{};
    KrausArgs ka{h->kraus, nops};
    rc = launch<3, M_KRAUS, 16>(h, G, cf, ka, 3);
    if (rc)
        return rc;
    // the host pointer `ops` is only read by the async copy: make it safe to free
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
}

int hs_apply_hadamard(hs_state* h, uint32_t target, hs_plan* plan) {
    int rc = check_targets(h, 1, &target);
    if (rc)
        return rc;
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, 1, &target, G, 1);
    Coef<16> cf{};
    KrausArgs ka{nullptr, 0};
    rc = launch<1, M_HAD, 16>(h, G, cf, ka, 1);
    if (rc)
        return rc;
    rc = finish_plan(h, G, 1, &target, HS_PATH_NATIVE_HADAMARD, plan, 2 * state_bytes(h));
    if (plan)  // apply_hadamard reports no subcase counters (native.cpp:343-361)
        plan->subcases[0] = plan->subcases[1] = plan->subcases[2] = 0;
    return rc;
}

int hs_apply_monomial(hs_state* h, int k, const uint32_t* perm, const double* diag, const uint32_t* t,
                      hs_plan* plan) {
    int rc = check_targets(h, k, t);
    if (rc)
        return rc;
    const uint32_t D = 1u << k;
    uint32_t p[8], pinv[8];
    for (uint32_t x = 0; x < D; ++x)
        p[x] = perm ? perm[x] : x;
    for (uint32_t x = 0; x < D; ++x)
        pinv[x] = 0xff;
    for (uint32_t x = 0; x < D; ++x) {
        if (p[x] >= D || pinv[p[x]] != 0xff)
            return set_err(HS_ERR_INVALID, "permutation table is not a bijection");
        pinv[p[x]] = x;
    }
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, k, t, G, 1);
    // a monomial moves elements only along the local bits its permutation flips: remote tiles that
    // differ in a stationary top target (a diagonal phase, a control) are never read, so those
    // shards need no exchange (multigpu.op_mask mirrors this)
    {
        uint32_t moving = 0;
        for (uint32_t x = 0; x < D; ++x)
            moving |= x ^ p[x];
        if (G.cmask) {
            const uint32_t top0 = h->m + ilog2(h->G) - h->Plog;
            uint32_t need = 0;
            for (int l = 0; l < k; ++l)
                if (t[l] >= top0 && (moving >> l & 1u))
                    need |= 1u << (t[l] - top0);
            G.cmask = need;
        }
    }
    Coef<64> cf{};
    {
        bool ident = true;
        for (uint32_t x = 0; x < D; ++x)
            ident &= p[x] == x;
        cf.diag = ident ? 1u : 0u;
        cf.nib = 0;
        for (int l = 0; l < k; ++l)  // ascending bound targets: in-tile ones first
            if (t[l] < (uint32_t)h->m)
                cf.ibit[cf.nib++] = (uint8_t)t[l];
    }
    const double2* dg2 = reinterpret_cast<const double2*>(diag);
    // U = P Dg with P|x> = |p[x]>: (U B U^dag)(r, c) = d[pinv r] conj(d[pinv c]) B(pinv r, pinv c).
    // Factor exactly 1 when the two diagonal entries are identical (equal-bit elements stay
    // untouched bit-exactly, native.cpp:238-245); mirrored factors use f(c, r) = conj(f(r, c))
    // as the reference's f01 = conj(f10) (native.cpp:251-252).
    for (uint32_t r = 0; r < D; ++r)
        for (uint32_t c = 0; c < D; ++c) {
            const uint32_t i = r * D + c;
            cf.pinv[r] = (uint8_t)pinv[r];
            double2 a = dg2 ? dg2[pinv[r]] : make_double2(1.0, 0.0);
            double2 b = dg2 ? dg2[pinv[c]] : make_double2(1.0, 0.0);
            if (a.x == b.x && a.y == b.y) {
                cf.s[i] = make_double2(1.0, 0.0);
                cf.fone |= 1ull << i;
            } else if (r < c) {
                // f(r, c) = conj(f(c, r)) with f(c, r) = b * conj(a) ... computed below
                std::swap(a, b);
                const double2 f = make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);
                cf.s[i] = make_double2(f.x, -f.y);
            } else {
                cf.s[i] = make_double2(a.x * b.x + a.y * b.y, a.y * b.x - a.x * b.y);  // a * conj(b)
            }
        }
    // cycles of the component map c = (r, c') -> src(c) = (pinv r, pinv c') for the in-place
    // transform; fixed components with factor exactly 1 are left out (never touched)
    {
        bool seen[64] = {false};
        uint32_t pos = 0;
        cf.ncyc = 0;
        cf.cyc_off[0] = 0;
        for (uint32_t c0 = 0; c0 < D * D; ++c0) {
            if (seen[c0])
                continue;
            uint32_t len = 0, c = c0;
            do {
                seen[c] = true;
                cf.cyc[pos + len++] = (uint8_t)c;
                c = pinv[c / D] * D + pinv[c % D];
            } while (c != c0);
            if (len == 1 && ((cf.fone >> c0) & 1ull))
                continue;  // untouched element
            pos += len;
            cf.cyc_off[++cf.ncyc] = (uint8_t)pos;
        }
    }
    // logical tiles whose components all stay in place with factor 1 are skipped entirely
    const uint32_t NG = 1u << G.g, kin = G.kin, KI = 1u << kin;
    uint64_t active = 0;
    for (uint32_t R = 0; R < NG; ++R)
        for (uint32_t C = 0; C < NG; ++C) {
            bool moves = false;
            for (uint32_t r = 0; r < KI && !moves; ++r)
                for (uint32_t c = 0; c < KI && !moves; ++c) {
                    const uint32_t rho = (R << kin) | r, gam = (C << kin) | c;
                    if (pinv[rho] != rho || pinv[gam] != gam || !((cf.fone >> (rho * D + gam)) & 1ull))
                        moves = true;
                }
            if (moves)
                active |= 1ull << (R * NG + C);
        }
    G.active = active;
    G.groups = 0;
    cf.ngroups = 0;
    if (G.kin == 0 && G.g >= 2 && G.M >= 2) {
        // a tile permutation: pack the tile cycles into groups of <= 4 tiles (component index ==
        // logical tile index when every target is a grid bit)
        uint32_t ng = 0, fill = 0;
        uint64_t mask = 0;
        bool ok = true;
        cf.gcyc_off[0] = 0;
        for (uint32_t ci = 0; ci < cf.ncyc && ok; ++ci) {
            const uint32_t len = cf.cyc_off[ci + 1] - cf.cyc_off[ci];
            if (len > 4) {
                ok = false;
                break;
            }
            if (fill + len > 4) {
                G.gmask[ng] = mask;
                cf.gcyc_off[++ng] = (uint8_t)ci;
                fill = 0;
                mask = 0;
                if (ng >= 16) {
                    ok = false;
                    break;
                }
            }
            for (uint32_t j = 0; j < len; ++j)
                mask |= 1ull << cf.cyc[cf.cyc_off[ci] + j];
            fill += len;
        }
        if (ok && fill) {
            G.gmask[ng] = mask;
            cf.gcyc_off[++ng] = (uint8_t)cf.ncyc;
        }
        if (ok && ng >= 1 && ng <= 16) {
            G.groups = ng;
            cf.ngroups = ng;
        }
    }
    KrausArgs ka{nullptr, 0};
    if (active != 0) {
        if (k == 1)
            rc = launch<1, M_MONO, 64>(h, G, cf, ka, 1);
        else if (k == 2)
            rc = launch<2, M_MONO, 64>(h, G, cf, ka, 1);
        else
            rc = launch<3, M_MONO, 64>(h, G, cf, ka, 1);
        if (rc)
            return rc;
    }
    const uint64_t touched = 2 * state_bytes(h) * (uint64_t)__builtin_popcountll(active) / (NG * NG);
    return finish_plan(h, G, k, t, HS_PATH_NATIVE_PERMUTATION, plan, touched);
}

int hs_apply_permutation(hs_state* h, int k, const uint32_t* table, const uint32_t* t, hs_plan* plan) {
    if (!table)
        return set_err(HS_ERR_INVALID, "null permutation table");
    int rc = hs_apply_monomial(h, k, table, nullptr, t, plan);
    if (!rc && plan) {
        plan->path = HS_PATH_NATIVE_PERMUTATION;
        plan->subcases[0] = plan->subcases[1] = plan->subcases[2] = 0;
    }
    return rc;
}

int hs_apply_pauli(hs_state* h, uint32_t target, int y, hs_plan* plan) {
    const uint32_t perm[2] = {1, 0};
    // Y = [[0, -i], [i, 0]] = P diag(i, -i) with P the swap: U|0> = i|1>, U|1> = -i|0>.
    const double dy[4] = {0.0, 1.0, 0.0, -1.0};
    int rc = hs_apply_monomial(h, 1, perm, y ? dy : nullptr, &target, plan);
    if (!rc && plan) {
        plan->path = y ? HS_PATH_NATIVE_PAULI_Y : HS_PATH_NATIVE_PAULI_X;
        plan->subcases[0] = plan->subcases[1] = plan->subcases[2] = 0;
    }
    return rc;
}

int hs_apply_diagonal_phase(hs_state* h, uint32_t target, const double* phases, hs_plan* plan) {
    if (!phases)
        return set_err(HS_ERR_INVALID, "null phases");
    for (int i = 0; i < 2; ++i)
        if (std::fabs(std::hypot(phases[2 * i], phases[2 * i + 1]) - 1.0) > 1e-15)
            return set_err(HS_ERR_INVALID, "diagonal phase: non-unit modulus");
    int rc = hs_apply_monomial(h, 1, nullptr, phases, &target, plan);
    if (!rc && plan) {
        plan->path = HS_PATH_NATIVE_PHASE;
        plan->subcases[0] = plan->subcases[1] = plan->subcases[2] = 0;
    }
    return rc;
}

// --------------------------------------------------------------------------- observables
static int reduce(const hs_state* a, const hs_state* b, int kind, double* out) {
    if (!a || !b || !out)
        return set_err(HS_ERR_INVALID, "null argument");
    if (a->n != b->n || a->m != b->m)
        return set_err(HS_ERR_INVALID, "expectation: operands differ in size");
    DeviceGuard dg(a->device);
    if (b != a)
        CUDA_TRY(cudaStreamSynchronize(b->stream));
    if (a->Plog != b->Plog || a->shard != b->shard)
        return set_err(HS_ERR_INVALID, "expectation: operands are different shards");
    const uint64_t ntiles = a->count >> (2 * a->m);
    reduce_kernel<<<RED_BLOCKS, NTHR, 0, a->stream>>>(a->d, b->d, ntiles, (uint32_t)a->m, kind, a->red,
                                                       SD{a->Plog, a->logB, a->shard});
    finish_kernel<<<1, 32, 0, a->stream>>>(a->red, RED_BLOCKS, kind, a->red + 2 * RED_BLOCKS);
    g_launches.fetch_add(2, std::memory_order_relaxed);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaMemcpyAsync(out, a->red + 2 * RED_BLOCKS, sizeof(double), cudaMemcpyDeviceToHost, a->stream));
    CUDA_TRY(cudaStreamSynchronize(a->stream));
    return HS_OK;
}

int hs_expectation(const hs_state* rho, const hs_state* obs, double* out) { return reduce(obs, rho, 0, out); }
// Linear partial sums of one shard (kind 0: tr(rho O) part, 1: squared Frobenius part, 2: trace part);
// the operator's value is the sum over shards.
int hs_reduce_partial(const hs_state* a, const hs_state* b, int kind, double* out) {
    if (kind < 0 || kind > 2)
        return set_err(HS_ERR_INVALID, "bad reduction kind");
    return reduce(a, b ? b : a, kind, out);
}
int hs_frobenius(const hs_state* h, double* out) {
    int rc = reduce(h, h, 1, out);
    if (!rc)
        *out = std::sqrt(*out);
    return rc;
}
int hs_trace(const hs_state* h, double* out) { return reduce(h, h, 2, out); }

// ---------------------------------------------------------------------------- generators
int hs_state_fill_mixture(hs_state* h, int rank, const double* psi) {
    if (!h || !psi || rank < 1)
        return set_err(HS_ERR_INVALID, "bad mixture arguments");
    DeviceGuard dg(h->device);
    double2* dpsi = nullptr;
    const size_t bytes = (size_t)rank * h->N * sizeof(double2);
    CUDA_TRY(cudaMalloc(&dpsi, bytes));
    CUDA_TRY(cudaMemcpyAsync(dpsi, psi, bytes, cudaMemcpyHostToDevice, h->stream));
    const double inv = 1.0 / rank;
    fill_mixture_kernel<<<148 * 16, NTHR, 0, h->stream>>>(h->d, h->count, (uint32_t)h->m, h->N, dpsi, rank, inv,
                                                          SD{h->Plog, h->logB, h->shard});
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(h->stream);
    cudaFree(dpsi);
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, cudaGetErrorString(e));
    return HS_OK;
}

// hermsim::random_hermitian(n, seed, tiled, m) (storage.cpp:195-201) and basis_projector (:230-239)
// generated on the device into this state (any shard).
int hs_state_fill_random_hermitian(hs_state* h, uint64_t seed) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    DeviceGuard dg(h->device);
    fill_seeded_kernel<<<148 * 16, NTHR, 0, h->stream>>>(h->d, h->count, (uint32_t)h->m, h->N, seed, 0,
                                                         SD{h->Plog, h->logB, h->shard});
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

int hs_state_fill_basis_projector(hs_state* h, uint64_t basis) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (basis >= h->N)
        return set_err(HS_ERR_RANGE, "basis_projector: basis index out of range");
    DeviceGuard dg(h->device);
    fill_seeded_kernel<<<148 * 16, NTHR, 0, h->stream>>>(h->d, h->count, (uint32_t)h->m, h->N, basis, 1,
                                                         SD{h->Plog, h->logB, h->shard});
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}

int hs_state_fill_pauli_sum(hs_state* h, int count, const uint64_t* x, const uint64_t* z, const int32_t* ny,
                            const double* coef) {
    if (!h || count < 0 || (count && (!x || !z || !ny || !coef)))
        return set_err(HS_ERR_INVALID, "bad Pauli-sum arguments");
    DeviceGuard dg(h->device);
    const size_t n8 = (size_t)std::max(count, 1);
    char* buf = nullptr;
    CUDA_TRY(cudaMalloc(&buf, n8 * (8 + 8 + 4 + 8)));
    uint64_t* dx = (uint64_t*)buf;
    uint64_t* dz = dx + n8;
    double* dc = (double*)(dz + n8);
    int32_t* dn = (int32_t*)(dc + n8);
    if (count) {
        CUDA_TRY(cudaMemcpyAsync(dx, x, count * 8, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemcpyAsync(dz, z, count * 8, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemcpyAsync(dc, coef, count * 8, cudaMemcpyHostToDevice, h->stream));
        CUDA_TRY(cudaMemcpyAsync(dn, ny, count * 4, cudaMemcpyHostToDevice, h->stream));
    }
    PauliArgs pa{dx, dz, dn, dc, count};
    fill_pauli_kernel<<<148 * 16, NTHR, 0, h->stream>>>(h->d, h->count, (uint32_t)h->m, h->N, pa,
                                                        SD{h->Plog, h->logB, h->shard});
    g_launches.fetch_add(1, std::memory_order_relaxed);
    cudaError_t e = cudaGetLastError();
    cudaStreamSynchronize(h->stream);
    cudaFree(buf);
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, cudaGetErrorString(e));
    return HS_OK;
}


int hs_state_distance_mixture(const hs_state* h, int rank, const double* psi, double* max_abs) {
    if (!h || !psi || rank < 1 || !max_abs)
        return set_err(HS_ERR_INVALID, "bad distance arguments");
    DeviceGuard dg(h->device);
    double2* dpsi = nullptr;
    const size_t bytes = (size_t)rank * h->N * sizeof(double2);
    CUDA_TRY(cudaMalloc(&dpsi, bytes));
    CUDA_TRY(cudaMemcpyAsync(dpsi, psi, bytes, cudaMemcpyHostToDevice, h->stream));
    dist_mixture_kernel<<<RED_BLOCKS, NTHR, 0, h->stream>>>(h->d, h->count, (uint32_t)h->m, h->N, dpsi, rank,
                                                             1.0 / rank, h->red, SD{h->Plog, h->logB, h->shard});
    g_launches.fetch_add(1, std::memory_order_relaxed);
    std::vector<double> part(RED_BLOCKS);
    cudaError_t e = cudaGetLastError();
    if (e == cudaSuccess)
        e = cudaMemcpyAsync(part.data(), h->red, RED_BLOCKS * sizeof(double), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(h->stream);
    cudaFree(dpsi);
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, cudaGetErrorString(e));
    double mx = 0.0;
    for (double v : part)
        mx = std::max(mx, v);
    *max_abs = mx;
    return HS_OK;
}

// ------------------------------------------------------------------------------- timing
int hs_event_create(void** ev) {
    if (!ev)
        return set_err(HS_ERR_INVALID, "null out");
    cudaEvent_t e;
    CUDA_TRY(cudaEventCreate(&e));
    *ev = e;
    return HS_OK;
}
int hs_event_destroy(void* ev) {
    CUDA_TRY(cudaEventDestroy((cudaEvent_t)ev));
    return HS_OK;
}
int hs_event_record(void* ev, const hs_state* h) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    CUDA_TRY(cudaEventRecord((cudaEvent_t)ev, h->stream));
    return HS_OK;
}
int hs_event_elapsed_ms(void* start, void* stop, float* ms) {
    CUDA_TRY(cudaEventSynchronize((cudaEvent_t)stop));
    CUDA_TRY(cudaEventElapsedTime(ms, (cudaEvent_t)start, (cudaEvent_t)stop));
    return HS_OK;
}

}  // extern "C"

// Diagnostics: gather-kernel phase cycles summed over CTAs (HS_DEBUG_FLAGS bit 4), read and reset.
extern "C" int hs_debug_phase_cycles(unsigned long long* out8) {
    if (!out8)
        return set_err(HS_ERR_INVALID, "null out");
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpyFromSymbol(out8, g_phase_cycles, 8 * sizeof(unsigned long long)));
    unsigned long long z[8] = {0};
    CUDA_TRY(cudaMemcpyToSymbol(g_phase_cycles, z, sizeof(z)));
    return HS_OK;
}

// ---------------------------------------------------------------------- OHRM save / load
// The reference's container (storage_io.cpp:34-118, storage_io.hpp:22-29): magic "OHRM", version
// u32 = 1, format tag u8 (tiled = 2, types.hpp:15), n u8, m u8, five reserved zero bytes, then the
// payload as little-endian (re, im) binary64 pairs in native element order.  The payload streams
// between HBM and the file through two pinned 64 MiB buffers (copy of chunk i+1 overlaps the write /
// read of chunk i), so a 137 GB n = 17 operator never needs host RAM.  Error messages carry the
// reference's IoErrorKind names.
namespace {
constexpr uint64_t IO_CHUNK = 64ull << 20;  // bytes
struct PinnedPair {
    void* b[2] = {nullptr, nullptr};
    ~PinnedPair() {
        for (void* p : b)
            if (p)
                cudaFreeHost(p);
    }
};
}  // namespace

int hs_state_save(const hs_state* h, const char* path) {
    if (!h || !path)
        return set_err(HS_ERR_INVALID, "null argument");
    if (h->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "save: sharded operators are saved shard by shard (download_full)");
    FILE* f = std::fopen(path, "wb");
    if (!f)
        return set_err(HS_ERR_IO, std::string("io_failure: save: cannot open ") + path);
    unsigned char hdr[16] = {'O', 'H', 'R', 'M', 1, 0, 0, 0, 2, (unsigned char)h->n, (unsigned char)h->m, 0, 0, 0, 0, 0};
    bool ok = std::fwrite(hdr, 1, 16, f) == 16;
    DeviceGuard dg(h->device);
    PinnedPair pp;
    const uint64_t total = h->count * sizeof(double2);
    for (int i = 0; i < 2 && ok; ++i)
        if (cudaHostAlloc(&pp.b[i], IO_CHUNK, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            std::fclose(f);
            return set_err(HS_ERR_NOMEM, "save: pinned staging buffer");
        }
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    const char* src = reinterpret_cast<const char*>(h->d);
    uint64_t off = 0, prev = 0;
    int cur = 0;
    bool pending = false;
    uint64_t prev_len = 0;
    while (ok && (off < total || pending)) {
        const uint64_t len = std::min<uint64_t>(IO_CHUNK, total - off);
        if (off < total) {
            if (cudaMemcpyAsync(pp.b[cur], src + off, len, cudaMemcpyDeviceToHost, h->stream) != cudaSuccess) {
                ok = false;
                break;
            }
            cudaEventRecord(ev[cur], h->stream);
        }
        if (pending) {  // write the previous chunk while this one copies
            cudaEventSynchronize(ev[cur ^ 1]);
            ok = std::fwrite(pp.b[cur ^ 1], 1, prev_len, f) == prev_len;
        }
        pending = off < total;
        prev = off;
        prev_len = len;
        off += len;
        cur ^= 1;
    }
    (void)prev;
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    ok = (std::fclose(f) == 0) && ok;
    if (cudaGetLastError() != cudaSuccess)
        return set_err(HS_ERR_CUDA, "save: device copy failed");
    if (!ok)
        return set_err(HS_ERR_IO, "io_failure: save: stream write failed");
    return HS_OK;
}

int hs_state_load(const char* path, int device, hs_state** out) {
    if (!path || !out)
        return set_err(HS_ERR_INVALID, "null argument");
    *out = nullptr;
    FILE* f = std::fopen(path, "rb");
    if (!f)
        return set_err(HS_ERR_IO, std::string("io_failure: load: cannot open ") + path);
    unsigned char hdr[16];
    auto fail = [&](int code, const char* msg) {
        std::fclose(f);
        return set_err(code, msg);
    };
    if (std::fread(hdr, 1, 16, f) != 16)
        return fail(HS_ERR_IO, "truncated: load: header truncated");
    if (std::memcmp(hdr, "OHRM", 4) != 0)
        return fail(HS_ERR_IO, "bad_magic: load: bad magic bytes");
    const uint32_t ver = hdr[4] | (hdr[5] << 8) | (hdr[6] << 16) | ((uint32_t)hdr[7] << 24);
    if (ver != 1)
        return fail(HS_ERR_IO, "bad_version: load: unsupported version");
    const int tag = hdr[8], n = hdr[9], m = hdr[10];
    if (tag > 2)
        return fail(HS_ERR_IO, "bad_header: load: unknown format tag");
    if (n < 1 || n > 30)
        return fail(HS_ERR_IO, "bad_header: load: qubit count out of range");
    if (tag != 2 && m != 0)
        return fail(HS_ERR_IO, "bad_header: load: tile exponent set for non-tiled format");
    if (tag == 2 && (m < 0 || m > n + 2))
        return fail(HS_ERR_IO, "bad_header: load: tile exponent out of range");
    if (tag != 2)
        return fail(HS_ERR_UNSUPPORTED, "load: dense / packed payloads are not device formats (tiled only)");
    hs_state* h = nullptr;
    int rc = hs_state_create(n, m, device, &h);
    if (rc) {
        std::fclose(f);
        return rc;
    }
    DeviceGuard dg(h->device);
    PinnedPair pp;
    for (int i = 0; i < 2; ++i)
        if (cudaHostAlloc(&pp.b[i], IO_CHUNK, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            hs_state_free(h);
            return fail(HS_ERR_NOMEM, "load: pinned staging buffer");
        }
    const uint64_t total = h->count * sizeof(double2);
    char* dst = reinterpret_cast<char*>(h->d);
    uint64_t off = 0;
    int cur = 0;
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    bool used[2] = {false, false};
    bool ok = true;
    while (off < total) {
        const uint64_t len = std::min<uint64_t>(IO_CHUNK, total - off);
        if (used[cur])
            cudaEventSynchronize(ev[cur]);  // the buffer's previous upload has left it
        if (std::fread(pp.b[cur], 1, len, f) != len) {
            ok = false;
            break;
        }
        cudaMemcpyAsync(dst + off, pp.b[cur], len, cudaMemcpyHostToDevice, h->stream);
        cudaEventRecord(ev[cur], h->stream);
        used[cur] = true;
        off += len;
        cur ^= 1;
    }
    cudaStreamSynchronize(h->stream);
    cudaEventDestroy(ev[0]);
    cudaEventDestroy(ev[1]);
    if (!ok) {
        hs_state_free(h);
        return fail(HS_ERR_IO, "truncated: load: payload truncated");
    }
    char probe;
    if (std::fread(&probe, 1, 1, f) != 0) {
        hs_state_free(h);
        return fail(HS_ERR_IO, "length_mismatch: load: trailing bytes after payload");
    }
    std::fclose(f);
    if (cudaGetLastError() != cudaSuccess) {
        hs_state_free(h);
        return set_err(HS_ERR_CUDA, "load: device copy failed");
    }
    *out = h;
    return HS_OK;
}

// ------------------------------------------------------------------ peer-memory sharding
// Peer mode: a cross-shard operation reads the group members' current payloads where
// they lie -- peer memory over NVLink (CUDA IPC across processes, or peer access in one process) or
// the same device -- inside the operation's own kernels, and writes this shard's result into its
// second buffer, which then becomes current.  The collective is the kernel's remote tile reads;
// nothing is staged through an exchange buffer.  The caller orders operations across shards: before
// a cross-shard operation every group member must have finished its previous operations (a
// barrier), because members read each other's current buffers while writing their own other one.
int hs_state_peer_enable(hs_state* h) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (h->peer_mode)
        return HS_OK;
    DeviceGuard dg(h->device);
    double2* alt = nullptr;
    cudaError_t e = cudaMalloc(&alt, h->count * sizeof(double2));
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(HS_ERR_NOMEM, std::string("peer mode: second payload buffer: ") + cudaGetErrorString(e));
    }
    h->buf[0] = h->d;
    h->buf[1] = alt;
    h->flip = 0;
    h->peer_mode = true;
    return HS_OK;
}

int hs_state_peer_buffers(const hs_state* h, void** b0, void** b1) {
    if (!h || !h->peer_mode)
        return set_err(HS_ERR_INVALID, "peer mode not enabled");
    if (b0)
        *b0 = h->buf[0];
    if (b1)
        *b1 = h->buf[1];
    return HS_OK;
}

int hs_state_set_peer(hs_state* h, int shard, const void* b0, const void* b1) {
    if (!h || !b0 || !b1)
        return set_err(HS_ERR_INVALID, "null argument");
    if (shard < 0 || shard >= (1 << h->Plog) || shard >= 64 || shard == (int)h->shard)
        return set_err(HS_ERR_RANGE, "bad peer shard");
    h->peer_buf[shard][0] = static_cast<const double2*>(b0);
    h->peer_buf[shard][1] = static_cast<const double2*>(b1);
    return HS_OK;
}

int hs_state_peer_flip(const hs_state* h, int* flip) {
    if (!h || !flip)
        return set_err(HS_ERR_INVALID, "null argument");
    *flip = (int)h->flip;
    return HS_OK;
}

int hs_ipc_handles(const hs_state* h, void* out128) {
    if (!h || !out128 || !h->peer_mode)
        return set_err(HS_ERR_INVALID, "peer mode not enabled");
    DeviceGuard dg(h->device);
    cudaIpcMemHandle_t a, b;
    CUDA_TRY(cudaIpcGetMemHandle(&a, h->buf[0]));
    CUDA_TRY(cudaIpcGetMemHandle(&b, h->buf[1]));
    std::memcpy(out128, &a, 64);
    std::memcpy(static_cast<char*>(out128) + 64, &b, 64);
    return HS_OK;
}

int hs_ipc_open(const void* handle64, int device, void** ptr) {
    if (!handle64 || !ptr)
        return set_err(HS_ERR_INVALID, "null argument");
    DeviceGuard dg(device);
    cudaIpcMemHandle_t hd;
    std::memcpy(&hd, handle64, 64);
    CUDA_TRY(cudaIpcOpenMemHandle(ptr, hd, cudaIpcMemLazyEnablePeerAccess));
    return HS_OK;
}

int hs_ipc_close(void* ptr, int device) {
    if (!ptr)
        return HS_OK;
    DeviceGuard dg(device);
    CUDA_TRY(cudaIpcCloseMemHandle(ptr));
    return HS_OK;
}

int hs_peer_access(int device, int peer_device) {
    if (device == peer_device)
        return HS_OK;
    DeviceGuard dg(device);
    int can = 0;
    CUDA_TRY(cudaDeviceCanAccessPeer(&can, device, peer_device));
    if (!can)
        return set_err(HS_ERR_UNSUPPORTED, "no peer access between the devices");
    const cudaError_t e = cudaDeviceEnablePeerAccess(peer_device, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled)
        return set_err(HS_ERR_CUDA, std::string("cudaDeviceEnablePeerAccess: ") + cudaGetErrorString(e));
    cudaGetLastError();
    return HS_OK;
}

// ------------------------------------------------------------------------- CUDA graphs
// A sequence of operations on one state captured once and replayed: the host-side planning (tables,
// geometry, dispatch) runs at capture time only, the replay is one cudaGraphLaunch on the state's
// stream.  For circuits repeated many times and for small states, where launch latency and host
// dispatch approach the kernel time.  Not for peer-mode states (buffer flips are host state).
struct hs_graph {
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    int device = 0;
};

int hs_graph_begin(hs_state* h) {
    if (!h)
        return set_err(HS_ERR_INVALID, "null state");
    if (h->peer_mode)
        return set_err(HS_ERR_UNSUPPORTED, "graphs: peer-mode states flip buffers on the host");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaStreamBeginCapture(h->stream, cudaStreamCaptureModeThreadLocal));
    return HS_OK;
}

int hs_graph_end(hs_state* h, hs_graph** out) {
    if (!h || !out)
        return set_err(HS_ERR_INVALID, "null argument");
    *out = nullptr;
    DeviceGuard dg(h->device);
    cudaGraph_t g = nullptr;
    const cudaError_t e = cudaStreamEndCapture(h->stream, &g);
    if (e != cudaSuccess) {
        cudaGetLastError();
        return set_err(HS_ERR_CUDA, std::string("graph capture failed: ") + cudaGetErrorString(e));
    }
    auto* hg = new hs_graph();
    hg->graph = g;
    hg->device = h->device;
    const cudaError_t e2 = cudaGraphInstantiate(&hg->exec, g, 0);
    if (e2 != cudaSuccess) {
        cudaGetLastError();
        cudaGraphDestroy(g);
        delete hg;
        return set_err(HS_ERR_CUDA, std::string("cudaGraphInstantiate: ") + cudaGetErrorString(e2));
    }
    *out = hg;
    return HS_OK;
}

int hs_graph_launch(const hs_graph* g, hs_state* h) {
    if (!g || !h)
        return set_err(HS_ERR_INVALID, "null argument");
    DeviceGuard dg(h->device);
    CUDA_TRY(cudaGraphLaunch(g->exec, h->stream));
    return HS_OK;
}

int hs_graph_nodes(const hs_graph* g, uint64_t* n) {
    if (!g || !n)
        return set_err(HS_ERR_INVALID, "null argument");
    size_t c = 0;
    CUDA_TRY(cudaGraphGetNodes(g->graph, nullptr, &c));
    *n = c;
    return HS_OK;
}

int hs_graph_free(hs_graph* g) {
    if (!g)
        return HS_OK;
    DeviceGuard dg(g->device);
    cudaGraphExecDestroy(g->exec);
    cudaGraphDestroy(g->graph);
    delete g;
    return HS_OK;
}
