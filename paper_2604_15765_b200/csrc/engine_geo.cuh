// engine_geo.cuh -- part of engine.cu (one translation unit; included in order).
// Geometry of an operation (Geo), coefficient blocks (Coef), per-CTA tables, bit
// helpers, tile / unit / shard addressing shared by every kernel of the engine.
#pragma once

namespace {

constexpr int NTHR = 256;          // threads per CTA
constexpr uint32_t CAP = 2048;     // target complex elements staged per CTA item (32 KiB)
constexpr uint32_t CAPD = 2048;    // same for diagonal-unit items
constexpr uint32_t CAP_WHOLE = 4096;  // units up to 64 KiB are staged as whole stored tiles
constexpr uint32_t MAX_TT = 256;   // max logical tiles per item (tile table in smem)
constexpr uint32_t DBG_POISON = 1024u;  // HS_DEBUG_FLAGS bit: NaN-fill ring stages between uses
// NaN-fill n elements of a ring stage (threads t of nt), then order those generic-proxy writes before
// the async-proxy (TMA / bulk) loads the caller issues next
__device__ __forceinline__ void poison_stage(double2* sb, uint32_t n, uint32_t t, uint32_t nt) {
    const double nan = __longlong_as_double(0x7ff8dead0000beefll);
    for (uint32_t e = t; e < n; e += nt)
        sb[e] = make_double2(nan, nan);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
constexpr uint64_t F_ADJ = 1ull << 63, F_SKIP = 1ull << 62, F_BAD = 1ull << 61, F_NOSTORE = 1ull << 60,
                   F_REMOTE = 1ull << 59, F_MIRROR = 1ull << 55, F_MASK = (1ull << 55) - 1;

enum Mode : int { M_S1 = 0, M_HAD = 1, M_S2 = 2, M_DIRECT = 3, M_MONO = 4, M_KRAUS = 5, M_PROG = 6, M_SF2 = 7, M_SF3 = 8 };

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
    uint32_t dbg;                 // diagnostics (HS_DEBUG_FLAGS): gather bit 0 skips the transform, bit 1 the loads,
                                  // bit 2 the stores, bit 4 phase timing, bit 5 ping-pong kernel, bit 6 no bulk rows,
                                  // bit 8 no TMA boxes
    uint32_t ws_diag;             // gather_ws: units include the diagonal base pairs (grid programs)
    uint32_t qstride;             // gather_ws, k = 2 DMMA: position offset between paired blocks
    uint32_t rev;                 // sweep the items in reverse order (alternates per launch: L2 reuse)
    uint32_t bulk;                // gather_ws: sub-block rows move as cp.async.bulk runs (>= 8 contiguous
                                  // elements), every tile staged in its STORED orientation (cadj: adjoint offsets)
    uint32_t logRun;              // bulk: log2 of the run length (contiguous low in-tile bits of the sub-block)
    uint32_t tma;                 // gather_ws (with bulk groups): 8 x 8 boxes by tensor map, SWIZZLE_128B;
                                  // cdir[slot] = box base (16-B units, phase included), tsk[slot] = phase
    uint32_t tq;                  // tma: 4 when bit 3 of the sub-block is a block-position bit (quadrant per warp)
    uint32_t grp4;                // gather_ws, in-tile k = 3: an item is 4 consecutive local stored tiles
    uint64_t nloc_tiles;          // grp4: local stored tiles
    // bulk staging: row x of a staged tile sits at x * PD + (x >> 3) * s8 (rows 8 apart share banks
    // otherwise; the offset is additive over disjoint row bits, so block bases and component offsets
    // still add)
    uint32_t s8;
    // S-form transform (M_SF2, k = 2 transfer matrix on the FP64 tensor path): contraction order
    // (k-step ks, lane column c) -> component sf_pi[4 ks + c], output order (n-tile, column) ->
    // component sf_sigma[8 nt + n]; blocks of a pass run along rows (sf_xfast) or columns
    uint8_t sf_pi[16], sf_sigma[16];
    uint32_t sf_xfast;
    uint32_t sf_cost, sf_ideal;   // planner diagnostics: bank-group cost of the chosen S-form layout / its ideal
    // k = 3 Kraus sums in the hermitian basis (M_SF3): B fragments of the real 64 x 64 matrix R in
    // fragment order [k-step 16][n-tile 8][lane 32] (32 KiB, device memory; staged in shared memory
    // per CTA); hf_in[16 c + ks]: block element lane c loads at k-step ks; hf_out[2 (4 nt + c) + e]:
    // the two block elements lane c writes for n-tile nt
    const double* sf3;
    uint8_t hf_in[64], hf_out[64];
    // hform3 on TMA boxes: staging slot (tile, box) of each block component, direct / adjoint tile
    uint8_t hsd[64], hsa[64];
};

// Per-CTA copies of the small index tables of Geo (shared memory).
struct Tabs {
    uint8_t xdep[32], xb[32], yb[32], xs_rin[32], xs_base[32], y_cin[32], y_base[32], xs_in[8], y_in[8];
    uint16_t cdir[64], cadj[64];  // component offsets (copied from Geo: indexed per thread)
    uint8_t ttr[64];
    uint8_t tsk[64];
    uint8_t slt[64];  // pipe kernel, monomials: staging slot -> logical tile (compacted active tiles)
    uint8_t hsd[64], hsa[64];  // hform3 on TMA boxes: slot of each component (direct / adjoint tile)
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
    // k = 2 Kraus sum on the tensor-core gather: nk (2..4) operators L_a in s[16a .. 16a + 15]
    uint32_t nk;
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

}  // namespace
