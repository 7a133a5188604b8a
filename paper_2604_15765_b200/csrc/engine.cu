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
// All data is complex128 (double2).  The path is HBM-bound; only the k = 3 (and
// paired k = 2) transforms run on the FP64 tensor path (mma.sync f64, engine_gather.cuh).
//
// Files (one translation unit): engine_geo.cuh (geometry, addressing), engine_kernels.cuh (block
// transforms, slab kernel, TMA pipeline), engine_gather.cuh (gather kernels, DMMA transforms, grid
// programs), engine_aux.cuh (reductions, generators); this file: state, launch planning, C-ABI
// (include/hs_cuda.h), sharding / exchange, OHRM I/O, CUDA graphs.
#include <cuda.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <mutex>
#include <unordered_map>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "hs_cuda.h"


#include "engine_geo.cuh"
#include "engine_kernels.cuh"
#include "engine_gather.cuh"
#include "engine_aux.cuh"
#include "engine_convert.cuh"


// =============================================================================== host side
constexpr size_t HCACHE_MAX = 1024;  // cached k = 3 Kraus sets per state (32 KiB of fragments each)
struct HCacheEntry {
    uint64_t key = 0;
    int nops = 0;
    std::vector<double2> ops;
    double* dev = nullptr;
};
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
    std::vector<HCacheEntry> hcache;           // device fragments of the k = 3 Kraus sets seen (hform3)
    double* hscratch = nullptr;                // fragments of an uncached set once the cache is full
    // tile exponents m > 5: the operator lives in HBM in the m = 5 layout (every kernel unchanged);
    // the user-facing payload (info, upload / download, save / load) is the mu layout, converted on
    // the fly by the retile kernel.  mu == m and ucount == count otherwise.
    int mu = 0;
    uint64_t ucount = 0, uG = 0;
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
// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda)
using EncodeTiledFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                   const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                   CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn tensor_map_encoder() {
    static EncodeTiledFn fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            return (EncodeTiledFn) nullptr;
        return (EncodeTiledFn)p;
    }();
    return fn;
}
// The payload as rows of one 32-element tile row (64 doubles, 512 B), boxes of 8 rows x 8 complex
// elements (128 B: the SWIZZLE_128B span).
bool encode_tile_map(CUtensorMap* tm, const void* base, uint64_t elems) {
    const EncodeTiledFn fn = tensor_map_encoder();
    if (!fn || elems / 32 >= (1ull << 32))
        return false;
    cuuint64_t dims[2] = {64, elems / 32};
    cuuint64_t strides[1] = {512};
    cuuint32_t box[2] = {16, 8}, estr[2] = {1, 1};
    return fn(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<void*>(base), dims, strides, box, estr,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// Bank-spreading searches of plan_gather (skews / swizzle phases) depend only on the shape of an
// operation (in-tile targets, number of grid targets, sub-block), not on its grid qubits or the
// state: their results are cached per shape (a search costs up to a few ms of host time, more than
// a small state's kernel).
std::mutex g_search_mu;
std::unordered_map<uint64_t, std::array<uint8_t, 65>> g_search_cache;
uint64_t search_key(const Geo& G, uint32_t kind, uint32_t qstride) {
    return (uint64_t)G.in_mask | (uint64_t)G.g << 8 | (uint64_t)G.S0 << 12 | (uint64_t)G.D << 20 |
           (uint64_t)G.kin << 26 | (uint64_t)qstride << 30 | (uint64_t)G.M << 36 | (uint64_t)G.nxb << 44 |
           (uint64_t)G.nyb << 51 | (uint64_t)kind << 58;
}
bool search_get(uint64_t key, std::array<uint8_t, 65>& out) {
    std::lock_guard<std::mutex> lk(g_search_mu);
    auto it = g_search_cache.find(key);
    if (it == g_search_cache.end())
        return false;
    out = it->second;
    return true;
}
void search_put(uint64_t key, const std::array<uint8_t, 65>& v) {
    std::lock_guard<std::mutex> lk(g_search_mu);
    g_search_cache[key] = v;
}

// bulk: stage sub-block rows with cp.async.bulk, one copy per run of >= 8 contiguous elements
// (tiles keep their stored orientation, adjoint components addressed through cadj).
// element tables of the hermitian-basis transform (hform3; built by hform_tables below)
struct HForm {
    uint8_t in[64], out[64];
};
const HForm& hform_tables();
void plan_gather(Geo& G, bool dmma = false, bool bulk = false, uint32_t qstride = 0, bool tma = false,
                 bool prog = false, bool sform = false, uint32_t min_run = 4, bool hform = false) {
    const uint32_t M = G.M, g = G.g, NT = G.grp4 ? 4u : 1u << (2 * g), NG = 1u << g, kin = G.kin;
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
    // bulk rows: runs of the low contiguous sub-block bits, at least 16 elements (256 B; 128-B runs
    // are bound by the bulk-copy engine's operation rate: C3 g = 3 15.4 -> 20.7 ms measured)
    G.logRun = std::min<uint32_t>(__builtin_ctz(~cmask), G.logS0);
    G.bulk = bulk && (dmma || sform) && G.logRun >= min_run;
    G.TS = S0 * (S0 + 1);
    G.s8 = 0;
    G.sf_xfast = 0;
    for (uint32_t i = 0; i < 16; ++i)
        G.sf_pi[i] = G.sf_sigma[i] = (uint8_t)i;
    const uint32_t D = G.D, kinm = (1u << kin) - 1;
    for (uint32_t t = 0; t < 64; ++t)
        G.tsk[t] = 0;
    auto tables = [&]() {
        for (uint32_t rho = 0; rho < D; ++rho)
            for (uint32_t gam = 0; gam < D; ++gam) {
                const uint32_t R = rho >> kin, C = gam >> kin, i = rho * D + gam, t = R * NG + C;
                G.ttr[i] = (uint8_t)t;
                const uint32_t xr = G.xs_in[rho & kinm], yc = G.y_in[gam & kinm];
                G.cdir[i] = G.cadj[i] = (uint16_t)(t * G.TS + G.tsk[t] + xr * G.PD + (xr >> 3) * G.s8 + yc);
                if (G.bulk)  // adjoint tiles in stored orientation: logical (x, y) at row y, column x
                    G.cadj[i] = (uint16_t)(t * G.TS + G.tsk[t] + yc * G.PD + (yc >> 3) * G.s8 + xr);
            }
    };
    tables();
    uint32_t extra = 0;
    if (sform && G.bulk && D == 4) {
        // S-form transform (sform2): a quarter-warp touches blocks 2ph, 2ph + 1 of a pass x the four
        // components of a k-step (loads) or of an output pair (stores).  Spread each over the eight
        // 16-byte bank groups: search the block order, the row skew s8, the tile pitch, the
        // contraction / output orders and per-tile skews (cached per shape).
        const uint32_t lbt = G.logNxb + G.logNyb, npass = ((G.grp4 ? 4u : 1u) << lbt) >> 3;
        const uint32_t TS0 = G.TS, NTs = NT;
        const uint32_t smp[4] = {0, npass > 1 ? 1u : 0u, npass / 2, npass - 1};
        const bool any_adj = !G.grp4 && g > 0;
        auto cost_of = [&]() {
            const uint32_t lf = G.sf_xfast ? G.logNxb : G.logNyb;
            uint32_t cost = 0;
            for (uint32_t si = 0; si < 4; ++si)
                for (uint32_t adj = 0; adj < (any_adj ? 2u : 1u); ++adj)
                    for (uint32_t pat = 0; pat < 8; ++pat)
                        for (uint32_t ph = 0; ph < 4; ++ph) {
                            uint32_t cnt[8] = {0}, mx = 0;
                            for (uint32_t l = 8 * ph; l < 8 * ph + 8; ++l) {
                                const uint32_t gq = l >> 2, cq = l & 3u, b = 8 * smp[si] + gq;
                                const uint32_t bq = b & ((1u << lbt) - 1), i0 = bq & ((1u << lf) - 1), i1 = bq >> lf;
                                const uint32_t xbv = G.xb_tab[G.sf_xfast ? i0 : i1], ybv = G.yb_tab[G.sf_xfast ? i1 : i0];
                                const uint32_t slot = (b >> lbt) * G.TS;
                                const uint32_t comp = pat < 4 ? G.sf_pi[4 * pat + cq]
                                                              : G.sf_sigma[8 * ((pat - 4) >> 1) + 2 * cq + ((pat - 4) & 1u)];
                                const uint32_t a = adj ? slot + ybv * G.PD + (ybv >> 3) * G.s8 + xbv + G.cadj[comp]
                                                       : slot + xbv * G.PD + (xbv >> 3) * G.s8 + ybv + G.cdir[comp];
                                mx = std::max(mx, ++cnt[a & 7u]);
                            }
                            cost += mx;
                        }
            return cost;
        };
        // one descent pass over pairwise swaps of the contraction and output orders
        auto swap_pass = [&](uint32_t& cur) {
            for (int which = 0; which < 2; ++which) {
                uint8_t* perm = which ? G.sf_sigma : G.sf_pi;
                for (uint32_t a = 0; a < 16; ++a)
                    for (uint32_t b = a + 1; b < 16; ++b) {
                        std::swap(perm[a], perm[b]);
                        const uint32_t c = cost_of();
                        if (c < cur)
                            cur = c;
                        else
                            std::swap(perm[a], perm[b]);
                    }
            }
        };
        const uint32_t ideal = 4u * (any_adj ? 2u : 1u) * 8u * 4u;
        const size_t stage_cap = 213u * 1024u / 16u;  // elements per stage (3 stages + static tables)
        const uint64_t key = search_key(G, 3, 0);
        std::array<uint8_t, 65> cached;
        if (search_get(key, cached)) {
            for (uint32_t t = 0; t < NTs; ++t)
                G.tsk[t] = cached[t];
            for (uint32_t i = 0; i < 16; ++i) {
                G.sf_pi[i] = cached[16 + i];
                G.sf_sigma[i] = cached[32 + i];
            }
            G.s8 = cached[48];
            G.sf_xfast = cached[49];
            G.TS = TS0 + (S0 >> 3) * G.s8 + cached[50];
            tables();
        } else {
            uint32_t best = ~0u, bx = 0, bs = 0, be = 0;
            uint8_t bpi[16], bsig[16];
            for (uint32_t xf = 0; xf < 2 && best > ideal; ++xf)
                for (uint32_t s8 = 0; s8 < 8 && best > ideal; ++s8)
                    for (uint32_t e = 0; e < 8 && best > ideal; ++e) {
                        const uint32_t TS = TS0 + (S0 >> 3) * s8 + e;
                        if (NTs * TS + 7 > stage_cap)
                            continue;
                        G.sf_xfast = xf;
                        G.s8 = s8;
                        G.TS = TS;
                        for (uint32_t i = 0; i < 16; ++i)
                            G.sf_pi[i] = G.sf_sigma[i] = (uint8_t)i;
                        for (uint32_t t = 0; t < 64; ++t)
                            G.tsk[t] = 0;
                        tables();
                        uint32_t cur = cost_of();
                        if (cur > ideal)
                            swap_pass(cur);
                        if (cur < best) {
                            best = cur;
                            bx = xf;
                            bs = s8;
                            be = e;
                            std::memcpy(bpi, G.sf_pi, 16);
                            std::memcpy(bsig, G.sf_sigma, 16);
                        }
                    }
            G.sf_xfast = bx;
            G.s8 = bs;
            G.TS = TS0 + (S0 >> 3) * bs + be;
            std::memcpy(G.sf_pi, bpi, 16);
            std::memcpy(G.sf_sigma, bsig, 16);
            tables();
            uint32_t cur = best;
            for (uint32_t pass = 0; pass < 2 && cur > ideal; ++pass) {
                for (uint32_t t = 0; t < NTs && NTs > 1; ++t) {  // per-tile skews
                    uint8_t bv = G.tsk[t];
                    for (uint32_t v = 0; v < 8; ++v) {
                        G.tsk[t] = (uint8_t)v;
                        tables();
                        const uint32_t c = cost_of();
                        if (c < cur) {
                            cur = c;
                            bv = (uint8_t)v;
                        }
                    }
                    G.tsk[t] = bv;
                    tables();
                }
                swap_pass(cur);
            }
            std::array<uint8_t, 65> v{};
            for (uint32_t t = 0; t < NTs; ++t)
                v[t] = G.tsk[t];
            for (uint32_t i = 0; i < 16; ++i) {
                v[16 + i] = G.sf_pi[i];
                v[32 + i] = G.sf_sigma[i];
            }
            v[48] = (uint8_t)G.s8;
            v[49] = (uint8_t)G.sf_xfast;
            v[50] = (uint8_t)(G.TS - TS0 - (S0 >> 3) * G.s8);
            search_put(key, v);
        }
        if (G.grp4) {  // independent tiles at slot t * TS: one skew
            for (uint32_t t = 1; t < NTs; ++t)
                G.tsk[t] = G.tsk[0];
            tables();
        }
        G.sf_cost = cost_of();
        G.sf_ideal = ideal;
        extra = 7;
    } else if (dmma && (D == 8 || (D == 4 && qstride))) {
        // the DMMA transform's lane patterns (load B[2c+j][g], store Z[g][2c+j]; k = 2: the 8 x 8
        // matrix of four quadrant blocks at offset qstride) hit 16-byte bank groups (addr mod 8) by
        // component offset: pick a tile pitch and per-tile skews that spread every quarter-warp
        // over 8 groups (the offsets are additive in the block base, so one block decides)
        auto comp = [&](uint32_t row, uint32_t col) -> uint32_t {
            if (D == 8)
                return G.cdir[row * 8 + col];
            return G.cdir[(row & 3) * 4 + (col & 3)] + ((row >> 2) * G.PD + (col >> 2)) * qstride;
        };
        auto cost_of = [&]() {
            uint32_t cost = 0;
            for (int pat = 0; pat < 2; ++pat)
                for (uint32_t j = 0; j < 2; ++j)
                    for (uint32_t ph = 0; ph < 4; ++ph) {
                        uint32_t cnt[8] = {0}, mx = 0;
                        for (uint32_t l = 8 * ph; l < 8 * ph + 8; ++l) {
                            const uint32_t gq = l >> 2, cq = l & 3;
                            const uint32_t a = pat ? comp(gq, 2 * cq + j) : comp(2 * cq + j, gq);
                            mx = std::max(mx, ++cnt[a & 7u]);
                        }
                        cost += mx;
                    }
            return cost;
        };
        const uint32_t TS0 = G.TS;
        const uint64_t key = search_key(G, 1, qstride);
        std::array<uint8_t, 65> cached;
        const bool hit = search_get(key, cached);
        uint32_t best = ~0u, bestE = 0, bestS = 0;
        for (uint32_t e = 0; e < 8 && !hit; ++e)
            for (uint32_t sk = 0; sk < 8; ++sk) {
                G.TS = TS0 + e;
                for (uint32_t t = 0; t < NT; ++t)
                    G.tsk[t] = (uint8_t)((sk * (t >> g)) & 7u);
                tables();
                const uint32_t cost = cost_of() * 64 + e + sk;  // ties: the smallest footprint
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
        // then per-tile skews by coordinate descent (a linear skew in the tile row cannot spread
        // four tile rows x two columns of stride 2 over 8 groups)
        if (hit) {
            G.TS = TS0 + cached[64];
            for (uint32_t t = 0; t < NT; ++t)
                G.tsk[t] = cached[t];
            tables();
        }
        uint32_t cur = hit ? 0u : cost_of();
        for (uint32_t pass = 0; pass < 3 && cur > 16; ++pass)
            for (uint32_t t = 0; t < NT; ++t) {
                const uint8_t keep = G.tsk[t];
                uint8_t bv = keep;
                for (uint32_t v = 0; v < 8; ++v) {
                    G.tsk[t] = (uint8_t)v;
                    tables();
                    const uint32_t c = cost_of();
                    if (c < cur) {
                        cur = c;
                        bv = (uint8_t)v;
                    }
                }
                G.tsk[t] = bv;
                tables();
            }
        if (!hit) {
            std::array<uint8_t, 65> v{};
            for (uint32_t t = 0; t < NT; ++t)
                v[t] = G.tsk[t];
            v[64] = (uint8_t)(G.TS - TS0);
            search_put(key, v);
        }
        if (G.grp4) {  // independent tiles at slot t * TS: one skew (the transform adds t * TS)
            for (uint32_t t = 1; t < NT; ++t)
                G.tsk[t] = G.tsk[0];
            tables();
        }
        extra = 7;
    }
    G.tma = 0;
    const uint32_t nbx = S0 >> 3, bpt = nbx * nbx;
    // (preferred to bulk rows where both apply: 64 box copies per item instead of 256 row copies,
    // C3 g = 2 ops 13.5-14.5 ms with rows vs 12.0-12.8 ms with boxes)
    G.tq = 1;
    if (tma && hform && D == 8 && M == 32 && (S0 == 8 || S0 == 16) && NT * bpt == 64 && G.logRun >= 3 &&
        G.nxb == 8 && G.nyb == 8) {
        // hform3 (k = 3 Kraus sums) with 8 x 8 boxes on two or three grid targets: 64 box copies per
        // item instead of 512 bulk rows of 128 / 256 B.  Component ci of block (xb, yb) sits at
        // sub-block position (xb | xr, yb | yc) of logical tile t; the box is (x >> 3, y >> 3) of the
        // tile (stored orientation: transposed for adjoint tiles).  A quarter-warp of a hform3 load /
        // store touches 2 blocks (yb, yb' at one xb) x the 4 components of its lanes (hin / hout);
        // pick each slot's swizzle phase by coordinate descent so those 8 accesses fall into
        // distinct 16-byte bank groups, for all-direct and all-adjoint units.
        G.tma = 1;
        G.bulk = 0;
        const HForm& hf = hform_tables();
        for (uint32_t ci = 0; ci < 64; ++ci) {
            const uint32_t rho = ci >> 3, gam = ci & 7u, t = (rho >> kin) * NG + (gam >> kin);
            G.hsd[ci] = (uint8_t)(t * bpt);
            G.hsa[ci] = (uint8_t)((G.xs_in[rho & kinm] << 4) | G.y_in[gam & kinm]);
        }
        uint8_t phi[64];
        for (uint32_t t = 0; t < 64; ++t)
            phi[t] = (uint8_t)((2 * t) & 7u);
        const uint32_t nbx_ = nbx;
        auto chunk = [&](uint32_t ci, uint32_t xb, uint32_t yb, uint32_t ori) {
            uint32_t x = xb | (G.hsa[ci] >> 4), y = yb | (G.hsa[ci] & 15u);
            if (ori)
                std::swap(x, y);
            const uint32_t sl = G.hsd[ci] + (x >> 3) * nbx_ + (y >> 3);
            return (y & 7u) ^ (((x & 7u) + phi[sl]) & 7u);
        };
        auto hcost = [&]() {
            uint32_t cost = 0;
            for (uint32_t xi = 0; xi < 8; xi += 3)  // sample passes (block row xi of the sub-block)
                for (uint32_t ori = 0; ori < 2; ++ori)
                    for (uint32_t ins = 0; ins < 32; ++ins)  // 16 loads (j, e), 16 stores (nt, e)
                        for (uint32_t ph = 0; ph < 4; ++ph) {
                            uint32_t cnt[8] = {0}, mx = 0;
                            for (uint32_t l = 8 * ph; l < 8 * ph + 8; ++l) {
                                const uint32_t gq = l >> 2, cq = l & 3u;
                                const uint32_t ci = ins < 16 ? hf.in[16 * cq + ins]
                                                             : hf.out[2 * (4 * ((ins - 16) >> 1) + cq) + (ins & 1u)];
                                mx = std::max(mx, ++cnt[chunk(ci, G.xb_tab[xi], G.yb_tab[gq], ori)]);
                            }
                            cost += mx;
                        }
            return cost;
        };
        const uint64_t key = search_key(G, 4, 0);
        std::array<uint8_t, 65> cached;
        const bool hit = search_get(key, cached);
        if (hit)
            for (uint32_t q = 0; q < 64; ++q)
                phi[q] = cached[q];
        const uint32_t ideal = 3u * 2u * 32u * 4u;
        uint32_t cur = hit ? 0u : hcost();
        for (uint32_t pass = 0; pass < 4 && cur > ideal; ++pass)
            for (uint32_t q = 0; q < 64; ++q) {
                uint8_t bv = phi[q];
                for (uint32_t v = 0; v < 8; ++v) {
                    phi[q] = (uint8_t)v;
                    const uint32_t c = hcost();
                    if (c < cur) {
                        cur = c;
                        bv = (uint8_t)v;
                    }
                }
                phi[q] = bv;
            }
        if (!hit) {
            std::array<uint8_t, 65> v{};
            for (uint32_t q = 0; q < 64; ++q)
                v[q] = phi[q];
            search_put(key, v);
        }
        uint32_t k = 0;  // slots in order of phase (see below)
        for (uint32_t v = 0; v < 8; ++v)
            for (uint32_t q = 0; q < 64; ++q)
                if (phi[q] == v) {
                    G.cdir[q] = (uint16_t)(k++ * 64 + v * 8);
                    G.tsk[q] = (uint8_t)v;
                }
    } else if (tma && prog && M == 32 && G.logRun >= 3 && S0 >= 8 && NT * bpt <= 64) {
        // grid programs: consecutive threads take consecutive positions of one logical tile, so
        // any phase is conflict-free in both placements (the in-box chunk y ^ x, resp. x ^ y, is a
        // bijection along the row): phase 0, boxes packed
        G.tma = 1;
        G.bulk = 0;
        for (uint32_t q = 0; q < NT * bpt; ++q) {
            G.cdir[q] = (uint16_t)(q * 64);
            G.tsk[q] = 0;
        }
    } else if (tma && dmma && !hform && D == 8 && M == 32 && G.logRun >= 3 && (S0 == 8 || S0 == 16) && NT * bpt <= 64 &&
        (!(((S0 - 1) & ~xs_tmask) & 8u) || (G.nxb == 8 && G.nyb == 8))) {
        G.bulk = 0;
        G.tq = (((S0 - 1) & ~xs_tmask) & 8u) ? 4 : 1;  // bit 3 free: it selects the box per block
        // 8 x 8 boxes through the tensor map (SWIZZLE_128B): slot = (tile, box) with a swizzle phase
        // phi (16-B chunk c of box row x lands at c ^ ((x + phi) & 7)).  The DMMA patterns touch the
        // in-box positions of (block base | component offset) in direct or transposed placement;
        // pick the phases by coordinate descent over sample blocks and both placements
        G.tma = 1;
        const uint32_t nslot = NT * bpt;
        uint8_t phi[64];
        for (uint32_t q = 0; q < nslot; ++q) {
            const uint32_t t = q / bpt, b = q % bpt;
            phi[q] = (uint8_t)(((t >> g) + (t & (NG - 1)) + (b / nbx) + 2 * (b % nbx)) & 7u);
        }
        const uint32_t smp[4][2] = {{0, 0}, {7 & (G.nxb - 1), 5 & (G.nyb - 1)}, {3 & (G.nxb - 1), 6 & (G.nyb - 1)},
                                    {6 & (G.nxb - 1), 1 & (G.nyb - 1)}};
        auto tcost = [&]() {
            uint32_t cost = 0;
            for (uint32_t sb = 0; sb < 4; ++sb)
                for (uint32_t ori = 0; ori < 2; ++ori)
                    for (int pat = 0; pat < 2; ++pat)
                        for (uint32_t j = 0; j < 2; ++j)
                            for (uint32_t ph = 0; ph < 4; ++ph) {
                                uint32_t cnt[8] = {0}, mx = 0;
                                for (uint32_t l = 8 * ph; l < 8 * ph + 8; ++l) {
                                    const uint32_t gq = l >> 2, cq = l & 3;
                                    const uint32_t row = pat ? gq : 2 * cq + j, col = pat ? 2 * cq + j : gq;
                                    const uint32_t t = G.ttr[row * 8 + col];
                                    const uint32_t xo = G.xb_tab[smp[sb][0]] | G.xs_in[row & kinm];
                                    const uint32_t yo = G.yb_tab[smp[sb][1]] | G.y_in[col & kinm];
                                    const uint32_t xs = ori ? yo : xo, ys = ori ? xo : yo;
                                    const uint32_t q = t * bpt + (xs >> 3) * nbx + (ys >> 3);
                                    mx = std::max(mx, ++cnt[((ys & 7u) ^ ((xs + phi[q]) & 7u))]);
                                }
                                cost += mx;
                            }
            return cost;
        };
        const uint64_t key = search_key(G, 2, G.tq);
        std::array<uint8_t, 65> cached;
        const bool hit = search_get(key, cached);
        if (hit)
            for (uint32_t q = 0; q < nslot; ++q)
                phi[q] = cached[q];
        uint32_t cur = hit ? 0u : tcost();
        for (uint32_t pass = 0; pass < 3 && cur > 128; ++pass)
            for (uint32_t q = 0; q < nslot; ++q) {
                uint8_t bv = phi[q];
                for (uint32_t v = 0; v < 8; ++v) {
                    phi[q] = (uint8_t)v;
                    const uint32_t c = tcost();
                    if (c < cur) {
                        cur = c;
                        bv = (uint8_t)v;
                    }
                }
                phi[q] = bv;
            }
        if (!hit) {
            std::array<uint8_t, 65> v{};
            for (uint32_t q = 0; q < nslot; ++q)
                v[q] = phi[q];
            search_put(key, v);
        }
        // slots in order of phase: box k at k * 1 KiB + phi * 128 B never overlaps box k + 1
        uint32_t k = 0;
        for (uint32_t v = 0; v < 8; ++v)
            for (uint32_t q = 0; q < nslot; ++q)
                if (phi[q] == v) {
                    G.cdir[q] = (uint16_t)(k++ * 64 + v * 8);
                    G.tsk[q] = (uint8_t)v;
                }
    }
    G.diag_map = (G.nxb >= 8 && G.nyb >= 8) ? 1 : 0;
    G.U = 1;
    G.logU = 0;
    G.stage_elems = G.tma ? NT * bpt * 64 + 64 : (NT * G.TS + extra + 7) & ~7u;
    G.stages = 3;
    G.nG_items = G.nU_strict << (2 * G.log_nsb_side);
}

// internal: a k = 2 Kraus sum the tensor-core gather cannot take (hs_apply_kraus falls back)
constexpr int RC_NO_KRAUS_SUM = -1000;

// Element tables of the hermitian-basis transform (hform3): lane c of a quad loads 7 mirrored pairs
// (r, c), (c, r) of the 8 x 8 block and the diagonal elements 2c, 2c + 1 (in[16 c + 2 j + e]);
// output pair q = 4 nt + c: the 28 upper pairs, then 4 pairs of diagonal elements (out[2 q + e]).
const HForm& hform_tables() {
    static const HForm tabs = [] {
    HForm t{};
    uint8_t pr[28][2];
    int np = 0;
    for (int d = 1; d < 8; ++d)  // by distance from the diagonal: a lane's pairs spread over the block
        for (int r = 0; r + d < 8; ++r) {
            pr[np][0] = (uint8_t)r;
            pr[np][1] = (uint8_t)(r + d);
            ++np;
        }
    for (int c = 0; c < 4; ++c) {
        for (int j = 0; j < 7; ++j) {
            const int p = 4 * j + c;  // interleaved: the four lanes of a k-step take neighbouring pairs
            t.in[16 * c + 2 * j] = (uint8_t)(pr[p][0] * 8 + pr[p][1]);
            t.in[16 * c + 2 * j + 1] = (uint8_t)(pr[p][1] * 8 + pr[p][0]);
        }
        t.in[16 * c + 14] = (uint8_t)((2 * c) * 9);
        t.in[16 * c + 15] = (uint8_t)((2 * c + 1) * 9);
    }
    for (int q = 0; q < 32; ++q) {
        if (q < 28) {
            t.out[2 * q] = (uint8_t)(pr[q][0] * 8 + pr[q][1]);
            t.out[2 * q + 1] = (uint8_t)(pr[q][1] * 8 + pr[q][0]);
        } else {
            t.out[2 * q] = (uint8_t)((2 * (q - 28)) * 9);
            t.out[2 * q + 1] = (uint8_t)((2 * (q - 28) + 1) * 9);
        }
    }
    return t;
    }();
    return tabs;
}
// k = 2 Kraus sums of rank 2..4: the per-operator direct form on the k = 3 gather (96 FMA per element
// per operator pair through I2 (x) L) instead of the S form (48 per element, any rank); off by
// default, kept for comparison (HS_KRAUS2_DIRECT=1)
constexpr bool g_gather_narrow_default = false;
// k = 3 Kraus sums of rank >= 4 through the direct per-operator sum (rank 4) / the three-buffer sum
// instead of the S form (HS_KRAUS3_DIRECT=1, for comparison)
const bool g_kraus3_direct = [] {
    const char* e = getenv("HS_KRAUS3_DIRECT");
    return e && atoi(e) != 0;
}();
const bool g_kraus2_direct = [] {
    const char* e = getenv("HS_KRAUS2_DIRECT");
    return e && atoi(e) != 0;
}();

// HS_DEBUG_FLAGS (diagnostics; read once).  DBG_POISON: the copy side fills every ring stage with
// NaN after its write-back has left the stage and before the next load is issued, so a transform
// that reads a stage before its load landed, or a write-back that reads after the refill started,
// puts NaN into the result (the race / synchronisation check that replaces compute-sanitizer, which
// this pool does not run: tests/test_gpu_races.py).  Schedule variants for A/B runs, same results bit
// for bit: bit 11 one quad per thread in program passes, bit 12 unskewed program tiles, bit 13 one
// barrier over all transform warps after every grid-program pass, bit 14 CX layers without sibling
// tile groups, bit 15 program passes without the shuffle pairing.
uint32_t debug_flags() {
    static const uint32_t v = [] {
        const char* e = getenv("HS_DEBUG_FLAGS");
        return e ? (uint32_t)atoi(e) : 0u;
    }();
    return v;
}

// Persistent-grid size: the SM count, or HS_DEBUG_GRID (tests: a different number of CTAs takes a
// different share of the items, so inter-CTA ordering bugs change the result)
int sm_count(int device) {
    static const int grid_override = [] {
        const char* e = getenv("HS_DEBUG_GRID");
        return e ? atoi(e) : 0;
    }();
    if (grid_override > 0)
        return grid_override;
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

// Shard prelude of every launch: a cross-shard operation reads the group members' tiles -- in
// place (peer mode: their current buffers; the result goes to this shard's other buffer) or from
// the exchange slots of the last exchange.  carry_over: tiles the operation leaves untouched must be
// copied into the output buffer first (monomials, three-buffer Kraus sums in peer mode).
int shard_prelude(hs_state* h, const Geo& G0, bool carry_over, Geo& G) {
    const bool peer = G0.cmask && h->peer_mode;
    if (peer) {
        for (uint32_t d = 1; d < 32; ++d)
            if (!(d & ~G0.cmask) && !h->peer_buf[h->shard ^ d][h->flip])
                return set_err(HS_ERR_INVALID, "peer mode: a group member's buffers are not registered");
    } else if (G0.cmask && (!h->recv || (G0.cmask & ~h->recv_mask) ||
                            h->recv_slots < (1u << __builtin_popcount(h->recv_mask)) - 1))
        return set_err(HS_ERR_INVALID, "cross-shard operation: exchange with the group's shards first");
    G = G0;
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
        if (carry_over)  // tiles a monomial leaves untouched must carry over
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
    G.dbg = debug_flags() & (DBG_POISON | 2048u | 32768u);  // the pipeline takes the stage-poisoning bit, bit 11 (one-quad program loop) and bit 15 (no paired passes)
    return HS_OK;
}

template <int K, int MODE, int NS>
int launch_impl(hs_state* h, const Geo& G0, const Coef<NS>& cf, const KrausArgs& ka, int buffers) {
    Geo G;
    {
        const int rc = shard_prelude(h, G0, MODE == M_MONO || MODE == M_KRAUS, G);
        if (rc)
            return rc;
    }
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
    // k = 2 unitaries on one grid bit: the tensor-core gather (bulk rows, two copy groups) when the
    // I2 (x) L pairing applies (0.83 -> 0.70 ms at n = 14), else the whole-tile pipeline below
    // k = 3 unitaries on in-tile qubits (m = 5): items of 4 consecutive local tiles through the same
    // gather (bulk rows, DMMA) instead of the pipeline's scalar two-stage transform
    if (MODE != M_KRAUS && ((G.g >= 2 && G.slabs > 1) || (K == 3 && MODE == M_DIRECT && G.g == 1) ||
                            (K == 2 && MODE == M_DIRECT && G.g == 1) ||
                            (K == 3 && MODE == M_DIRECT && G.g == 0 && G.M == 32 && G.kin == 3))) {
        // units of 16 / 64 stored tiles (and k = 3 unitaries on one grid bit, whose 4-tile units
        // are whole gather items for the FP64 tensor transform): sub-block gather kernel for the
        // off-diagonal units, the slab kernel's wedge path for the diagonal ones
        cudaError_t e;
        Geo Gg = G;
        constexpr bool dmma = K == 3 && MODE == M_DIRECT;
        if (G.g == 0) {
            Gg.grp4 = 1;
            Gg.logNT = 2;  // four tile slots per item
            Gg.nloc_tiles = h->count >> 10;
        }
        plan_gather(Gg, dmma);
        {
            static const char* dbg = getenv("HS_DEBUG_FLAGS");
            Gg.dbg = dbg ? (uint32_t)atoi(dbg) : 0u;
        }
        // tensor maps of this shard's payload for the TMA-box staging (bit 8: off); not for ops that
        // read remote tiles (the maps cover the local payload only)
        CUtensorMap tin{}, tout{};
        const bool maps = K == 3 && (MODE == M_DIRECT || MODE == M_PROG) && !Gg.cmask && !(Gg.dbg & 256u) &&
                          Gg.M == 32 && encode_tile_map(&tin, h->d, h->count) &&
                          encode_tile_map(&tout, Gg.out, h->count);
        if (MODE == M_PROG && maps && !(Gg.dbg & 64u)) {
            const uint32_t dbgf = Gg.dbg;
            plan_gather(Gg, false, false, 0, true, true);
            Gg.dbg = dbgf;
        }
        // the warp-specialised kernel runs grid programs and the tensor-core transforms (bit 5: the
        // ping-pong kernel instead); k = 2 pairs blocks two by two in each direction, the quadrant
        // blocks (2X + R1, 2Y + C1) sitting at a constant offset qstride
        bool ws = MODE == M_PROG;
        if constexpr (K == 3 ? dmma : (K == 2 && MODE == M_DIRECT)) {
            bool quad_ok = K == 3;
            if (K == 2 && Gg.nxb >= 2 && Gg.nyb >= 2 && Gg.kin <= 1) {
                const uint32_t d = Gg.xb_tab[1] - Gg.xb_tab[0];
                quad_ok = d == Gg.yb_tab[1] - Gg.yb_tab[0];
                for (uint32_t x = 0; quad_ok && 2 * x + 1 < Gg.nxb; ++x)
                    quad_ok = Gg.xb_tab[2 * x + 1] - Gg.xb_tab[2 * x] == d && Gg.yb_tab[2 * x + 1] - Gg.yb_tab[2 * x] == d;
                Gg.qstride = d;
            }
            ws = !(Gg.dbg & 32u) && quad_ok;
            if constexpr (MODE == M_DIRECT && (K == 2 || NS == 256))
                if (cf.nk > 1 && !ws)
                    return RC_NO_KRAUS_SUM;  // the caller falls back (transfer matrix / three-buffer sum)
            if (ws && !(Gg.dbg & 64u)) {  // contiguous sub-block rows: bulk row copies (bit 6: off)
                const uint32_t qs = Gg.qstride, dbgf = Gg.dbg;
                // k = 3 sub-blocks with 128-B rows: tensor-map boxes (bit 8: off); not for ops reading
                // remote tiles (the maps cover this shard's payload only)
                plan_gather(Gg, dmma || K == 2, true, K == 2 ? qs : 0, maps);
                Gg.qstride = qs;
                Gg.dbg = dbgf;
            }
        }
        if (ws) {
            // every unit including the diagonal ones: logical (R, C), R < C, of a diagonal unit is a
            // read-only staged copy of stored (C, R), never written back (no separate wedge launch)
            Gg.ws_diag = 1;
            Gg.nG_items = Gg.grp4 ? (Gg.nloc_tiles + 3) / 4 : Gg.nU_loose << (2 * Gg.log_nsb_side);
            const size_t smem = (size_t)Gg.stages * Gg.stage_elems * sizeof(double2) + (Gg.tma ? 1024 : 0);
            auto kw = gather_ws_kernel<K, NS, MODE == M_PROG ? M_PROG : M_DIRECT>;
            if constexpr ((K == 3 && MODE == M_DIRECT) || (K == 2 && MODE == M_DIRECT))
                if (Gg.bulk)
                    kw = gather_ws_kernel<K, NS, M_DIRECT, true>;
            if constexpr (K == 2 && MODE == M_DIRECT && NS == 64)
                if (cf.nk > 1) {
                    if (!Gg.bulk)
                        return RC_NO_KRAUS_SUM;
                    kw = gather_ws_kernel<K, NS, M_DIRECT, true, false, true>;
                }
            if constexpr (K == 3 && MODE == M_PROG)
                if (Gg.tma)
                    kw = gather_ws_kernel<K, NS, M_PROG, true, true>;
            if constexpr (K == 3 && MODE == M_DIRECT)
                if (Gg.tma)
                    kw = gather_ws_kernel<K, NS, M_DIRECT, true, true>;
            if constexpr (K == 3 && MODE == M_DIRECT && NS == 256)
                if (cf.nk > 1)  // last: overrides the unitary choices above; k = 3 Kraus sums in every staging mode (the same arithmetic sharded or not)
                    kw = Gg.tma ? gather_ws_kernel<K, NS, M_DIRECT, true, true, true>
                                : Gg.bulk ? gather_ws_kernel<K, NS, M_DIRECT, true, false, true>
                                          : gather_ws_kernel<K, NS, M_DIRECT, false, false, true>;
            // k = 3 on bulk / TMA staging: 8 transform warps at 128 registers instead of 16 at 80
            // (HS_GATHER_NARROW=0/1 overrides the default)
            unsigned threads = 768;
            if constexpr (K == 3 && MODE == M_DIRECT) {
                static const int narrow_env = [] {
                    const char* e = getenv("HS_GATHER_NARROW");
                    return e ? atoi(e) : -1;
                }();
                const bool narrow = narrow_env >= 0 ? narrow_env != 0 : g_gather_narrow_default;
                if (narrow && Gg.bulk) {
                    threads = 512;
                    if constexpr (NS == 256)
                        kw = cf.nk > 1 ? (Gg.tma ? gather_ws_kernel<K, NS, M_DIRECT, true, true, true, true>
                                                 : gather_ws_kernel<K, NS, M_DIRECT, true, false, true, true>)
                                       : (Gg.tma ? gather_ws_kernel<K, NS, M_DIRECT, true, true, false, true>
                                                 : gather_ws_kernel<K, NS, M_DIRECT, true, false, false, true>);
                    else
                        kw = Gg.tma ? gather_ws_kernel<K, NS, M_DIRECT, true, true, false, true>
                                    : gather_ws_kernel<K, NS, M_DIRECT, true, false, false, true>;
                }
            }
            e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
            if (e != cudaSuccess)
                return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(gather_ws): ") + cudaGetErrorString(e));
            const uint64_t grid = std::min<uint64_t>(Gg.nG_items, (uint64_t)sm_count(h->device));
            if (grid) {
                kw<<<(unsigned)grid, threads, smem, h->stream>>>(Gg, cf, h->d, tin, tout);
                g_launches.fetch_add(1, std::memory_order_relaxed);
                e = cudaGetLastError();
                if (e != cudaSuccess)
                    return set_err(HS_ERR_CUDA, std::string("gather_ws_kernel launch: ") + cudaGetErrorString(e));
            }
            return HS_OK;
        }
        if (K == 2 && G.g == 1)
            goto pipe_path;  // no pairing (or the ping-pong debug switch): whole-tile pipeline
        if (G.nD_items) {  // diagonal units: the slab kernel's wedge path
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
        if (Gg.nG_items) {
            const size_t smem = (size_t)Gg.stages * Gg.stage_elems * sizeof(double2);
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
pipe_path:
    if constexpr (MODE == M_DIRECT && (K == 2 || NS == 256))
        if (cf.nk > 1)
            return RC_NO_KRAUS_SUM;  // the pipeline's direct transform applies one operator
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

// k = 2 Kraus sum in S form (16 x 16 transfer matrix) on the tensor-core gather, every regime:
// whole tiles (no grid target: items of 4 local tiles; one grid target: 2 x 2-tile units) or 16 x 16
// sub-blocks of 4 x 4-tile units (two grid targets), bulk-row staging, sform2 transform.
int launch_sform2_impl(hs_state* h, const Geo& G0, const Coef<256>& cf) {
    if (h->m != 5)
        return RC_NO_KRAUS_SUM;
    Geo G;
    {
        const int rc = shard_prelude(h, G0, false, G);
        if (rc)
            return rc;
    }
    if (G.g == 0) {
        G.grp4 = 1;
        G.logNT = 2;
        G.nloc_tiles = h->count >> 10;
    }
    plan_gather(G, false, true, 0, false, false, true);
    {
        static const char* dbg = getenv("HS_DEBUG_FLAGS");
        G.dbg = dbg ? (uint32_t)atoi(dbg) : 0u;
    }
    if (!G.bulk)
        return RC_NO_KRAUS_SUM;
    if (G.dbg & 512u)
        fprintf(stderr, "sform2: g=%u in_mask=%x S0=%u TS=%u s8=%u xfast=%u bank cost %u (ideal %u) stage %u elems\n", G.g,
                G.in_mask, G.S0, G.TS, G.s8, G.sf_xfast, G.sf_cost, G.sf_ideal, G.stage_elems);
    G.ws_diag = 1;
    G.nG_items = G.grp4 ? (G.nloc_tiles + 3) / 4 : G.nU_loose << (2 * G.log_nsb_side);
    const size_t smem = (size_t)G.stages * G.stage_elems * sizeof(double2);
    auto kw = gather_ws_kernel<2, 256, M_SF2, true>;
    cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(sform2): ") + cudaGetErrorString(e));
    const uint64_t grid = std::min<uint64_t>(G.nG_items, (uint64_t)sm_count(h->device));
    if (grid) {
        CUtensorMap tin{}, tout{};
        kw<<<(unsigned)grid, 512, smem, h->stream>>>(G, cf, h->d, tin, tout);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("gather_ws_kernel(sform2) launch: ") + cudaGetErrorString(e));
    }
    return HS_OK;
}

// k = 3 Kraus sum in S form (64 x 64 transfer matrix, fragments at `frag` in device memory) on the
// tensor-core gather, bulk-row staging in every regime (128-B rows for three grid targets: this
// transform is bound by the FP64 pipe, not by the copies), two ring stages + the fragments.
int launch_sform3_impl(hs_state* h, const Geo& G0, const double* frag) {
    if (h->m != 5)
        return RC_NO_KRAUS_SUM;
    Geo G;
    {
        const int rc = shard_prelude(h, G0, false, G);
        if (rc)
            return rc;
    }
    if (G.g == 0) {
        G.grp4 = 1;
        G.logNT = 2;
        G.nloc_tiles = h->count >> 10;
    }
    // two / three grid targets: 8 x 8 TMA boxes instead of 128-B bulk rows where plan_gather can
    // place them (local tiles only: the tensor maps cover this shard's payload; HS_DEBUG_FLAGS bit 8:
    // off)
    const uint32_t dbgf = debug_flags();
    CUtensorMap tin{}, tout{};
    const bool maps = G.g >= 2 && !G.cmask && !(dbgf & 256u) && G.M == 32 && encode_tile_map(&tin, h->d, h->count) &&
                      encode_tile_map(&tout, G.out, h->count);
    plan_gather(G, true, true, 0, maps, false, false, 3, true);
    G.dbg = dbgf;
    if (!G.bulk && !G.tma)
        return RC_NO_KRAUS_SUM;
    G.sf3 = frag;
    G.ws_diag = 1;
    G.nG_items = G.grp4 ? (G.nloc_tiles + 3) / 4 : G.nU_loose << (2 * G.log_nsb_side);
    const size_t smem = (size_t)2 * G.stage_elems * sizeof(double2) + 4096 * sizeof(double) + (G.tma ? 1024 : 0);
    auto kw = G.tma ? gather_ws_kernel<3, 64, M_SF3, true, true> : gather_ws_kernel<3, 64, M_SF3, true>;
    cudaError_t e = cudaFuncSetAttribute(kw, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, std::string("cudaFuncSetAttribute(sform3): ") + cudaGetErrorString(e));
    const uint64_t grid = std::min<uint64_t>(G.nG_items, (uint64_t)sm_count(h->device));
    if (grid) {
        Coef<64> cf{};
        kw<<<(unsigned)grid, 512, smem, h->stream>>>(G, cf, h->d, tin, tout);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        e = cudaGetLastError();
        if (e != cudaSuccess)
            return set_err(HS_ERR_CUDA, std::string("gather_ws_kernel(sform3) launch: ") + cudaGetErrorString(e));
    }
    return HS_OK;
}

// R of a k = 3 Kraus set in hform3's fragment order, on the device.  Cached per state by the bytes
// of the Kraus set (a noise channel is typically applied to many qubit triples): a hit costs no host
// work, no copy and no synchronisation, and is allowed inside a graph capture (the buffer lives as
// long as the state); a miss builds R on the host and uploads it synchronously (refused while
// capturing).
int hform_fragments(hs_state* h, int nops, const double2* L, const double** out) {
    uint64_t key = 1469598103934665603ull ^ (uint64_t)nops;
    const unsigned char* bytes = reinterpret_cast<const unsigned char*>(L);
    for (size_t b = 0; b < (size_t)nops * 64 * sizeof(double2); ++b)
        key = (key ^ bytes[b]) * 1099511628211ull;
    for (const auto& e : h->hcache)
        if (e.key == key && e.nops == nops && std::memcmp(e.ops.data(), L, e.ops.size() * sizeof(double2)) == 0) {
            *out = e.dev;
            return HS_OK;
        }
    {
        cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
        CUDA_TRY(cudaStreamIsCapturing(h->stream, &cs));
        if (cs != cudaStreamCaptureStatusNone)
            return set_err(HS_ERR_UNSUPPORTED, "k = 3 Kraus set not yet seen by this state: apply it once before capturing");
    }
    const HForm& hf = hform_tables();
    // input coordinate (ks, c): hermitian basis element E; output coordinate (nt, n): a real
    // coordinate of S(E) = sum_a L_a E L_a^dagger.  E has two nonzeros (one on the diagonal).
    std::vector<double> frag(4096);
    for (int c = 0; c < 4; ++c)
        for (int ks = 0; ks < 16; ++ks) {
            const int j = ks >> 1, which = ks & 1;
            const int e0 = hf.in[16 * c + 2 * j], e1 = hf.in[16 * c + 2 * j + 1];
            int pos[2];
            double2 val[2];
            int nz = 0;
            if (j < 7) {  // (|r><c| + |c><r|) / 2  or  (i|r><c| - i|c><r|) / 2, e0 = (r, c), e1 = (c, r)
                pos[0] = e0;
                val[0] = which ? make_double2(0.0, 0.5) : make_double2(0.5, 0.0);
                pos[1] = e1;
                val[1] = which ? make_double2(0.0, -0.5) : make_double2(0.5, 0.0);
                nz = 2;
            } else {      // |d><d|
                pos[0] = which ? e1 : e0;
                val[0] = make_double2(1.0, 0.0);
                nz = 1;
            }
            double2 Y[64];
            for (int x = 0; x < 8; ++x)
                for (int y = 0; y < 8; ++y) {
                    double yr = 0.0, yi = 0.0;
                    for (int a = 0; a < nops; ++a)
                        for (int z = 0; z < nz; ++z) {
                            const int u = pos[z] >> 3, v = pos[z] & 7;
                            const double2 ee = val[z], lx = L[a * 64 + x * 8 + u], ly = L[a * 64 + y * 8 + v];
                            const double tr = lx.x * ee.x - lx.y * ee.y, ti = lx.x * ee.y + lx.y * ee.x;  // lx * ee
                            yr += tr * ly.x + ti * ly.y;  // * conj(ly)
                            yi += ti * ly.x - tr * ly.y;
                        }
                    Y[x * 8 + y] = make_double2(yr, yi);
                }
            for (int nt = 0; nt < 8; ++nt)
                for (int g = 0; g < 8; ++g) {
                    const int q = 4 * nt + (g >> 1), jo = g & 1;
                    const int o0 = hf.out[2 * q], o1 = hf.out[2 * q + 1];
                    const double v = nt < 7 ? (jo ? Y[o0].y : Y[o0].x) : (jo ? Y[o1].x : Y[o0].x);
                    frag[(ks * 8 + nt) * 32 + g * 4 + c] = v;
                }
        }
    if (h->hcache.size() >= HCACHE_MAX) {
        // cache full (32 MiB of fragments): a scratch buffer, uploaded in stream order and not cached
        // (cached entries are never freed before the state, so captured graphs stay valid)
        if (!h->hscratch)
            CUDA_TRY(cudaMalloc(&h->hscratch, frag.size() * sizeof(double)));
        CUDA_TRY(cudaMemcpyAsync(h->hscratch, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice,
                                 h->stream));
        CUDA_TRY(cudaStreamSynchronize(h->stream));  // `frag` is freed on return
        *out = h->hscratch;
        return HS_OK;
    }
    HCacheEntry e;
    e.key = key;
    e.nops = nops;
    e.ops.assign(L, L + (size_t)nops * 64);
    CUDA_TRY(cudaMalloc(&e.dev, frag.size() * sizeof(double)));
    const cudaError_t ce = cudaMemcpy(e.dev, frag.data(), frag.size() * sizeof(double), cudaMemcpyHostToDevice);
    if (ce != cudaSuccess) {
        cudaFree(e.dev);
        return set_err(HS_ERR_CUDA, std::string("hform fragments: ") + cudaGetErrorString(ce));
    }
    h->hcache.push_back(std::move(e));
    *out = h->hcache.back().dev;
    return HS_OK;
}

// After a launch: peer mode makes the output buffer current; an exchange licenses one operation.
int after_launch(hs_state* h, const Geo& G0, int rc) {
    if (rc == HS_OK && G0.cmask && h->peer_mode) {
        h->flip ^= 1u;
        h->d = h->buf[h->flip];
    }
    if (rc == HS_OK && G0.cmask && !h->peer_mode)
        h->recv_mask = 0;
    return rc;
}

int launch_sform2(hs_state* h, const Geo& G0, const Coef<256>& cf) {
    return after_launch(h, G0, launch_sform2_impl(h, G0, cf));
}
int launch_sform3(hs_state* h, const Geo& G0, const double* frag) {
    return after_launch(h, G0, launch_sform3_impl(h, G0, frag));
}

// One operation's kernels.  Peer mode: the result went to the other buffer, which becomes current.
template <int K, int MODE, int NS>
int launch(hs_state* h, const Geo& G0, const Coef<NS>& cf, const KrausArgs& ka, int buffers) {
    return after_launch(h, G0, launch_impl<K, MODE, NS>(h, G0, cf, ka, buffers));
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

void user_plan(const hs_state* h, hs_plan* plan);
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
    user_plan(h, plan);
    return HS_OK;
}

uint64_t state_bytes(const hs_state* h) { return h->count * sizeof(double2); }

// m > 5: the user-layout payload (mu) in a stream-ordered temporary, from / into the internal m = 5
// layout (retile_kernel, engine_convert.cuh).  The temporary is freed stream-ordered as well.
bool big_tiles(const hs_state* h) { return h->mu > h->m; }
struct UserTemp {
    double2* p = nullptr;
    cudaStream_t s = nullptr;
    void release() {
        if (p)
            cudaFreeAsync(p, s);
        p = nullptr;
    }
    ~UserTemp() { release(); }
};
int user_alloc(const hs_state* h, UserTemp& t) {
    t.s = h->stream;
    if (cudaMallocAsync(&t.p, h->ucount * sizeof(double2), h->stream) != cudaSuccess) {
        cudaGetLastError();
        t.p = nullptr;
        return set_err(HS_ERR_NOMEM, "user-layout staging buffer (tile exponent > 5)");
    }
    return HS_OK;
}
int retile_launch(double2* dst, uint32_t m2, uint64_t cnt2, uint64_t N, const double2* src, uint32_t m1,
                  cudaStream_t s);
int to_user(const hs_state* h, UserTemp& t) {  // t.p <- the operator in the mu layout
    int rc = user_alloc(h, t);
    return rc ? rc : retile_launch(t.p, (uint32_t)h->mu, h->ucount, h->N, h->d, (uint32_t)h->m, h->stream);
}
int from_user(hs_state* h, const double2* u) {  // the operator <- u in the mu layout
    return retile_launch(h->d, (uint32_t)h->m, h->count, h->N, u, (uint32_t)h->mu, h->stream);
}
// the path tag, grid-target count and subcase counters as the reference reports them for the
// user's tile exponent (kernels.cpp:448-549 classify by a < m)
void user_plan(const hs_state* h, hs_plan* plan) {
    if (!plan || !big_tiles(h))
        return;
    Geo U{};
    U.k = (uint32_t)plan->k;
    U.g = 0;
    for (int i = 0; i < plan->k; ++i)
        if (plan->targets[i] >= (uint32_t)h->mu)
            U.gr_pos[U.g++] = plan->targets[i] - (uint32_t)h->mu;
    U.nb = h->uG >> U.g;
    plan->grid_bits = (int)U.g;
    if (plan->path == HS_PATH_TILED_INTRA || plan->path == HS_PATH_TILED_CROSS || plan->path == HS_PATH_TILED_MIXED)
        plan->path = U.g == 0 ? HS_PATH_TILED_INTRA : U.g == U.k ? HS_PATH_TILED_CROSS : HS_PATH_TILED_MIXED;
    if (g_plan_subcases)
        count_subcases(h, U, plan->subcases);
}

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
    if (m > 5 && nshards != 1)
        return set_err(HS_ERR_UNSUPPORTED, "tile exponents m > 5 are supported for unsharded operators");
    const int mu = m;
    if (m > 5)
        m = 5;  // internal layout (see hs_state::mu)
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
    h->mu = mu;
    h->ucount = h->count;
    h->uG = h->G;
    if (mu > m) {
        const uint64_t Mu = 1ull << mu;
        h->uG = h->N >= Mu ? h->N / Mu : 1;
        h->ucount = h->uG * (h->uG + 1) / 2 * Mu * Mu;
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
    for (auto& e : h->hcache)
        cudaFree(e.dev);
    cudaFree(h->hscratch);
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
        *m = h->mu;
    if (count)
        *count = h->ucount;
    if (grid)
        *grid = h->uG;
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
    if (offset > h->ucount || count > h->ucount - offset)
        return set_err(HS_ERR_RANGE, "upload range exceeds the payload");
    DeviceGuard dg(h->device);
    if (big_tiles(h)) {  // into the user-layout image of the operator, then back to the m = 5 layout
        UserTemp t;
        int rc = count == h->ucount ? user_alloc(h, t) : to_user(h, t);
        if (rc)
            return rc;
        CUDA_TRY(cudaMemcpyAsync(t.p + offset, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
        rc = from_user(h, t.p);
        if (rc)
            return rc;
    } else {
        CUDA_TRY(cudaMemcpyAsync(h->d + offset, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return HS_OK;
}

int hs_state_download_range(const hs_state* h, double* host, uint64_t offset, uint64_t count) {
    if (!h || (!host && count))
        return set_err(HS_ERR_INVALID, "null argument");
    if (offset > h->ucount || count > h->ucount - offset)
        return set_err(HS_ERR_RANGE, "download range exceeds the payload");
    DeviceGuard dg(h->device);
    if (big_tiles(h)) {
        UserTemp t;
        const int rc = to_user(h, t);
        if (rc)
            return rc;
        CUDA_TRY(cudaMemcpyAsync(host, t.p + offset, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    } else {
        CUDA_TRY(cudaMemcpyAsync(host, h->d + offset, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    }
    CUDA_TRY(cudaStreamSynchronize(h->stream));
    return HS_OK;
}

int hs_state_upload(hs_state* h, const double* host, uint64_t count) {
    if (h && count != h->ucount)
        return set_err(HS_ERR_INVALID, "payload length mismatch");
    return hs_state_upload_range(h, host, 0, count);
}

int hs_state_download(const hs_state* h, double* host, uint64_t count) {
    if (h && count != h->ucount)
        return set_err(HS_ERR_INVALID, "payload length mismatch");
    return hs_state_download_range(h, host, 0, count);
}

int hs_state_upload_async(hs_state* h, const double* host, uint64_t count) {
    if (!h || !host || count != h->ucount)
        return set_err(HS_ERR_INVALID, "bad upload arguments");
    DeviceGuard dg(h->device);
    if (big_tiles(h)) {
        UserTemp t;
        const int rc = user_alloc(h, t);
        if (rc)
            return rc;
        CUDA_TRY(cudaMemcpyAsync(t.p, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
        return from_user(h, t.p);
    }
    CUDA_TRY(cudaMemcpyAsync(h->d, host, count * sizeof(double2), cudaMemcpyHostToDevice, h->stream));
    return HS_OK;
}

int hs_state_download_async(const hs_state* h, double* host, uint64_t count) {
    if (!h || !host || count != h->ucount)
        return set_err(HS_ERR_INVALID, "bad download arguments");
    DeviceGuard dg(h->device);
    if (big_tiles(h)) {
        UserTemp t;
        const int rc = to_user(h, t);
        if (rc)
            return rc;
        CUDA_TRY(cudaMemcpyAsync(host, t.p, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
        return HS_OK;
    }
    CUDA_TRY(cudaMemcpyAsync(host, h->d, count * sizeof(double2), cudaMemcpyDeviceToHost, h->stream));
    return HS_OK;
}

int hs_state_copy(hs_state* dst, const hs_state* src) {
    if (!dst || !src)
        return set_err(HS_ERR_INVALID, "null state");
    if (dst->count != src->count || dst->m != src->m || dst->n != src->n || dst->mu != src->mu)
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
        // the 16 x 16 transfer matrix on the FP64 tensor path (sform2), else the scalar pipeline
        auto* cf = new Coef<256>();
        std::memcpy(cf->s, s, sizeof(cf->s));
        rc = launch_sform2(h, G, *cf);
        if (rc == RC_NO_KRAUS_SUM)
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
// transfer (s diagonal used), 3 / 4 real (00,11)/(01,10) transfer / real (00,11) block with a complex
// diagonal on (01,10).  Equivalent to applying the steps one by one (hs_apply_transfer).
int hs_apply_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s, hs_plan* plan) {
    if (!h || nsteps < 1 || nsteps > 16 || !kinds || !bits || !s)
        return set_err(HS_ERR_INVALID, "bad program");
    const uint32_t edge = std::min<uint32_t>((uint32_t)h->m, (uint32_t)h->n);
    for (int p = 0; p < nsteps; ++p) {
        if (bits[p] >= edge)
            return set_err(HS_ERR_RANGE, "program steps act on in-tile qubits (< m) only");
        if (kinds[p] < 0 || kinds[p] > 5)
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
    // four whole 32 x 32 tiles per item: one spare element between them puts consecutive tiles one
    // 16-B bank group apart (pipe_kernel's program passes on qubits 0 and 1 use it)
    if (G.M == 32 && G.SR == G.M && G.TS == G.M * G.M && !G.g && !(debug_flags() & 4096u)) {  // bit 12: dense tiles
        G.TS = G.M * G.M + 1;
        G.stage_elems = ((G.U << G.logNT) * G.TS + 7) & ~7u;
        G.stages = std::min<uint32_t>(MAX_STAGES, (200u * 1024u / 16u) / G.stage_elems);
    }
    int rc = launch<1, M_PROG, 256>(h, G, *cf, ka, 1);
    delete cf;
    if (rc)
        return rc;
    return finish_plan(h, G, 1, bits, HS_PATH_TILED_INTRA, plan, 2 * state_bytes(h));
}

// CX layer (SURVEY 8f fusion): CX gates on disjoint qubit pairs in ONE in-place pass
// (cx_layer_kernel); equal to applying them one by one (native.cpp:433-549 per gate), bit for bit.
// Single-GPU states.
int hs_apply_cx_layer(hs_state* h, int npairs, const uint32_t* controls, const uint32_t* targets, hs_plan* plan) {
    if (!h || npairs < 1 || npairs > 32 || !controls || !targets)
        return set_err(HS_ERR_INVALID, "bad CX layer (1 .. 32 pairs)");
    if (h->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "CX layers run on single-GPU states");
    uint64_t used = 0;
    CxLayer L{};
    L.n = (uint32_t)npairs;
    for (int k = 0; k < npairs; ++k) {
        if (controls[k] >= (uint32_t)h->n || targets[k] >= (uint32_t)h->n)
            return set_err(HS_ERR_RANGE, "CX layer: qubit out of range");
        const uint64_t b = (1ull << controls[k]) | (1ull << targets[k]);
        if (controls[k] == targets[k] || (used & b))
            return set_err(HS_ERR_INVALID, "CX layer: the pairs must be disjoint");
        used |= b;
        L.c[k] = controls[k];
        L.t[k] = targets[k];
        // sibling groups (cx_layer_kernel): in-tile controls 0 / 1 with a grid target; bit 14: off
        // (controls 0 .. 2: partner runs of 16 / 32 / 64 B; the first two such pairs; measured at n = 17)
        if (h->m >= 3 && controls[k] < 3 && targets[k] >= (uint32_t)h->m && !(debug_flags() & 16384u) &&
            __builtin_popcount(L.gmask) < 2)
            L.gmask |= 1u << (targets[k] - (uint32_t)h->m);
    }
    DeviceGuard dg(h->device);
    const uint64_t ntiles = h->count >> (2 * h->m);
    const uint64_t grid = std::min<uint64_t>(ntiles, (uint64_t)sm_count(h->device) * 8);
    cx_layer_kernel<<<(unsigned)grid, 256, 0, h->stream>>>(h->d, ntiles, (uint32_t)h->m, (uint32_t)h->n, L);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, std::string("cx_layer_kernel launch: ") + cudaGetErrorString(e));
    if (plan) {
        std::memset(plan, 0, sizeof(*plan));
        plan->path = HS_PATH_NATIVE_PERMUTATION;
        plan->k = 2;
        plan->targets[0] = std::min(controls[0], targets[0]);
        plan->targets[1] = std::max(controls[0], targets[0]);
        plan->touched_bytes = 2 * state_bytes(h);
    }
    return HS_OK;
}

// Fused grid program: one k = 1 step on each of nsteps (<= 3) distinct grid qubits
// (>= m), applied in ONE pass: the units of the g = nsteps grid bits are gathered (warp-specialised
// gather) and the steps run one after another on the staged logical tiles.  kinds / s as for
// hs_apply_program.  Single-GPU states only (a cross-shard step would need its own exchange).
int hs_apply_grid_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s,
                          hs_plan* plan) {
    if (!h || nsteps < 2 || nsteps > 16 || !kinds || !bits || !s)
        return set_err(HS_ERR_INVALID, "bad grid program (2 .. 16 steps on 2 or 3 qubits)");
    if (h->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "grid programs run on single-GPU states");
    uint32_t t[3];
    int nq = 0;
    for (int p = 0; p < nsteps; ++p) {
        if (bits[p] < (uint32_t)h->m || bits[p] >= (uint32_t)h->n)
            return set_err(HS_ERR_RANGE, "grid program steps act on grid qubits (>= m) only");
        if (kinds[p] < 0 || kinds[p] > 5)
            return set_err(HS_ERR_INVALID, "bad program step kind");
        if (p > 0 && bits[p] == bits[p - 1])
            continue;  // the qubit's chain continues
        for (int q = 0; q < nq; ++q)
            if (t[q] == bits[p])
                return set_err(HS_ERR_INVALID, "grid program: a qubit's steps must be consecutive");
        if (nq == 3)
            return set_err(HS_ERR_INVALID, "grid program: at most 3 qubits");
        t[nq++] = bits[p];
    }
    if (nq < 2)
        return set_err(HS_ERR_INVALID, "grid program: 2 or 3 qubits (one qubit: hs_apply_transfer)");
    std::sort(t, t + nq);
    if (h->m != 5 || ((uint64_t)1 << (2 * nq)) * 1024 < 4096)
        return set_err(HS_ERR_UNSUPPORTED, "grid programs need 32 x 32 tiles");
    DeviceGuard dg(h->device);
    Geo G;
    plan_geo(h, nq, t, G, 1);
    auto* cf = new Coef<256>();
    for (int p = 0; p < nsteps; ++p) {
        std::memcpy(cf->s + 16 * p, s + 32 * p, 16 * sizeof(double2));
        uint32_t l = 0;
        while (t[l] != bits[p])
            ++l;
        cf->pbit[p] = (uint8_t)l;  // local grid bit of the step
        cf->pkind[p] = (uint8_t)kinds[p];
    }
    cf->nsteps = (uint32_t)nsteps;
    int rc = launch<3, M_PROG, 256>(h, G, *cf, KrausArgs{nullptr, 0}, 1);
    delete cf;
    if (rc)
        return rc;
    return finish_plan(h, G, nq, t, HS_PATH_TILED_CROSS, plan, 2 * state_bytes(h));
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
    } else if (k == 2 && G.g == 0 && h->m == 5 && h->n >= h->m + 4 && (uint32_t)(h->n - h->m) > h->Plog) {
        // both targets in-tile: run I2 (x) L on (t0, t1, m) -- the lowest grid qubit m as the most
        // significant local bit; only when m is not a shard bit (n - m > log2 P), so the promoted op
        // stays shard-local; the same choice sharded or not -- through the k = 3 tensor-core gather (bulk
        // rows): identical result up to rounding, 0.96 -> ~0.70 ms at n = 14 instead of the
        // scalar two-stage transform of the whole-tile pipeline
        uint32_t t3[3] = {t[0], t[1], (uint32_t)h->m};
        Geo G3;
        plan_geo(h, 3, t3, G3, 1);
        Coef<64> cf{};
        for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b)
                cf.s[a * 8 + b] = (a >> 2) == (b >> 2) ? U[(a & 3) * 4 + (b & 3)] : make_double2(0.0, 0.0);
        rc = launch<3, M_DIRECT, 64>(h, G3, cf, ka, 1);
    } else if (k == 2 && G.g == 2 && h->m == 5) {
        // both targets on grid bits: L (x) I2 on (m - 1, t0, t1) -- the in-tile qubit 4 as the least
        // significant local bit -- through the k = 3 gather's TMA boxes (5.4 TB/s) instead of the
        // k = 2 pairing on bulk rows (4.9 TB/s); the extra target is in-tile, so the shards an op
        // reads are those of its own targets
        uint32_t t3[3] = {(uint32_t)h->m - 1, t[0], t[1]};
        Geo G3;
        plan_geo(h, 3, t3, G3, 1);
        Coef<64> cf{};
        for (int a = 0; a < 8; ++a)
            for (int b = 0; b < 8; ++b)
                cf.s[a * 8 + b] = (a & 1) == (b & 1) ? U[(a >> 1) * 4 + (b >> 1)] : make_double2(0.0, 0.0);
        rc = launch<3, M_DIRECT, 64>(h, G3, cf, ka, 1);
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
    if (k == 3 && nops >= 3 && h->m == 5 && !g_kraus3_direct) {
        // rank >= 3: the hermitian-basis form (hform3): one real 64 x 64 matrix R on the coordinates
        // of hermitian 8 x 8 blocks, two real products per block (128 FMA per element whatever the
        // rank; the direct sum costs 48 per element per operator)
        DeviceGuard dg(h->device);
        const HForm& hf = hform_tables();
        const double* frag = nullptr;
        rc = hform_fragments(h, nops, L, &frag);
        if (rc)
            return rc;
        Geo G;
        plan_geo(h, 3, t, G, 1);
        std::memcpy(G.hf_in, hf.in, 64);
        std::memcpy(G.hf_out, hf.out, 64);
        rc = launch_sform3(h, G, frag);
        if (rc != RC_NO_KRAUS_SUM) {
            if (rc)
                return rc;
            return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
        }
    }
    if (k == 3 && nops <= 4 && h->m == 5) {
        // sum_a L_a B L_a^dagger on the k = 3 tensor-core gather (every regime), per-operator fragments
        DeviceGuard dg(h->device);
        Geo G;
        plan_geo(h, 3, t, G, 1);
        auto* cf = new Coef<256>();
        std::memcpy(cf->s, ops, (size_t)nops * 64 * sizeof(double2));
        cf->nk = (uint32_t)nops;
        KrausArgs ka{nullptr, 0};
        rc = launch<3, M_DIRECT, 256>(h, G, *cf, ka, 1);
        delete cf;
        if (rc != RC_NO_KRAUS_SUM) {
            if (rc)
                return rc;
            return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
        }
    }
    if (k == 2 && nops <= 4 && h->m == 5 && g_kraus2_direct) {
        // sum_a L_a B L_a^dagger on the tensor-core gather (I2 (x) L pairing) when it applies: at
        // least one grid target and the paired geometry; otherwise the transfer matrix below
        DeviceGuard dg(h->device);
        Geo G;
        plan_geo(h, 2, t, G, 1);
        if (G.g == 0 && h->n >= h->m + 4 && (uint32_t)(h->n - h->m) > h->Plog) {
            // both targets in-tile: the k = 3 sum of I2 (x) L_a on (t0, t1, m), as for unitaries
            // (the extra qubit m is never one of the top three: the same path sharded or not)
            uint32_t t3[3] = {t[0], t[1], (uint32_t)h->m};
            Geo G3;
            plan_geo(h, 3, t3, G3, 1);
            auto* cf = new Coef<256>();
            for (int a = 0; a < nops; ++a)
                for (int r = 0; r < 8; ++r)
                    for (int c = 0; c < 8; ++c)
                        cf->s[64 * a + r * 8 + c] =
                            (r >> 2) == (c >> 2) ? L[16 * a + (r & 3) * 4 + (c & 3)] : make_double2(0.0, 0.0);
            cf->nk = (uint32_t)nops;
            KrausArgs ka{nullptr, 0};
            rc = launch<3, M_DIRECT, 256>(h, G3, *cf, ka, 1);
            delete cf;
            if (rc != RC_NO_KRAUS_SUM) {
                if (rc)
                    return rc;
                return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
            }
        }
        if (G.g >= 1) {
            Coef<64> cf{};
            std::memcpy(cf.s, ops, (size_t)nops * 16 * sizeof(double2));
            cf.nk = (uint32_t)nops;
            KrausArgs ka{nullptr, 0};
            rc = launch<2, M_DIRECT, 64>(h, G, cf, ka, 1);
            if (rc != RC_NO_KRAUS_SUM) {
                if (rc)
                    return rc;
                return finish_plan(h, G, k, t, generic_path(G), plan, 2 * state_bytes(h));
            }
        }
    }
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

// ------------------------------------------------------------------- format conversions
// hermsim::to_dense / convert (storage.cpp:241-292) on the device: engine_convert.cuh.  Host buffers
// stream through two device staging bands of <= CV_BAND bytes (band b + 1's kernel overlaps band b's
// copy on a second stream).
namespace {
constexpr uint64_t CV_BAND = 256ull << 20;
int conv_grid(uint64_t items) { return (int)std::min<uint64_t>(std::max<uint64_t>(items, 1), 148ull * 8); }
uint64_t packed_off_h(uint64_t N, uint64_t j) { return j * N - j * (j - 1) / 2; }
uint64_t tri_h(uint64_t t) { return t * (t + 1) / 2; }

// Tile-row (dense) or tile-column (packed) bands of <= CV_BAND bytes: [b[i], b[i + 1])
std::vector<uint64_t> conv_bands(const hs_state* h, bool packed) {
    const uint64_t M = h->M, G = h->G, N = h->N, E = std::min(M, N);
    std::vector<uint64_t> b{0};
    uint64_t acc = 0;
    for (uint64_t t = 0; t < G; ++t) {
        const uint64_t j0 = t * E, j1 = std::min(N, (t + 1) * E);
        const uint64_t bytes = 16 * (packed ? packed_off_h(N, j1) - packed_off_h(N, j0) : (j1 - j0) * N);
        if (acc && acc + bytes > CV_BAND) {
            b.push_back(t);
            acc = 0;
        }
        acc += bytes;
    }
    b.push_back(G);
    return b;
}

int conv_check(const hs_state* h, const void* buf) {
    if (!h || !buf)
        return set_err(HS_ERR_INVALID, "null argument");
    if (h->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "format conversion of a sharded state: gather the shards first");
    return HS_OK;
}

// out: to_dense / to_packed of the whole state (dir = 0), or in: from_dense / from_packed (dir = 1)
int convert_linear(hs_state* h, double2* buf, bool packed, bool from, bool on_device) {
    DeviceGuard dg(h->device);
    const uint32_t m = (uint32_t)h->m;
    const uint64_t N = h->N, G = h->G, M = h->M, E = std::min(M, N);
    auto launch_band = [&](uint64_t t0, uint64_t t1, double2* p, cudaStream_t s) {
        if (!from && !packed)
            to_dense_kernel<<<conv_grid(tri_h(t1) - tri_h(t0) + (t1 - t0) * G), CV_T, 0, s>>>(h->d, m, N, G, t0, t1, p);
        else if (!from)
            to_packed_kernel<<<conv_grid((t1 - t0) * G), CV_T, 0, s>>>(h->d, m, N, G, t0, t1, p);
        else if (!packed)
            from_dense_kernel<<<conv_grid(tri_h(t1) - tri_h(t0)), CV_T, 0, s>>>(h->d, m, N, t0, t1, p);
        else
            from_packed_kernel<<<conv_grid((t1 - t0) * G), CV_T, 0, s>>>(h->d, m, N, G, t0, t1, p);
        g_launches.fetch_add(1, std::memory_order_relaxed);
        return cudaGetLastError();
    };
    auto band_bytes = [&](uint64_t t0, uint64_t t1) {
        const uint64_t j0 = t0 * E, j1 = std::min(N, t1 * E);
        return 16 * (packed ? packed_off_h(N, j1) - packed_off_h(N, j0) : (j1 - j0) * N);
    };
    auto band_elem = [&](uint64_t t0) { return packed ? packed_off_h(N, t0 * E) : t0 * E * N; };
    if (on_device) {
        CUDA_TRY(launch_band(0, G, buf, h->stream));
        return HS_OK;
    }
    const std::vector<uint64_t> b = conv_bands(h, packed);
    uint64_t cap = 0;
    for (size_t i = 0; i + 1 < b.size(); ++i)
        cap = std::max(cap, band_bytes(b[i], b[i + 1]));
    double2* stage[2] = {nullptr, nullptr};
    cudaEvent_t done[2] = {nullptr, nullptr};
    cudaError_t e = cudaSuccess;
    for (int k = 0; k < 2 && e == cudaSuccess; ++k) {
        e = cudaMalloc(&stage[k], cap);
        if (e == cudaSuccess)
            e = cudaEventCreateWithFlags(&done[k], cudaEventDisableTiming);
    }
    // band i: (from) host -> stage -> kernel, or kernel -> stage -> host; stage i & 1 is reused
    // once band i - 2 finished with it (events on the state's stream)
    for (size_t i = 0; e == cudaSuccess && i + 1 < b.size(); ++i) {
        const int k = (int)(i & 1);
        double2* hp = buf + band_elem(b[i]);
        const uint64_t bytes = band_bytes(b[i], b[i + 1]);
        if (i >= 2)
            e = cudaEventSynchronize(done[k]);  // the host copy of band i - 2 has left stage k
        if (e == cudaSuccess && from)
            e = cudaMemcpyAsync(stage[k], hp, bytes, cudaMemcpyHostToDevice, h->stream);
        if (e == cudaSuccess)
            e = launch_band(b[i], b[i + 1], stage[k], h->stream);
        if (e == cudaSuccess && !from)
            e = cudaMemcpyAsync(hp, stage[k], bytes, cudaMemcpyDeviceToHost, h->stream);
        if (e == cudaSuccess)
            e = cudaEventRecord(done[k], h->stream);
    }
    if (e == cudaSuccess)
        e = cudaStreamSynchronize(h->stream);
    for (int k = 0; k < 2; ++k) {
        cudaFree(stage[k]);
        if (done[k])
            cudaEventDestroy(done[k]);
    }
    if (e != cudaSuccess)
        return set_err(HS_ERR_CUDA, std::string("format conversion: ") + cudaGetErrorString(e));
    return HS_OK;
}
}  // namespace

namespace {
int retile_launch(double2* dst, uint32_t m2, uint64_t cnt2, uint64_t N, const double2* src, uint32_t m1,
                  cudaStream_t s) {
    retile_kernel<<<conv_grid((cnt2 + CV_T - 1) / CV_T), CV_T, 0, s>>>(dst, m2, cnt2, N, src, m1);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    CUDA_TRY(cudaGetLastError());
    return HS_OK;
}
}  // namespace

extern "C" {
int hs_state_to_dense(const hs_state* h, double* out, int on_device) {
    int rc = conv_check(h, out);
    return rc ? rc : convert_linear(const_cast<hs_state*>(h), reinterpret_cast<double2*>(out), false, false, on_device);
}
int hs_state_to_packed(const hs_state* h, double* out, int on_device) {
    int rc = conv_check(h, out);
    return rc ? rc : convert_linear(const_cast<hs_state*>(h), reinterpret_cast<double2*>(out), true, false, on_device);
}
int hs_state_from_dense(hs_state* h, const double* in, int on_device) {
    int rc = conv_check(h, in);
    return rc ? rc : convert_linear(h, reinterpret_cast<double2*>(const_cast<double*>(in)), false, true, on_device);
}
int hs_state_from_packed(hs_state* h, const double* in, int on_device) {
    int rc = conv_check(h, in);
    return rc ? rc : convert_linear(h, reinterpret_cast<double2*>(const_cast<double*>(in)), true, true, on_device);
}
int hs_state_convert(const hs_state* src, hs_state* dst) {
    int rc = conv_check(src, dst);
    if (rc)
        return rc;
    if (dst->Plog)
        return set_err(HS_ERR_UNSUPPORTED, "format conversion of a sharded state: gather the shards first");
    if (src->n != dst->n)
        return set_err(HS_ERR_INVALID, "convert: qubit counts differ");
    if (src->device != dst->device)
        return set_err(HS_ERR_INVALID, "convert: states on different devices");
    if (src == dst)
        return HS_OK;
    DeviceGuard dg(dst->device);
    // dst's stream waits for src's pending work
    cudaEvent_t ev;
    CUDA_TRY(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(ev, src->stream));
    CUDA_TRY(cudaStreamWaitEvent(dst->stream, ev, 0));
    CUDA_TRY(cudaEventDestroy(ev));
    return retile_launch(dst->d, (uint32_t)dst->m, dst->count, dst->N, src->d, (uint32_t)src->m, dst->stream);
}
int hs_device_alloc(int device, uint64_t bytes, void** out) {
    if (!out)
        return set_err(HS_ERR_INVALID, "null out");
    DeviceGuard dg(device);
    if (cudaMalloc(out, bytes) != cudaSuccess) {
        cudaGetLastError();
        *out = nullptr;
        return set_err(HS_ERR_NOMEM, "cudaMalloc failed");
    }
    return HS_OK;
}
int hs_device_free(int device, void* p) {
    DeviceGuard dg(device);
    CUDA_TRY(cudaFree(p));
    return HS_OK;
}
int hs_copy_d2h(int device, void* host, const void* dev, uint64_t bytes) {
    DeviceGuard dg(device);
    CUDA_TRY(cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost));
    return HS_OK;
}
}  // extern "C"

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
    unsigned char hdr[16] = {'O', 'H', 'R', 'M', 1, 0, 0, 0, 2, (unsigned char)h->n, (unsigned char)h->mu, 0, 0, 0, 0, 0};
    bool ok = std::fwrite(hdr, 1, 16, f) == 16;
    DeviceGuard dg(h->device);
    UserTemp ut;  // m > 5: stream the user-layout image
    if (big_tiles(h) && to_user(h, ut)) {
        std::fclose(f);
        return HS_ERR_NOMEM;
    }
    PinnedPair pp;
    const uint64_t total = h->ucount * sizeof(double2);
    for (int i = 0; i < 2 && ok; ++i)
        if (cudaHostAlloc(&pp.b[i], IO_CHUNK, cudaHostAllocDefault) != cudaSuccess) {
            cudaGetLastError();
            std::fclose(f);
            return set_err(HS_ERR_NOMEM, "save: pinned staging buffer");
        }
    cudaEvent_t ev[2];
    cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming);
    const char* src = reinterpret_cast<const char*>(ut.p ? ut.p : h->d);
    uint64_t off = 0;
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
        prev_len = len;
        off += len;
        cur ^= 1;
    }
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
    UserTemp ut;  // m > 5: read the user-layout image, then convert
    if (big_tiles(h) && user_alloc(h, ut)) {
        hs_state_free(h);
        std::fclose(f);
        return HS_ERR_NOMEM;
    }
    const uint64_t total = h->ucount * sizeof(double2);
    char* dst = reinterpret_cast<char*>(ut.p ? ut.p : h->d);
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
    if (ok && ut.p)
        ok = from_user(h, ut.p) == HS_OK;
    ut.release();
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
