/*
 * hs_cuda.h -- thin C-ABI over the B200 (sm_100a) conjugation engine.
 *
 * This is the drop-in boundary of the hot path named in BASELINE.json north_star: the
 * single-pass k-local conjugation rho -> U rho U^dagger and the Kraus sum
 * sum_a K_a rho K_a^dagger on a hermitian operator stored in the reference's tiled
 * lower-triangle layout.  Plain pointers and sizes only; every entry point returns an int
 * status (HS_OK == 0) and never throws; hs_last_error() gives the message of the calling
 * thread's last failure.  The C++ host API (include/hermsim_b200/hermsim.hpp), which keeps
 * the reference's C++ surface, is layered on top of these calls.
 *
 * Reference interfaces replaced (arXiv 2604.15765, /root/reference/proj):
 *   hs_state_*            TiledHermitian(n, m) ctor/dtor, data(), element_count()
 *                         (include/hermsim/storage.hpp:60-96, src/storage.cpp:77-84)
 *   hs_apply_transfer     apply_tiled_intra / apply_tiled_cross / apply_tiled_twoqubit
 *                         (include/hermsim/kernels.hpp:73-83, src/kernels.cpp:176-188,430-444)
 *   hs_apply_unitary      rank-1 channels through the direct block update of SPEC.md
 *                         conjugation_kernels ("Unitary rank-1 channels may use the direct block
 *                         update Eq. (2)"); also replaces the k = 3 dense round trip
 *                         (src/kernels.cpp:498-505)
 *   hs_apply_kraus        apply_generic for any k <= 3 (src/kernels.cpp:457-506)
 *   hs_apply_hadamard     apply_hadamard (include/hermsim/native.hpp:43-44, src/native.cpp:343-361)
 *   hs_apply_diagonal_phase  apply_diagonal_phase (native.hpp:39-41, native.cpp:238-324)
 *   hs_apply_pauli        apply_pauli_x / apply_pauli_y (native.hpp:29-34, native.cpp:99-230)
 *   hs_apply_permutation  apply_permutation (native.hpp:46-47, native.cpp:511-549)
 *   hs_expectation        tr(rho O) of PAPER.md:412-417 / SPEC.md observables (absent from the
 *                         reference code; strict ti > tj bound per SPEC.md)
 *
 * Conventions
 *   - Payload layout is byte-identical to TiledHermitian: tile (ti >= tj) at element offset
 *     (ti(ti+1)/2 + tj) * M^2, tiles and elements row-major, diagonal tiles hold all M^2
 *     elements, complex128 interleaved (re, im).  `count` arguments are complex elements.
 *   - "Bound" entry points take targets ASCENDING; local basis bit l <-> targets[l] (the result
 *     of bind_channel, src/channel.cpp:196-268).  Matrices are row-major complex128.
 *   - All device work is ordered on the state's CUDA stream and asynchronous, except the
 *     calls documented as synchronising (download, expectation, trace, frobenius).
 *   - One state may be used by one host thread at a time (the reference's exclusive-access
 *     rule).
 */
#ifndef HS_CUDA_H
#define HS_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum hs_status {
    HS_OK = 0,
    HS_ERR_INVALID = -1,     /* std::invalid_argument in the reference */
    HS_ERR_RANGE = -2,       /* std::out_of_range in the reference */
    HS_ERR_CUDA = -3,        /* CUDA runtime failure (incl. missing device) */
    HS_ERR_NOMEM = -4,       /* device allocation failed */
    HS_ERR_UNSUPPORTED = -5, /* valid request this build does not implement */
    HS_ERR_IO = -6           /* hermsim::IoError (storage_io.hpp:11-20); message starts with the IoErrorKind */
};

/* KernelPath (include/hermsim/kernels.hpp:12-24); same numbering. */
enum hs_kernel_path {
    HS_PATH_DENSE_GENERIC = 0,
    HS_PATH_PACKED_GENERIC = 1,
    HS_PATH_TILED_INTRA = 2,
    HS_PATH_TILED_CROSS = 3,
    HS_PATH_TILED_MIXED = 4,
    HS_PATH_DENSE_FALLBACK = 5,
    HS_PATH_NATIVE_PAULI_X = 6,
    HS_PATH_NATIVE_PAULI_Y = 7,
    HS_PATH_NATIVE_PHASE = 8,
    HS_PATH_NATIVE_HADAMARD = 9,
    HS_PATH_NATIVE_PERMUTATION = 10
};

/* ApplyPlan (kernels.hpp:48-52) plus GPU launch facts. */
typedef struct hs_plan {
    int32_t path;           /* hs_kernel_path */
    int32_t k;              /* number of targets */
    uint32_t targets[3];    /* ascending */
    uint64_t subcases[3];   /* cross_tile (A), cross_tile_adj (B), cross_tile_diag (C) */
    int32_t grid_bits;      /* g: targets >= m */
    int32_t launches;       /* kernels launched by this call */
    uint64_t touched_bytes; /* bytes read + written by the launch (algorithmic) */
} hs_plan;

typedef struct hs_state hs_state;

const char* hs_last_error(void);
/* Calling thread: fill hs_plan.subcases (host-side enumeration for k = 2) or not (default 1). */
int hs_set_plan_subcases(int enable);
const char* hs_version(void);
int hs_device_count(int* out);

/* ---- state (TiledHermitian) ------------------------------------------------------------ */
/* Allocates the tiled payload in HBM (zero-filled, like AlignedArray, types.hpp:37-42).
 * Limits as the reference: 1 <= n <= 30, 0 <= m <= n + 2 (storage.cpp:12-20).  For m > 5 the
 * operator is held in HBM in the m = 5 layout (every kernel unchanged) and every payload-facing call
 * (info, upload / download and their ranges, save / load) speaks the m layout, converted on the fly
 * on the device; hs_state_device_ptr then exposes the internal m = 5 layout, and sharding needs
 * m <= 5. */
int hs_state_create(int n, int m, int device, hs_state** out);
int hs_state_free(hs_state* h);
int hs_state_info(const hs_state* h, int* n, int* m, uint64_t* count, uint64_t* grid);
/* Host payload <-> HBM.  `host` may be pageable or pinned; the copy is synchronous. */
int hs_state_upload(hs_state* h, const double* host, uint64_t count);
int hs_state_download(const hs_state* h, double* host, uint64_t count);
/* Stream-ordered variants: `host` must be pinned (cudaHostAlloc / hs_host_alloc). */
int hs_state_upload_async(hs_state* h, const double* host, uint64_t count);
int hs_state_download_async(const hs_state* h, double* host, uint64_t count);
/* Partial copies of `count` complex elements starting at element `offset`. */
int hs_state_upload_range(hs_state* h, const double* host, uint64_t offset, uint64_t count);
/* OHRM container (hermsim::save / load, storage_io.cpp:34-118; tiled format), streamed between
 * HBM and the file through pinned buffers. */
int hs_state_save(const hs_state* h, const char* path);
int hs_state_load(const char* path, int device, hs_state** out);
int hs_state_download_range(const hs_state* h, double* host, uint64_t offset, uint64_t count);
int hs_state_copy(hs_state* dst, const hs_state* src);
int hs_state_zero(hs_state* h);
int hs_state_synchronize(const hs_state* h);
/* Replaces the state's stream (cudaStream_t, NULL = a fresh non-blocking stream). */
int hs_state_set_stream(hs_state* h, void* stream);
void* hs_state_stream(const hs_state* h);
void* hs_state_device_ptr(hs_state* h);

/* Format conversions on the device (hermsim::to_dense / convert, storage.cpp:241-292; bit-identical
 * to the reference's results).  dense = N x N row-major complex128 (DenseHermitian, storage.hpp:12-35),
 * packed = column-major lower triangle, N(N+1)/2 complex128 (PackedHermitian, storage.hpp:37-58).
 * `on_device` != 0: the buffer is device memory on the state's device (the call is stream-ordered on
 * the state's stream); 0: host memory, streamed through device staging bands (synchronous).
 * from_* follow convert()'s fill_from_lower: stored (i >= j) = d(i, j), a diagonal tile's upper half
 * = conj(d(j, i)).  Unsharded states only (HS_ERR_UNSUPPORTED otherwise). */
int hs_state_to_dense(const hs_state* h, double* out, int on_device);
int hs_state_to_packed(const hs_state* h, double* out, int on_device);
int hs_state_from_dense(hs_state* h, const double* in, int on_device);
int hs_state_from_packed(hs_state* h, const double* in, int on_device);
/* convert(src, tiled, dst's tile exponent): same n, any m on both sides, same device. */
int hs_state_convert(const hs_state* src, hs_state* dst);
/* Device memory helpers for the conversion buffers (cudaMalloc / cudaFree on `device`). */
int hs_device_alloc(int device, uint64_t bytes, void** out);
int hs_device_free(int device, void* p);
int hs_copy_d2h(int device, void* host, const void* dev, uint64_t bytes);

int hs_host_alloc(uint64_t bytes, void** out);   /* pinned host memory */
int hs_host_free(void* p);

/* ---- bound engine entry points ------------------------------------------------------- */
/* Kraus channel through its row-stacked transfer matrix (kernels.cpp:27-37): `s` is
 * 4^k x 4^k complex, k in {1, 2}.  plan may be NULL. */
int hs_apply_transfer(hs_state* h, int k, const double* s_rowstacked, const uint32_t* targets, hs_plan* plan);
/* Fused program (no reference counterpart: the reference applies one op per pass):
 * nsteps <= 16 single-qubit steps on in-tile qubits (< m) in ONE pass over the triangle, equal to
 * applying them in order.  kinds[p]: 0 = row-stacked 4x4 transfer matrix s[16p..16p+15]
 * (interleaved complex), 1 = Hadamard (s ignored), 2 = diagonal transfer (diagonal of s used),
 * 3 = real transfer coupling only (00,11) and (01,10) (real parts of s[0,3,12,15] and s[5,6,9,10]
 * used: depolarising, amplitude damping, ...), 4 = real (00,11) block s[0,3,12,15] with a complex
 * diagonal s[5], s[10] on (01,10) (the same channels composed with Rz / phase gates), 5 = Hadamard
 * butterfly without its factor 1/2 (the caller has scaled the coefficients of the step before, on
 * the same qubit, by 1/2 -- exact in binary floating point).  The caller
 * vouches that s has the stated form; entries outside it are ignored. */
int hs_apply_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s, hs_plan* plan);
/* Fused grid program: 2 .. 16 steps on 2 or 3 distinct grid qubits (>= m), each qubit's steps
 * consecutive, in ONE pass over the triangle (the units of those grid bits are gathered; each qubit's
 * chain of steps runs on every quad in registers, one shared-memory round trip per qubit).
 * Single-GPU states, m = 5.  (hs_apply_program likewise runs consecutive steps on one qubit in one
 * round trip.) */
int hs_apply_grid_program(hs_state* h, int nsteps, const int* kinds, const uint32_t* bits, const double* s,
                          hs_plan* plan);
/* CX layer (fusion; no reference counterpart): CX gates on npairs (<= 32) disjoint (control,
 * target) pairs in ONE in-place pass, bit-identical to applying them one by one
 * (apply_permutation, native.cpp:433-549).  Single-GPU states. */
int hs_apply_cx_layer(hs_state* h, int npairs, const uint32_t* controls, const uint32_t* targets, hs_plan* plan);
/* Unitary conjugation B -> U B U^dagger per coupled block, direct form; k in {1, 2, 3}. */
int hs_apply_unitary(hs_state* h, int k, const double* u, const uint32_t* targets, hs_plan* plan);
/* Generic Kraus set {L_a} (nops matrices 2^k x 2^k), k in {1, 2, 3}. */
int hs_apply_kraus(hs_state* h, int k, int nops, const double* ops, const uint32_t* targets, hs_plan* plan);
int hs_apply_hadamard(hs_state* h, uint32_t target, hs_plan* plan);
/* Diagonal phase diag(p0, p1) (Z, S, T, Rz): phases = 2 complex of unit modulus. */
int hs_apply_diagonal_phase(hs_state* h, uint32_t target, const double* phases, hs_plan* plan);
/* Pauli X (y == 0) or Y (y != 0). */
int hs_apply_pauli(hs_state* h, uint32_t target, int y, hs_plan* plan);
/* Basis permutation (CX, SWAP, Toffoli, ...): table[x] = image of local basis x (bound). */
int hs_apply_permutation(hs_state* h, int k, const uint32_t* table, const uint32_t* targets, hs_plan* plan);
/* Generalised monomial U = P D: out(r, c) = d_r conj(d_c) B(pinv(r), pinv(c)); `perm` is the
 * bound table (NULL = identity), `diag` 2^k complex (NULL = all ones). */
int hs_apply_monomial(hs_state* h, int k, const uint32_t* perm, const double* diag, const uint32_t* targets,
                      hs_plan* plan);

/* ---- observables ---------------------------------------------------------------------- */
/* tr(rho O) = sum_diag Re<O_t, rho_t>_F + 2 sum_{ti > tj} Re<O_t, rho_t>_F; deterministic
 * fixed-order reduction; synchronising. */
int hs_expectation(const hs_state* rho, const hs_state* obs, double* out);
int hs_trace(const hs_state* h, double* out);
int hs_frobenius(const hs_state* h, double* out);

/* ---- seeded synthetic inputs (bench / test harness, computed on the device) ------------ */
/* rho = (1/rank) sum_i |psi_i><psi_i|; psi = rank x 2^n complex (host, normalised).  Every
 * stored element is formed with explicitly rounded products and sums in a fixed order, so
 * the payload is bit-identical to the host construction hsg_rho_payload (harness.c). */
int hs_state_fill_mixture(hs_state* h, int rank, const double* psi);
/* hermsim::random_hermitian(n, seed) and basis_projector(n, basis) (storage.cpp:195-239), generated
 * on the device (counter-based RNG: elements equal the reference's to ~1e-16 relative). */
int hs_state_fill_random_hermitian(hs_state* h, uint64_t seed);
int hs_state_fill_basis_projector(hs_state* h, uint64_t basis);
/* O = sum_s coef_s P_s for Pauli strings with X-mask x[s], Z-mask z[s] (Y sets both) and
 * ny[s] = #Y; bit-identical to hsg_pauli_payload (harness.c). */
int hs_state_fill_pauli_sum(hs_state* h, int count, const uint64_t* x, const uint64_t* z, const int32_t* ny,
                            const double* coef);

/* max over stored elements of |h - (1/rank) sum |psi_i><psi_i|| (componentwise), computed on
 * the device with the same rounding as hs_state_fill_mixture: full-size verification of a
 * state against evolved pure states without a second copy in HBM.  Synchronising. */
int hs_state_distance_mixture(const hs_state* h, int rank, const double* psi, double* max_abs);

/* ---- sharding across GPUs (XOR blocks over the top log2(P) tile-row bits) -----
 * Shard s of P holds the stored tiles (ti >= tj) with (ti >> logB) ^ (tj >> logB) == s, B = G / P:
 * shard 0 the P diagonal blocks (triangular), shard s != 0 the P/2 rectangular blocks (a, a ^ s),
 * a > a ^ s.  P = 1 is exactly the reference layout.  Operations whose targets avoid the top
 * log2(P) qubits are shard-local; an operation whose targets include top qubits c1.. (mask
 * 2^c1 | ..) couples the group of shards s ^ span(mask): every member needs the others' payloads
 * in its exchange slots (hs_state_exchange_group over NCCL, or hs_state_exchange_group_from per
 * peer for shards in one process), computes every unit of the group and stores only its own
 * tiles.  One top target = a pairwise butterfly step (partner s ^ 2^c). */
int hs_state_create_sharded(int n, int m, int device, int nshards, int shard, hs_state** out);
int hs_state_shard_info(const hs_state* h, int* nshards, int* shard, uint64_t* block_rows);
/* partner shard of an operation on `targets` (any order), -1 when shard-local */
int hs_op_partner(const hs_state* h, int k, const uint32_t* targets, int* partner); /* one top target */
/* group mask of an operation (0 = shard-local) */
int hs_op_group(const hs_state* h, int k, const uint32_t* targets, uint32_t* mask);
int hs_state_recv_alloc(hs_state* h);                       /* one exchange slot */
int hs_state_recv_reserve(hs_state* h, int slots);          /* 2^popcount(mask) - 1 slots, <= 7 */
int hs_state_exchange_from(hs_state* h, const hs_state* peer);  /* pair: slot <- peer payload (device/peer copy) */
int hs_state_exchange_group_from(hs_state* h, const hs_state* peer, uint32_t mask);  /* peer's slot of the group */
int hs_nccl_unique_id(void* id128);                               /* ncclUniqueId (128 bytes) */
int hs_state_comm_init(hs_state* h, const void* id128, int nranks, int rank);  /* rank == shard */
int hs_state_exchange(hs_state* h, int partner);                  /* NCCL send/recv, stream-ordered */
int hs_state_exchange_group(hs_state* h, uint32_t mask);          /* NCCL, every other member of the group */
/* Peer mode: cross-shard operations read the group members' payloads in place (peer memory over
 * NVLink via CUDA IPC / peer access, or the same device) inside their own kernels and write this
 * shard's result into its second buffer, which becomes current -- no exchange buffer.  The caller
 * must order operations across shards: before a cross-shard operation, every group member has
 * finished its previous ones (barrier). */
int hs_state_peer_enable(hs_state* h);                                   /* allocates the second buffer */
int hs_state_peer_buffers(const hs_state* h, void** b0, void** b1);      /* this shard's two buffers */
int hs_state_set_peer(hs_state* h, int shard, const void* b0, const void* b1);  /* a member's two buffers */
int hs_state_peer_flip(const hs_state* h, int* flip);                   /* index of the current buffer */
int hs_ipc_handles(const hs_state* h, void* out128);                     /* cudaIpcMemHandle of both buffers */
int hs_ipc_open(const void* handle64, int device, void** ptr);
int hs_ipc_close(void* ptr, int device);
int hs_peer_access(int device, int peer_device);
/* linear partial sums of one shard: kind 0 tr(rho O), 1 squared Frobenius, 2 trace (sum over shards) */
int hs_reduce_partial(const hs_state* a, const hs_state* b, int kind, double* out);

/* ---- CUDA graphs: capture a sequence of operations on one state, replay it with one launch ----
 * hs_graph_begin(h); ...apply calls on h...; hs_graph_end(h, &g); hs_graph_launch(g, h) (any
 * number of times, stream-ordered on h).  The captured kernels bake in the operations' parameters
 * and the state's payload pointer.  Not for peer-mode states; k = 3 multi-operator Kraus channels
 * cannot be captured. */
typedef struct hs_graph hs_graph;
int hs_graph_begin(hs_state* h);
int hs_graph_end(hs_state* h, hs_graph** out);
int hs_graph_launch(const hs_graph* g, hs_state* h);
int hs_graph_nodes(const hs_graph* g, uint64_t* n);
int hs_graph_free(hs_graph* g);

/* ---- device timing helpers (CUDA events on the state's stream) ------------------------ */
int hs_event_create(void** ev);
int hs_event_destroy(void* ev);
int hs_event_record(void* ev, const hs_state* h);
int hs_event_elapsed_ms(void* start, void* stop, float* ms);  /* synchronises on stop */
/* Number of kernel launches issued by this process so far (for gpu_launches accounting). */
uint64_t hs_launch_count(void);

#ifdef __cplusplus
}
#endif
#endif /* HS_CUDA_H */
