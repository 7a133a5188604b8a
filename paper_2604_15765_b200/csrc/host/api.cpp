// hermsim_b200 host API: device-resident TiledHermitian, the apply() dispatcher and the
// engine-level / native entry points, all calling the CUDA engine through include/hs_cuda.h.
// Dispatch mirrors hermsim::apply (kernels.cpp:510-549) and apply_generic (kernels.cpp:457-506)
// with one deliberate difference: k = 3 generic channels run on the tiled layout directly
// instead of the reference's dense round trip (kernels.cpp:498-505); the plan reports the
// tiled regime (intra / cross / mixed) that ran.
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>

#include "hermsim_b200/hermsim.hpp"

namespace hermsim_b200 {

namespace {

[[noreturn]] void raise(int rc, const char* where) {
    const std::string msg = std::string(where) + ": " + hs_last_error();
    if (rc == HS_ERR_INVALID)
        throw std::invalid_argument(msg);
    if (rc == HS_ERR_RANGE)
        throw std::out_of_range(msg);
    if (rc == HS_ERR_IO) {
        const std::string e = hs_last_error();
        IoErrorKind kind = IoErrorKind::io_failure;
        const std::pair<const char*, IoErrorKind> names[] = {
            {"bad_magic", IoErrorKind::bad_magic}, {"bad_version", IoErrorKind::bad_version},
            {"bad_header", IoErrorKind::bad_header}, {"truncated", IoErrorKind::truncated},
            {"length_mismatch", IoErrorKind::length_mismatch}};
        for (const auto& [name, k] : names)
            if (e.rfind(name, 0) == 0)
                kind = k;
        throw IoError(kind, msg);
    }
    throw std::runtime_error(msg);
}

void check(int rc, const char* where) {
    if (rc != HS_OK)
        raise(rc, where);
}

// row_stacked re-indexing of a column-stacked transfer matrix (kernels.cpp:27-37)
std::vector<cplx> row_stacked(const TransferMatrix& s) {
    const std::size_t d = std::size_t{1} << s.k, dim = d * d;
    std::vector<cplx> out(dim * dim);
    for (std::size_t a = 0; a < d; ++a)
        for (std::size_t ap = 0; ap < d; ++ap)
            for (std::size_t mu = 0; mu < d; ++mu)
                for (std::size_t nu = 0; nu < d; ++nu)
                    out[(a * d + ap) * dim + (mu * d + nu)] = s.s(a + ap * d, mu + nu * d);
    return out;
}

void check_transfer(const TransferMatrix& s, int k) {  // kernels.cpp:60-64
    const std::size_t want = std::size_t{1} << (2 * k);
    if (s.k != k || s.s.rows() != want || s.s.cols() != want)
        throw std::invalid_argument("transfer matrix dimension does not match target count");
}

SubcaseCounters counters(const hs_plan& p) { return {p.subcases[0], p.subcases[1], p.subcases[2]}; }

const double* dptr(const cplx* p) { return reinterpret_cast<const double*>(p); }

}  // namespace

const char* kernel_path_name(KernelPath p) {  // kernels.cpp:81-96
    switch (p) {
    case KernelPath::dense_generic: return "dense-generic";
    case KernelPath::packed_generic: return "packed-generic";
    case KernelPath::tiled_intra: return "tiled-intra";
    case KernelPath::tiled_cross: return "tiled-cross";
    case KernelPath::tiled_mixed: return "tiled-mixed";
    case KernelPath::dense_fallback: return "dense-fallback";
    case KernelPath::native_pauli_x: return "native-pauli-x";
    case KernelPath::native_pauli_y: return "native-pauli-y";
    case KernelPath::native_phase: return "native-phase";
    case KernelPath::native_hadamard: return "native-hadamard";
    case KernelPath::native_permutation: return "native-permutation";
    }
    return "?";
}

std::uint64_t footprint_bytes(int n, int tile_exp) {  // storage.cpp:294-310 (tiled)
    if (n < 1 || n > 30)
        throw std::invalid_argument("qubit count must be in [1, 30]");
    if (tile_exp < 0 || tile_exp > n + 2)
        throw std::invalid_argument("tile exponent must be in [0, n + 2]");
    const std::uint64_t dim = std::uint64_t{1} << n, edge = std::uint64_t{1} << tile_exp;
    const std::uint64_t grid = dim >= edge ? dim / edge : 1;
    return grid * (grid + 1) / 2 * edge * edge * 16;
}

// --------------------------------------------------------------------------- storage
TiledHermitian::TiledHermitian(int n_qubits, int tile_exp, int device) : n_(n_qubits), m_(tile_exp) {
    check(hs_state_create(n_qubits, tile_exp, device, &h_), "TiledHermitian");
    std::uint64_t count = 0, grid = 0;
    check(hs_state_info(h_, nullptr, nullptr, &count, &grid), "TiledHermitian");
    count_ = count;
    grid_ = grid;
}

TiledHermitian::~TiledHermitian() {
    if (h_)
        hs_state_free(h_);
}

TiledHermitian::TiledHermitian(const TiledHermitian& o) : TiledHermitian(o.n_, o.m_) {
    check(hs_state_copy(h_, o.h_), "TiledHermitian copy");
}

TiledHermitian& TiledHermitian::operator=(const TiledHermitian& o) {
    if (this != &o) {
        TiledHermitian tmp(o);
        *this = std::move(tmp);
    }
    return *this;
}

TiledHermitian::TiledHermitian(TiledHermitian&& o) noexcept
    : h_(o.h_), n_(o.n_), m_(o.m_), grid_(o.grid_), count_(o.count_) {
    o.h_ = nullptr;
}

TiledHermitian& TiledHermitian::operator=(TiledHermitian&& o) noexcept {
    if (this != &o) {
        if (h_)
            hs_state_free(h_);
        h_ = o.h_;
        n_ = o.n_;
        m_ = o.m_;
        grid_ = o.grid_;
        count_ = o.count_;
        o.h_ = nullptr;
    }
    return *this;
}

TiledHermitian TiledHermitian::adopt(hs_state* h) {
    TiledHermitian t;
    int n = 0, m = 0;
    std::uint64_t count = 0, grid = 0;
    check(hs_state_info(h, &n, &m, &count, &grid), "TiledHermitian");
    t.h_ = h;
    t.n_ = n;
    t.m_ = m;
    t.count_ = count;
    t.grid_ = grid;
    return t;
}

void save(const TiledHermitian& h, const std::string& path) { check(hs_state_save(h.handle(), path.c_str()), "save"); }

TiledHermitian random_hermitian(int n, std::uint64_t seed, int tile_exp, int device) {
    TiledHermitian t(n, tile_exp, device);
    check(hs_state_fill_random_hermitian(t.handle(), seed), "random_hermitian");
    return t;
}

TiledHermitian basis_projector(int n, std::uint64_t basis, int tile_exp, int device) {
    TiledHermitian t(n, tile_exp, device);
    check(hs_state_fill_basis_projector(t.handle(), basis), "basis_projector");
    return t;
}

TiledHermitian load(const std::string& path, int device) {
    hs_state* h = nullptr;
    check(hs_state_load(path.c_str(), device, &h), "load");
    return TiledHermitian::adopt(h);
}

void TiledHermitian::upload(const cplx* payload) { check(hs_state_upload(h_, dptr(payload), count_), "upload"); }

void TiledHermitian::download(cplx* payload) const {
    check(hs_state_download(h_, reinterpret_cast<double*>(payload), count_), "download");
}

std::vector<cplx> TiledHermitian::to_host() const {
    std::vector<cplx> out(count_);
    download(out.data());
    return out;
}

void TiledHermitian::synchronize() const { check(hs_state_synchronize(h_), "synchronize"); }

// --------------------------------------------------------------------- engine entry points
void apply_tiled_intra(TiledHermitian& h, const TransferMatrix& s, std::uint32_t target, int) {
    check_transfer(s, 1);
    if (target >= static_cast<std::uint32_t>(h.tile_exp()))
        throw std::invalid_argument("apply_tiled_intra: target must be < m");
    const auto sr = row_stacked(s);
    check(hs_apply_transfer(h.handle(), 1, dptr(sr.data()), &target, nullptr), "apply_tiled_intra");
}

SubcaseCounters apply_tiled_cross(TiledHermitian& h, const TransferMatrix& s, std::uint32_t target, int) {
    check_transfer(s, 1);
    if (target < static_cast<std::uint32_t>(h.tile_exp()) || target >= static_cast<std::uint32_t>(h.qubits()))
        throw std::invalid_argument("apply_tiled_cross: target must be in [m, n)");
    const auto sr = row_stacked(s);
    hs_plan p{};
    check(hs_apply_transfer(h.handle(), 1, dptr(sr.data()), &target, &p), "apply_tiled_cross");
    return counters(p);
}

SubcaseCounters apply_tiled_twoqubit(TiledHermitian& h, const TransferMatrix& s, const ActiveQubits& q, int) {
    if (q.count() != 2)
        throw std::invalid_argument("apply_tiled_twoqubit: needs exactly two targets");
    check_transfer(s, 2);
    const auto sr = row_stacked(s);
    hs_plan p{};
    check(hs_apply_transfer(h.handle(), 2, dptr(sr.data()), q.positions().data(), &p), "apply_tiled_twoqubit");
    return counters(p);
}

bool PermutationGate::is_involution() const {
    for (std::size_t x = 0; x < table.size(); ++x)
        if (table[table[x]] != x)
            return false;
    return true;
}

void apply_pauli_x(TiledHermitian& h, std::uint32_t target, int) {
    if (target >= static_cast<std::uint32_t>(h.qubits()))
        throw std::out_of_range("native path: target qubit out of range");
    check(hs_apply_pauli(h.handle(), target, 0, nullptr), "apply_pauli_x");
}

void apply_pauli_y(TiledHermitian& h, std::uint32_t target, int) {
    if (target >= static_cast<std::uint32_t>(h.qubits()))
        throw std::out_of_range("native path: target qubit out of range");
    check(hs_apply_pauli(h.handle(), target, 1, nullptr), "apply_pauli_y");
}

void apply_diagonal_phase(TiledHermitian& h, std::uint32_t target, const std::array<cplx, 2>& phases, int) {
    if (target >= static_cast<std::uint32_t>(h.qubits()))
        throw std::out_of_range("native path: target qubit out of range");
    check(hs_apply_diagonal_phase(h.handle(), target, dptr(phases.data()), nullptr), "apply_diagonal_phase");
}

void apply_hadamard(TiledHermitian& h, std::uint32_t target, int) {
    if (target >= static_cast<std::uint32_t>(h.qubits()))
        throw std::out_of_range("native path: target qubit out of range");
    check(hs_apply_hadamard(h.handle(), target, nullptr), "apply_hadamard");
}

void apply_permutation(TiledHermitian& h, const PermutationGate& gate, const ActiveQubits& qubits, int) {
    if (gate.k != qubits.count())  // native.cpp:511-520
        throw std::invalid_argument("apply_permutation: gate arity does not match target count");
    if (gate.table.size() != (std::size_t{1} << gate.k))
        throw std::invalid_argument("apply_permutation: bad permutation table size");
    for (std::uint32_t q : qubits.positions())
        if (q >= static_cast<std::uint32_t>(h.qubits()))
            throw std::out_of_range("apply_permutation: target out of range");
    check(hs_apply_permutation(h.handle(), gate.k, gate.table.data(), qubits.positions().data(), nullptr),
          "apply_permutation");
}

// ------------------------------------------------------------------------- dispatcher
ApplyPlan apply_on_handle(hs_state* hs, const ChannelSpec& spec, std::span<const std::uint32_t> targets,
                          const ApplyOptions& opts) {
    int n = 0, mm = 0;
    check(hs_state_info(hs, &n, &mm, nullptr, nullptr), "apply");
    if (static_cast<int>(targets.size()) != spec.locality())  // validate_targets, kernels.cpp:448-455
        throw std::invalid_argument("apply: target count does not match channel locality");
    for (std::uint32_t q : targets)
        if (q >= static_cast<std::uint32_t>(n))
            throw std::out_of_range("apply: target qubit out of range");
    const BoundChannel bc = bind_channel(spec, targets);
    const int k = bc.qubits.count();
    const std::uint32_t* tq = bc.qubits.positions().data();

    ApplyPlan plan;
    plan.targets = bc.qubits;
    hs_plan p{};
    hs_plan* pp = &p;
    hs_set_plan_subcases(opts.count_subcases ? 1 : 0);
    struct Restore {
        ~Restore() { hs_set_plan_subcases(1); }
    } restore;
    if (opts.allow_native) {
        switch (spec.kind) {
        case GateKind::pauli_x:
            check(hs_apply_pauli(hs, tq[0], 0, pp), "apply");
            plan.path = KernelPath::native_pauli_x;
            plan.touched_bytes = p.touched_bytes;
            return plan;
        case GateKind::pauli_y:
            check(hs_apply_pauli(hs, tq[0], 1, pp), "apply");
            plan.path = KernelPath::native_pauli_y;
            plan.touched_bytes = p.touched_bytes;
            return plan;
        case GateKind::diagonal_phase:
            check(hs_apply_diagonal_phase(hs, tq[0], dptr(bc.phases.data()), pp), "apply");
            plan.path = KernelPath::native_phase;
            plan.touched_bytes = p.touched_bytes;
            return plan;
        case GateKind::hadamard:
            check(hs_apply_hadamard(hs, tq[0], pp), "apply");
            plan.path = KernelPath::native_hadamard;
            plan.touched_bytes = p.touched_bytes;
            return plan;
        case GateKind::permutation:
            if (bc.perm.size() != (std::size_t{1} << k))
                throw std::invalid_argument("apply_permutation: bad permutation table size");
            check(hs_apply_permutation(hs, k, bc.perm.data(), tq, pp), "apply");
            plan.path = KernelPath::native_permutation;
            plan.touched_bytes = p.touched_bytes;
            return plan;
        case GateKind::generic_kraus:
            break;
        }
    }
    // apply_generic (kernels.cpp:457-506)
    const std::size_t d = std::size_t{1} << k;
    if (k == 2 && bc.kraus.ops.size() >= 2 && bc.kraus.ops.size() <= 4) {
        // small k = 2 Kraus sets: the engine sums L_a B L_a^dagger on the tensor cores where the
        // geometry allows, else it applies the transfer matrix itself
        std::vector<cplx> ops;
        ops.reserve(bc.kraus.ops.size() * d * d);
        for (const Mat& l : bc.kraus.ops)
            ops.insert(ops.end(), l.data(), l.data() + d * d);
        check(hs_apply_kraus(hs, k, static_cast<int>(bc.kraus.ops.size()), dptr(ops.data()), tq, pp), "apply");
    } else if (k <= 2 && !(k == 2 && bc.kraus.ops.size() == 1)) {
        const auto sr = row_stacked(bc.transfer);  // TransferQuad / matvec<16> engines
        check(hs_apply_transfer(hs, k, dptr(sr.data()), tq, pp), "apply");
    } else if (bc.kraus.ops.size() == 1) {
        // rank-1 k >= 2: direct block update B -> L B L^dagger (SPEC conjugation_kernels
        // "Unitary rank-1 channels may use the direct block update Eq. (2)")
        check(hs_apply_unitary(hs, k, dptr(bc.kraus.ops[0].data()), tq, pp), "apply");
    } else {
        std::vector<cplx> ops;
        ops.reserve(bc.kraus.ops.size() * d * d);
        for (const Mat& l : bc.kraus.ops)
            ops.insert(ops.end(), l.data(), l.data() + d * d);
        check(hs_apply_kraus(hs, k, static_cast<int>(bc.kraus.ops.size()), dptr(ops.data()), tq, pp),
              "apply");
    }
    const std::uint32_t m = static_cast<std::uint32_t>(mm);
    int grid = 0;
    for (int i = 0; i < k; ++i)
        grid += tq[i] >= m;
    plan.path = grid == 0 ? KernelPath::tiled_intra : grid == k ? KernelPath::tiled_cross : KernelPath::tiled_mixed;
    if (opts.count_subcases && (k <= 2) && grid > 0)
        plan.subcases = counters(p);
    plan.touched_bytes = p.touched_bytes;
    return plan;
}

ApplyPlan apply(TiledHermitian& h, const ChannelSpec& spec, std::span<const std::uint32_t> targets,
                const ApplyOptions& opts) {
    return apply_on_handle(h.handle(), spec, targets, opts);
}

ApplyPlan apply(TiledHermitian& h, const ChannelSpec& spec, std::initializer_list<std::uint32_t> targets,
                const ApplyOptions& opts) {
    return apply(h, spec, std::span<const std::uint32_t>(targets.begin(), targets.size()), opts);
}

// ------------------------------------------------------------------------ observables
double expectation(const TiledHermitian& rho, const TiledHermitian& obs) {
    if (rho.qubits() != obs.qubits() || rho.tile_exp() != obs.tile_exp())
        throw std::invalid_argument("expectation: size mismatch");
    double out = 0.0;
    check(hs_expectation(rho.handle(), obs.handle(), &out), "expectation");
    return out;
}

double trace(const TiledHermitian& h) {
    double out = 0.0;
    check(hs_trace(h.handle(), &out), "trace");
    return out;
}

cplx gaussian_entry(std::uint64_t seed, std::uint64_t counter) {  // storage.cpp:22-44
    auto splitmix64 = [](std::uint64_t x) {
        x += 0x9E3779B97F4A7C15ull;
        x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
        x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
        return x ^ (x >> 31);
    };
    const std::uint64_t base = splitmix64(seed ^ 0xD6E8FEB86659FD93ull);
    const std::uint64_t r1 = splitmix64(base + 2 * counter);
    const std::uint64_t r2 = splitmix64(base + 2 * counter + 1);
    const double u1 = static_cast<double>((r1 >> 11) + 1) * 0x1.0p-53;
    const double u2 = static_cast<double>(r2 >> 11) * 0x1.0p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double phi = 2.0 * 3.14159265358979323846 * u2;
    return {r * std::cos(phi), r * std::sin(phi)};
}

}  // namespace hermsim_b200
