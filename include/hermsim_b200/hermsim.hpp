// hermsim_b200 -- the reference's C++ surface (arXiv 2604.15765, /root/reference/proj/include/
// hermsim) re-hosted on the B200 engine.  Host code in C++ that calls the CUDA kernels through
// the thin C-ABI of include/hs_cuda.h.  Names, argument meaning and error behaviour follow the
// reference so that a caller of hermsim::apply can switch by changing the namespace and keeping
// the matrix on the device:
//
//   reference (hermsim::)                          here (hermsim_b200::)
//   TiledHermitian (storage.hpp:60-96, host RAM)   TiledHermitian (same payload layout, in HBM)
//   Mat / kron / adjoint (linalg.hpp)              Mat / kron / adjoint
//   KrausSet, TransferMatrix, ChannelSpec,         same (channel.hpp:14-92)
//   make_generic, depolarising, native_gate,
//   channel_library, validate_cptni, dual_channel,
//   BoundChannel, bind_channel
//   KernelPath, SubcaseCounters, ApplyOptions,     same (kernels.hpp:12-52)
//   ApplyPlan, apply(...)                          apply(...) (kernels.hpp:58-61)
//   apply_tiled_intra/cross/twoqubit               same (kernels.hpp:73-83)
//   apply_pauli_x/y, apply_diagonal_phase,         same (native.hpp:29-47)
//   apply_hadamard, apply_permutation
//   (absent) tr(rho O)                             expectation(rho, obs)
//
// Errors: std::invalid_argument / std::out_of_range exactly where the reference throws them;
// CUDA failures raise std::runtime_error.  ApplyOptions::threads is accepted and ignored (the
// CUDA grid replaces the std::thread pool, parallel.cpp:15-100).
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <initializer_list>
#include <span>
#include <string>
#include <vector>

#include "hs_cuda.h"

namespace hermsim_b200 {

using cplx = std::complex<double>;

// ------------------------------------------------------------------ linalg (linalg.hpp)
class Mat {
  public:
    Mat() = default;
    Mat(std::size_t rows, std::size_t cols) : rows_(rows), cols_(cols), a_(rows * cols) {}
    static Mat identity(std::size_t dim);
    std::size_t rows() const { return rows_; }
    std::size_t cols() const { return cols_; }
    cplx& operator()(std::size_t r, std::size_t c) { return a_[r * cols_ + c]; }
    const cplx& operator()(std::size_t r, std::size_t c) const { return a_[r * cols_ + c]; }
    cplx* data() { return a_.data(); }
    const cplx* data() const { return a_.data(); }
    bool operator==(const Mat& o) const { return rows_ == o.rows_ && cols_ == o.cols_ && a_ == o.a_; }

  private:
    std::size_t rows_ = 0, cols_ = 0;
    std::vector<cplx> a_;
};

Mat operator*(const Mat& x, const Mat& y);
Mat operator*(cplx s, const Mat& x);
Mat operator+(const Mat& x, const Mat& y);
Mat operator-(const Mat& x, const Mat& y);
Mat adjoint(const Mat& x);
Mat conjugate(const Mat& x);
Mat kron(const Mat& x, const Mat& y);
double max_abs(const Mat& x);
double frobenius_norm(const Mat& x);
std::vector<double> hermitian_eigenvalues(const Mat& h);

// ------------------------------------------------------------- bit index (bit_index.hpp)
class ActiveQubits {
  public:
    ActiveQubits() = default;
    ActiveQubits(std::initializer_list<std::uint32_t> positions)
        : ActiveQubits(std::span<const std::uint32_t>(positions.begin(), positions.size())) {}
    explicit ActiveQubits(std::span<const std::uint32_t> positions);
    int count() const { return k_; }
    std::uint32_t operator[](int i) const { return pos_[i]; }
    std::span<const std::uint32_t> positions() const { return {pos_.data(), static_cast<std::size_t>(k_)}; }

  private:
    std::array<std::uint32_t, 3> pos_{};
    int k_ = 0;
};

std::uint64_t insert_bits(std::uint64_t s, std::uint64_t a, const ActiveQubits& A);
std::uint64_t tile_offset(std::uint64_t t_i, std::uint64_t t_j, std::uint64_t M);

// ---------------------------------------------------------------- channel (channel.hpp)
struct KrausSet {
    int k = 0;
    std::vector<Mat> ops;
    std::size_t local_dim() const { return std::size_t{1} << k; }
};
KrausSet make_kraus_set(int k, std::vector<Mat> ops);

struct TransferMatrix {
    int k = 0;
    Mat s;  // column-stacked: v[mu + 2^k nu] = B(mu, nu)
    std::size_t dim() const { return s.rows(); }
};
TransferMatrix transfer_from_kraus(const KrausSet& ks);

enum class GateKind : std::uint8_t { generic_kraus, pauli_x, pauli_y, diagonal_phase, hadamard, permutation };

struct ChannelSpec {
    std::string name;
    GateKind kind = GateKind::generic_kraus;
    KrausSet kraus;
    TransferMatrix transfer;
    std::array<cplx, 2> phases{cplx{1.0, 0.0}, cplx{1.0, 0.0}};
    std::vector<std::uint32_t> perm;
    int locality() const { return kraus.k; }
};

ChannelSpec make_generic(std::string name, KrausSet ks, bool validate = false, double tol = 1e-10);
ChannelSpec depolarising(double p);
ChannelSpec native_gate(const std::string& name, double theta = 0.0);
std::vector<ChannelSpec> channel_library(double p = 0.1, double theta = 0.7);

enum class CptniClass { trace_preserving, trace_non_increasing, invalid };
struct ValidationReport {
    CptniClass classification;
    double max_deviation;
    double min_eigenvalue;
};
ValidationReport validate_cptni(const KrausSet& ks, double tol = 1e-10);
KrausSet dual_channel(const KrausSet& ks);

struct BoundChannel {
    ActiveQubits qubits;
    KrausSet kraus;
    TransferMatrix transfer;
    std::array<cplx, 2> phases;
    std::vector<std::uint32_t> perm;
    GateKind kind;
};
BoundChannel bind_channel(const ChannelSpec& spec, std::span<const std::uint32_t> targets);

// --------------------------------------------------------------- storage (storage.hpp)
std::uint64_t footprint_bytes(int n, int tile_exp);
cplx gaussian_entry(std::uint64_t seed, std::uint64_t counter);

// Device-resident lower-triangle tile storage; payload byte-identical to hermsim::TiledHermitian.
class TiledHermitian {
  public:
    static constexpr int default_tile_exp = 5;
    explicit TiledHermitian(int n_qubits, int tile_exp = default_tile_exp, int device = 0);
    ~TiledHermitian();
    TiledHermitian(const TiledHermitian& other);  // deep device copy (types.hpp:44-47)
    TiledHermitian& operator=(const TiledHermitian& other);
    TiledHermitian(TiledHermitian&& other) noexcept;
    TiledHermitian& operator=(TiledHermitian&& other) noexcept;

    int qubits() const { return n_; }
    int tile_exp() const { return m_; }
    std::uint64_t dim() const { return std::uint64_t{1} << n_; }
    std::uint64_t tile_edge() const { return std::uint64_t{1} << m_; }
    std::uint64_t grid_dim() const { return grid_; }
    std::uint64_t tile_count() const { return grid_ * (grid_ + 1) / 2; }
    std::size_t element_count() const { return count_; }

    void upload(const cplx* payload);           // host -> HBM (element_count() values)
    void download(cplx* payload) const;         // HBM -> host
    std::vector<cplx> to_host() const;
    void synchronize() const;
    hs_state* handle() const { return h_; }
    // takes ownership of an engine state (hs_state_load, ...)
    static TiledHermitian adopt(hs_state* h);

  private:
    TiledHermitian() = default;
    hs_state* h_ = nullptr;
    int n_ = 0, m_ = 0;
    std::uint64_t grid_ = 0;
    std::size_t count_ = 0;
};

// ------------------------------------------------------------- file I/O (storage_io.hpp)
// OHRM container (magic, version 1, format tag, n, m, payload), tiled format, streamed between
// HBM and the file.  Errors: IoError with the reference's kinds (storage_io.hpp:11-20).
enum class IoErrorKind { bad_magic, bad_version, bad_header, truncated, length_mismatch, io_failure };
class IoError : public std::runtime_error {
  public:
    IoError(IoErrorKind kind, const std::string& what) : std::runtime_error(what), kind_(kind) {}
    IoErrorKind kind() const { return kind_; }

  private:
    IoErrorKind kind_;
};
void save(const TiledHermitian& h, const std::string& path);
TiledHermitian load(const std::string& path, int device = 0);

// ------------------------------------------------------------ generators (storage.hpp:129-154)
// hermsim::random_hermitian / basis_projector, tiled format, generated on the device
TiledHermitian random_hermitian(int n, std::uint64_t seed, int tile_exp = TiledHermitian::default_tile_exp,
                                int device = 0);
TiledHermitian basis_projector(int n, std::uint64_t basis, int tile_exp = TiledHermitian::default_tile_exp,
                               int device = 0);

// ----------------------------------------------------------------- kernels (kernels.hpp)
enum class KernelPath : std::uint8_t {
    dense_generic,
    packed_generic,
    tiled_intra,
    tiled_cross,
    tiled_mixed,
    dense_fallback,
    native_pauli_x,
    native_pauli_y,
    native_phase,
    native_hadamard,
    native_permutation,
};
const char* kernel_path_name(KernelPath p);

struct SubcaseCounters {
    std::uint64_t cross_tile = 0;
    std::uint64_t cross_tile_adj = 0;
    std::uint64_t cross_tile_diag = 0;
    SubcaseCounters& operator+=(const SubcaseCounters& o) {
        cross_tile += o.cross_tile;
        cross_tile_adj += o.cross_tile_adj;
        cross_tile_diag += o.cross_tile_diag;
        return *this;
    }
};

struct ApplyOptions {
    int threads = 1;            // accepted for source compatibility; the CUDA grid is used
    bool allow_native = true;
    bool count_subcases = true; // host-side diagnostic counters (off for benchmarking)
};

struct ApplyPlan {
    KernelPath path = KernelPath::dense_generic;
    ActiveQubits targets;
    SubcaseCounters subcases;
    std::uint64_t touched_bytes = 0;  // HBM bytes the launch reads + writes (algorithmic); extension
};

ApplyPlan apply(TiledHermitian& h, const ChannelSpec& spec, std::span<const std::uint32_t> targets,
                const ApplyOptions& opts = {});
ApplyPlan apply(TiledHermitian& h, const ChannelSpec& spec, std::initializer_list<std::uint32_t> targets,
                const ApplyOptions& opts = {});

void apply_tiled_intra(TiledHermitian& h, const TransferMatrix& s, std::uint32_t target, int threads = 1);
SubcaseCounters apply_tiled_cross(TiledHermitian& h, const TransferMatrix& s, std::uint32_t target,
                                  int threads = 1);
SubcaseCounters apply_tiled_twoqubit(TiledHermitian& h, const TransferMatrix& s, const ActiveQubits& qubits,
                                     int threads = 1);

// ------------------------------------------------------------------ native (native.hpp)
struct PermutationGate {
    int k = 0;
    std::vector<std::uint32_t> table;
    bool is_involution() const;
};
void apply_pauli_x(TiledHermitian& h, std::uint32_t target, int threads = 1);
void apply_pauli_y(TiledHermitian& h, std::uint32_t target, int threads = 1);
void apply_diagonal_phase(TiledHermitian& h, std::uint32_t target, const std::array<cplx, 2>& phases,
                          int threads = 1);
void apply_hadamard(TiledHermitian& h, std::uint32_t target, int threads = 1);
void apply_permutation(TiledHermitian& h, const PermutationGate& gate, const ActiveQubits& qubits,
                       int threads = 1);

// ---------------------------------------------------------- observables
double expectation(const TiledHermitian& rho, const TiledHermitian& obs);
double trace(const TiledHermitian& h);

}  // namespace hermsim_b200
