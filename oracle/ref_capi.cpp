// C-ABI shim over the compiled reference library (arXiv 2604.15765, /root/reference/proj).
//
// TEST INFRASTRUCTURE ONLY.  Built by oracle/build_ref.sh into oracle/_ref/ and loaded by
// tests/ (as the parity anchor and golden-vector generator) and by bench.py's reference /
// cpu_baseline leg.  It only forwards to the reference's own public API:
//   hermsim::TiledHermitian / MatrixHandle   (storage.hpp:60-124)
//   hermsim::apply                           (kernels.hpp:58-61, kernels.cpp:510-549)
//   hermsim::native_gate / depolarising / make_generic / dual_channel (channel.hpp:54-92)
//   hermsim::gaussian_entry, footprint_bytes, to_dense (storage.hpp:129-154)
//   hermsim::insert_bits / tile_offset       (bit_index.hpp:40-83)
//   hermsim::save / load                     (storage_io.hpp:22-29)
// Errors are caught and reported as negative return codes (the reference throws).
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <vector>

#include "hermsim/bit_index.hpp"
#include "hermsim/channel.hpp"
#include "hermsim/kernels.hpp"
#include "hermsim/storage.hpp"
#include "hermsim/storage_io.hpp"

using namespace hermsim;

namespace {
thread_local std::string g_err;

int fail(const std::exception& e) {
    g_err = e.what();
    return -1;
}

std::vector<Mat> unpack_ops(int k, int nops, const double* ops) {
    const std::size_t d = std::size_t{1} << k;
    std::vector<Mat> v;
    for (int a = 0; a < nops; ++a) {
        Mat m(d, d);
        for (std::size_t i = 0; i < d * d; ++i)
            m.data()[i] = cplx(ops[2 * (a * d * d + i)], ops[2 * (a * d * d + i) + 1]);
        v.push_back(std::move(m));
    }
    return v;
}
} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_tiled_create(int n, int m) {
    try {
        return new MatrixHandle(TiledHermitian(n, m));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_dense_create(int n) {
    try {
        return new MatrixHandle(DenseHermitian(n));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_free(void* h) { delete static_cast<MatrixHandle*>(h); }

// hermsim::save / load (storage_io.cpp:34-118): the OHRM container.
int ref_save(void* h, const char* path) {
    try {
        save(*static_cast<MatrixHandle*>(h), std::string(path));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

void* ref_load(const char* path) {
    try {
        return new MatrixHandle(load(std::string(path)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

double* ref_payload(void* h) { return reinterpret_cast<double*>(static_cast<MatrixHandle*>(h)->payload()); }

uint64_t ref_payload_count(void* h) { return static_cast<MatrixHandle*>(h)->payload_count(); }

int ref_format(void* h) { return static_cast<int>(static_cast<MatrixHandle*>(h)->format()); }

// Converts into a fresh dense handle (storage.cpp:241-283).
void* ref_to_dense(void* h) {
    try {
        return new MatrixHandle(to_dense(*static_cast<MatrixHandle*>(h)));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

// hermsim::convert (storage.cpp:285-292) into a fresh handle of `format` (dense 0, packed 1, tiled 2).
void* ref_convert(void* h, int format, int m) {
    try {
        return new MatrixHandle(convert(*static_cast<MatrixHandle*>(h), static_cast<Format>(format), m));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void* ref_random_hermitian(int n, uint64_t seed, int format, int m) {
    try {
        return new MatrixHandle(random_hermitian(n, seed, static_cast<Format>(format), m));
    } catch (const std::exception& e) {
        fail(e);
        return nullptr;
    }
}

void ref_gaussian_entry(uint64_t seed, uint64_t counter, double* out2) {
    const cplx z = gaussian_entry(seed, counter);
    out2[0] = z.real();
    out2[1] = z.imag();
}

uint64_t ref_footprint_bytes(int n, int m, int format) {
    try {
        return footprint_bytes(n, m, static_cast<Format>(format));
    } catch (const std::exception& e) {
        fail(e);
        return 0;
    }
}

uint64_t ref_insert_bits(uint64_t s, uint64_t a, const uint32_t* pos, int k) {
    return insert_bits(s, a, ActiveQubits(std::span<const uint32_t>(pos, k)));
}

uint64_t ref_tile_offset(uint64_t ti, uint64_t tj, uint64_t M) { return tile_offset(ti, tj, M); }

static int finish_apply(void* h, const ChannelSpec& spec, const uint32_t* targets, int k, int threads,
                        int allow_native, uint64_t* subcases) {
    ApplyOptions o;
    o.threads = threads;
    o.allow_native = allow_native != 0;
    const ApplyPlan p = apply(*static_cast<MatrixHandle*>(h), spec, std::span<const uint32_t>(targets, k), o);
    if (subcases) {
        subcases[0] = p.subcases.cross_tile;
        subcases[1] = p.subcases.cross_tile_adj;
        subcases[2] = p.subcases.cross_tile_diag;
    }
    return static_cast<int>(p.path);
}

// hermsim::apply(h, native_gate(name, theta), targets, {threads, allow_native})
int ref_apply_native(void* h, const char* name, double theta, const uint32_t* targets, int k, int threads,
                     int allow_native, uint64_t* subcases) {
    try {
        return finish_apply(h, native_gate(name, theta), targets, k, threads, allow_native, subcases);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// hermsim::apply(h, depolarising(p), {target})
int ref_apply_depolarising(void* h, double p, uint32_t target, int threads, uint64_t* subcases) {
    try {
        return finish_apply(h, depolarising(p), &target, 1, threads, 1, subcases);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// hermsim::apply(h, make_generic("g", {ops}), targets); ops = nops row-major 2^k x 2^k complex;
// dual != 0 applies dual_channel (Heisenberg picture, channel.cpp:188-194).
int ref_apply_generic(void* h, int k, int nops, const double* ops, const uint32_t* targets, int threads, int dual,
                      uint64_t* subcases) {
    try {
        KrausSet ks = make_kraus_set(k, unpack_ops(k, nops, ops));
        if (dual)
            ks = dual_channel(ks);
        return finish_apply(h, make_generic("generic", std::move(ks)), targets, k, threads, 1, subcases);
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// Transfer matrix of a Kraus set (channel.cpp:24-34), column-stacked convention.
int ref_transfer_from_kraus(int k, int nops, const double* ops, double* s_out) {
    try {
        const TransferMatrix t = transfer_from_kraus(make_kraus_set(k, unpack_ops(k, nops, ops)));
        std::memcpy(s_out, t.s.data(), t.s.rows() * t.s.cols() * sizeof(cplx));
        return 0;
    } catch (const std::exception& e) {
        return fail(e);
    }
}

// bind_channel of native_gate(name) to targets (channel.cpp:196-268): sorted qubits, bound L, perm.
int ref_bind_native(const char* name, double theta, const uint32_t* targets, int k, uint32_t* sorted_out,
                    double* l_out, uint32_t* perm_out) {
    try {
        const BoundChannel b = bind_channel(native_gate(name, theta), std::span<const uint32_t>(targets, k));
        for (int i = 0; i < k; ++i)
            sorted_out[i] = b.qubits[i];
        const Mat& l = b.kraus.ops.at(0);
        std::memcpy(l_out, l.data(), l.rows() * l.cols() * sizeof(cplx));
        for (std::size_t i = 0; i < b.perm.size(); ++i)
            perm_out[i] = b.perm[i];
        return static_cast<int>(b.perm.size());
    } catch (const std::exception& e) {
        return fail(e);
    }
}

} // extern "C"
