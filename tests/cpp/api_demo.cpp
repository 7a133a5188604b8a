// C++ caller of the hermsim_b200 API, written like a reference caller.
// Exit code 0 = all checks passed.
#include <cmath>
#include <complex>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <stdexcept>
#include <vector>

#include "hermsim_b200/hermsim.hpp"

using namespace hermsim_b200;

int main() {
    const int n = 9;
    TiledHermitian rho(n);
    // |0><0| payload: element (0, 0) of tile (0, 0)
    std::vector<cplx> payload(rho.element_count(), cplx{0.0, 0.0});
    payload[0] = 1.0;
    rho.upload(payload.data());
    ApplyPlan p = apply(rho, native_gate("h"), {0});
    if (p.path != KernelPath::native_hadamard)
        return 1;
    p = apply(rho, depolarising(0.1), {7});
    if (p.path != KernelPath::tiled_cross || p.subcases.cross_tile_diag == 0)
        return 2;
    p = apply(rho, native_gate("cnot"), {0, 8});  // control 0 (now |+>), target 8
    if (p.path != KernelPath::native_permutation)
        return 3;
    if (std::fabs(trace(rho) - 1.0) > 1e-12)
        return 4;
    // <Z_0 Z_8> on the Bell-like state = 1 (CNOT copies the H'd qubit 0 onto qubit 8)
    TiledHermitian zz(n);
    std::vector<cplx> o(zz.element_count(), cplx{0.0, 0.0});
    const std::uint64_t M = zz.tile_edge();
    for (std::uint64_t i = 0; i < zz.dim(); ++i) {
        const double v = ((i & 1) ^ ((i >> 8) & 1)) ? -1.0 : 1.0;
        o[tile_offset(i / M, i / M, M) + (i % M) * M + (i % M)] = v;
    }
    zz.upload(o.data());
    const double e = expectation(rho, zz);
    if (std::fabs(e - 1.0) > 1e-12) {
        std::printf("<ZZ> = %.17g\n", e);
        return 5;
    }
    try {
        apply(rho, native_gate("h"), {n});
        return 6;
    } catch (const std::out_of_range&) {
    }
    try {
        apply(rho, native_gate("cnot"), {1, 1});
        return 7;
    } catch (const std::invalid_argument&) {
    }
    TiledHermitian copy = rho;  // deep device copy
    if (std::fabs(trace(copy) - 1.0) > 1e-12)
        return 8;
    // checkpoint / resume through the reference's OHRM container (storage_io.hpp:22-29)
    const char* path = std::getenv("API_DEMO_OHRM");
    if (path) {
        save(rho, path);
        TiledHermitian back = load(path);
        if (std::fabs(expectation(back, zz) - e) > 0.0 || back.qubits() != n)
            return 9;
        try {
            load(std::string(path) + ".missing");
            return 10;
        } catch (const IoError& err) {
            if (err.kind() != IoErrorKind::io_failure)
                return 11;
        }
    }
    // generators of the reference's storage API, on the device
    TiledHermitian proj = basis_projector(n, 0);
    if (std::fabs(trace(proj) - 1.0) > 0.0 || std::fabs(expectation(proj, zz) - 1.0) > 0.0)
        return 12;
    TiledHermitian rh = random_hermitian(n, 42);
    if (!std::isfinite(trace(rh)))
        return 13;
    std::printf("api_demo ok: <Z0 Z8> = %.15f\n", e);
    return 0;
}
