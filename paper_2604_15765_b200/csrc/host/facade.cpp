// extern "C" facade of the hermsim_b200 C++ host API (include/hermsim_b200_c.h).
// Exceptions never cross the ABI: they become status codes plus hb_last_error().
#include <cstring>
#include <stdexcept>
#include <string>

#include "hermsim_b200/hermsim.hpp"
#include "hermsim_b200_c.h"

using namespace hermsim_b200;

namespace hermsim_b200 {
// api.cpp: the dispatcher on a borrowed state handle
ApplyPlan apply_on_handle(hs_state* hs, const ChannelSpec& spec, std::span<const std::uint32_t> targets,
                          const ApplyOptions& opts);
}  // namespace hermsim_b200

struct hb_channel {
    ChannelSpec spec;
};

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
    try {
        return f();
    } catch (const std::out_of_range& e) {
        g_err = e.what();
        return HS_ERR_RANGE;
    } catch (const std::invalid_argument& e) {
        g_err = e.what();
        return HS_ERR_INVALID;
    } catch (const std::exception& e) {
        g_err = e.what();
        return HS_ERR_CUDA;
    }
}

std::vector<Mat> unpack(int k, int nops, const double* ops) {
    if (k < 1 || k > 3)
        throw std::invalid_argument("Kraus set: locality must be 1..3");
    if (nops < 1)
        throw std::invalid_argument("Kraus set: needs at least one operator");
    if (!ops)
        throw std::invalid_argument("null operator array");
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

int emit(hb_channel** out, ChannelSpec spec) {
    if (!out)
        throw std::invalid_argument("null out");
    *out = new hb_channel{std::move(spec)};
    return HS_OK;
}
}  // namespace

extern "C" {

const char* hb_last_error(void) { return g_err.c_str(); }

int hb_channel_native(const char* name, double theta, hb_channel** out) {
    return guard([&] { return emit(out, native_gate(name ? name : "", theta)); });
}

int hb_channel_depolarising(double p, hb_channel** out) {
    return guard([&] { return emit(out, depolarising(p)); });
}

int hb_channel_generic(const char* name, int k, int nops, const double* ops, int validate, double tol,
                       hb_channel** out) {
    return guard([&] {
        return emit(out, make_generic(name ? name : "generic", make_kraus_set(k, unpack(k, nops, ops)),
                                      validate != 0, tol));
    });
}

int hb_channel_dual(const hb_channel* ch, hb_channel** out) {
    return guard([&] {
        if (!ch)
            throw std::invalid_argument("null channel");
        return emit(out, make_generic(ch->spec.name + "^dual", dual_channel(ch->spec.kraus)));
    });
}

int hb_channel_free(hb_channel* ch) {
    delete ch;
    return HS_OK;
}

int hb_channel_info(const hb_channel* ch, int* kind, int* k, int* nops) {
    return guard([&] {
        if (!ch)
            throw std::invalid_argument("null channel");
        if (kind)
            *kind = static_cast<int>(ch->spec.kind);
        if (k)
            *k = ch->spec.locality();
        if (nops)
            *nops = static_cast<int>(ch->spec.kraus.ops.size());
        return HS_OK;
    });
}

int hb_channel_kraus(const hb_channel* ch, double* ops_out) {
    return guard([&] {
        if (!ch || !ops_out)
            throw std::invalid_argument("null argument");
        const std::size_t d = ch->spec.kraus.local_dim();
        for (std::size_t a = 0; a < ch->spec.kraus.ops.size(); ++a)
            std::memcpy(ops_out + 2 * a * d * d, ch->spec.kraus.ops[a].data(), d * d * sizeof(cplx));
        return HS_OK;
    });
}

int hb_channel_transfer(const hb_channel* ch, double* s_out) {
    return guard([&] {
        if (!ch || !s_out)
            throw std::invalid_argument("null argument");
        const Mat& s = ch->spec.transfer.s;
        std::memcpy(s_out, s.data(), s.rows() * s.cols() * sizeof(cplx));
        return HS_OK;
    });
}

int hb_channel_phases(const hb_channel* ch, double* phases_out) {
    return guard([&] {
        if (!ch || !phases_out)
            throw std::invalid_argument("null argument");
        std::memcpy(phases_out, ch->spec.phases.data(), 2 * sizeof(cplx));
        return HS_OK;
    });
}

int hb_channel_perm(const hb_channel* ch, uint32_t* perm_out) {
    return guard([&] {
        if (!ch)
            throw std::invalid_argument("null channel");
        if (perm_out)
            for (std::size_t i = 0; i < ch->spec.perm.size(); ++i)
                perm_out[i] = ch->spec.perm[i];
        return static_cast<int>(ch->spec.perm.size());
    });
}

int hb_bind(const hb_channel* ch, const uint32_t* targets, int ntargets, uint32_t* sorted_out, double* ops_out,
            uint32_t* perm_out) {
    return guard([&] {
        if (!ch || !targets || ntargets < 0)
            throw std::invalid_argument("null argument");
        const BoundChannel b = bind_channel(ch->spec, std::span<const uint32_t>(targets, ntargets));
        if (sorted_out)
            for (int i = 0; i < b.qubits.count(); ++i)
                sorted_out[i] = b.qubits[i];
        if (ops_out) {
            const std::size_t d = b.kraus.local_dim();
            for (std::size_t a = 0; a < b.kraus.ops.size(); ++a)
                std::memcpy(ops_out + 2 * a * d * d, b.kraus.ops[a].data(), d * d * sizeof(cplx));
        }
        if (perm_out)
            for (std::size_t i = 0; i < b.perm.size(); ++i)
                perm_out[i] = b.perm[i];
        return HS_OK;
    });
}

int hb_validate_cptni(const hb_channel* ch, double tol, int* classification, double* max_dev, double* min_eig) {
    return guard([&] {
        if (!ch)
            throw std::invalid_argument("null channel");
        const ValidationReport r = validate_cptni(ch->spec.kraus, tol);
        if (classification)
            *classification = static_cast<int>(r.classification);
        if (max_dev)
            *max_dev = r.max_deviation;
        if (min_eig)
            *min_eig = r.min_eigenvalue;
        return HS_OK;
    });
}

// hermsim::apply on a device state wrapped by a borrowed handle.
int hb_apply(hs_state* h, const hb_channel* ch, const uint32_t* targets, int ntargets, int allow_native,
             int count_subcases, hs_plan* plan) {
    return guard([&] {
        if (!h || !ch || (!targets && ntargets))
            throw std::invalid_argument("null argument");
        int n = 0;
        if (hs_state_info(h, &n, nullptr, nullptr, nullptr) != HS_OK)
            throw std::invalid_argument(hs_last_error());
        ApplyOptions o;
        o.allow_native = allow_native != 0;
        o.count_subcases = count_subcases != 0;
        const ApplyPlan p = apply_on_handle(h, ch->spec, std::span<const uint32_t>(targets, ntargets), o);
        if (plan) {
            std::memset(plan, 0, sizeof(*plan));
            plan->path = static_cast<int>(p.path);
            plan->k = p.targets.count();
            for (int i = 0; i < p.targets.count(); ++i)
                plan->targets[i] = p.targets[i];
            plan->subcases[0] = p.subcases.cross_tile;
            plan->subcases[1] = p.subcases.cross_tile_adj;
            plan->subcases[2] = p.subcases.cross_tile_diag;
            plan->touched_bytes = p.touched_bytes;
        }
        return HS_OK;
    });
}

}  // extern "C"
