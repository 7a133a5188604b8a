/*
 * hermsim_b200_c.h -- C facade of the hermsim_b200 C++ host API (channel model + apply
 * dispatcher) for FFI callers (Python ctypes in paper_2604_15765_b200/_native.py; the cgo /
 * JNI / ctypes stubs a reference maintainer would add are shown in INTEGRATION.md).
 *
 * Reference interfaces (arXiv 2604.15765, /root/reference/proj/include/hermsim):
 *   hb_channel_native       native_gate(name, theta)         channel.hpp:57-59, channel.cpp:95-154
 *   hb_channel_depolarising depolarising(p)                  channel.hpp:54-56, channel.cpp:82-93
 *   hb_channel_generic      make_generic(name, make_kraus_set(k, ops), validate, tol)
 *                                                            channel.hpp:52, channel.cpp:10-22,73-80
 *   hb_channel_dual         make_generic(dual_channel(kraus)) channel.hpp:74, channel.cpp:188-194
 *   hb_channel_transfer     ChannelSpec::transfer             channel.hpp:22-27, channel.cpp:24-34
 *   hb_bind                 bind_channel                      channel.hpp:78-92, channel.cpp:196-268
 *   hb_validate_cptni       validate_cptni                    channel.hpp:66-72, channel.cpp:168-186
 *   hb_apply                apply(h, spec, targets, opts)     kernels.hpp:58-61, kernels.cpp:510-549
 * States are the hs_state handles of hs_cuda.h (TiledHermitian in HBM).  Errors: HS_ERR_INVALID
 * for std::invalid_argument, HS_ERR_RANGE for std::out_of_range, message in hb_last_error().
 */
#ifndef HERMSIM_B200_C_H
#define HERMSIM_B200_C_H

#include "hs_cuda.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct hb_channel hb_channel;

/* GateKind (channel.hpp:36) */
enum hb_gate_kind { HB_GENERIC = 0, HB_PAULI_X = 1, HB_PAULI_Y = 2, HB_PHASE = 3, HB_HADAMARD = 4, HB_PERMUTATION = 5 };

const char* hb_last_error(void);
int hb_channel_native(const char* name, double theta, hb_channel** out);
int hb_channel_depolarising(double p, hb_channel** out);
/* ops: nops row-major 2^k x 2^k complex128 (interleaved re, im) */
int hb_channel_generic(const char* name, int k, int nops, const double* ops, int validate, double tol,
                       hb_channel** out);
int hb_channel_dual(const hb_channel* ch, hb_channel** out);
int hb_channel_free(hb_channel* ch);
int hb_channel_info(const hb_channel* ch, int* kind, int* k, int* nops);
int hb_channel_kraus(const hb_channel* ch, double* ops_out);      /* nops * 4^k complex */
int hb_channel_transfer(const hb_channel* ch, double* s_out);     /* 16^k complex, column-stacked */
int hb_channel_phases(const hb_channel* ch, double* phases_out);   /* 2 complex */
int hb_channel_perm(const hb_channel* ch, uint32_t* perm_out);     /* 2^k entries or none; returns count */
/* bind_channel: targets in constructor order -> ascending qubits, re-indexed Kraus ops (and perm). */
int hb_bind(const hb_channel* ch, const uint32_t* targets, int ntargets, uint32_t* sorted_out, double* ops_out,
            uint32_t* perm_out);
/* classification: 0 trace-preserving, 1 trace-non-increasing, 2 invalid */
int hb_validate_cptni(const hb_channel* ch, double tol, int* classification, double* max_dev, double* min_eig);
/* hermsim::apply.  plan may be NULL; count_subcases != 0 fills plan->subcases like the reference. */
int hb_apply(hs_state* h, const hb_channel* ch, const uint32_t* targets, int ntargets, int allow_native,
             int count_subcases, hs_plan* plan);

#ifdef __cplusplus
}
#endif
#endif /* HERMSIM_B200_C_H */
