/*
 * oracle_ops.h — TEST INFRASTRUCTURE ONLY (never linked into the product).
 *
 * Shared op-record layout used by the two CPU checkers under oracle/:
 *   - oracle/_ref/libqsimref_shim.so : the reference C++ library compiled from
 *     /root/reference/proj/src/*.cpp (see oracle/Makefile) behind a C shim
 *     (oracle/ref_shim.cpp);
 *   - oracle/_build/libqsim_oracle.so : the plain-C restatement
 *     (oracle/qsim_oracle.c).
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
 * either library.
 */
#ifndef QSIM_ORACLE_OPS_H
#define QSIM_ORACLE_OPS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum orc_op_kind {
    ORC_GATE = 0,      /* 2x2 matrix m on target, controls in ctrl_mask      */
    ORC_DEPHASE = 1,   /* density only: apply_dephasing(target, param)       */
    ORC_DEPOLARISE = 2,/* density only: apply_depolarising(target, param)    */
};

/* 96 bytes, no padding surprises: identical in C, C++ and numpy. */
typedef struct orc_op {
    int32_t kind;
    int32_t target;     /* ket qubit (density) or qubit (state vector)      */
    uint64_t ctrl_mask; /* bit c set <=> qubit c is a control               */
    double m[8];        /* re/im of m00, m01, m10, m11                      */
    double param;       /* channel probability                              */
    double pad;
} orc_op;

#ifdef __cplusplus
}
#endif

#endif
