/*
 * QuEST.h — the C-ABI of the B200-native gate-path backend (libqgpu.so).
 *
 * Drop-in boundary. The entry points carry QuEST's names and argument meaning
 * (BASELINE.json north star); each one replaces the reference operation cited
 * beside it (paths under /root/reference/proj). Semantics follow the
 * reference where it has the operation; operations the reference lacks are
 * restated and marked "restated".
 *
 * Conventions
 *  - Amplitudes are complex double, qubit q contributes 2^q to an index
 *    (register.hpp:47-50); a density matrix rho_jk lives at flat index
 *    j + 2^N k. All state lives in HBM; nothing is mirrored on the host.
 *  - Calls are stream-ordered and asynchronous. Gates, channels and collapse
 *    are queued and fused into HBM passes; any call that returns a value
 *    (probabilities, amplitudes) or syncQuESTEnv() completes all queued work
 *    first. Results are identical to applying every call immediately.
 *  - Errors: invalid input is detected on the host BEFORE any mutation, with
 *    the reference's rules (kernels.cpp:22-41, density.cpp:17-22, 121-123,
 *    135-138, register.cpp:31-53, 106-117). The call then invokes
 *    invalidQuESTInputError(msg, func) and returns without effect. The
 *    library's default handler records the message (qgpuGetLastError) instead
 *    of exiting; a program may define its own invalidQuESTInputError (as with
 *    QuEST) or install one with qgpuSetErrorHandler. Nothing throws across
 *    the ABI.
 *  - Handles are plain structs passed by value; the library owns all device
 *    memory.
 */
#ifndef QGPU_QUEST_H
#define QGPU_QUEST_H

#ifdef __cplusplus
extern "C" {
#endif

typedef double qreal;

typedef struct Complex {
    qreal real;
    qreal imag;
} Complex;

typedef struct ComplexMatrix2 {
    qreal real[2][2];
    qreal imag[2][2];
} ComplexMatrix2;

typedef struct Vector {
    qreal x, y, z;
} Vector;

/* One process per GPU. rank/numRanks describe the amplitude partition
 * (distributed.hpp:26-44); the single-GPU env has rank 0 of 1. */
typedef struct QuESTEnv {
    int rank;
    int numRanks;
    void* impl;
} QuESTEnv;

/* Mirrors the reference Register (register.hpp:51-86). numAmpsPerChunk is
 * this rank's share 2^(flat-k); chunkId = rank. */
typedef struct Qureg {
    int isDensityMatrix;
    int numQubitsRepresented;
    int numQubitsInStateVec;
    long long int numAmpsPerChunk;
    long long int numAmpsTotal;
    int chunkId;
    int numChunks;
    void* impl;
} Qureg;

/* ------------------------------------------------------------ environment */
QuESTEnv createQuESTEnv(void);                 /* device 0, single rank */
void destroyQuESTEnv(QuESTEnv env);
void syncQuESTEnv(QuESTEnv env);                /* transport.barrier(), distributed.cpp:348-352 */
int syncQuESTSuccess(int successCode);
void reportQuESTEnv(QuESTEnv env);
/* seedQuEST: the measurement RNG (SplitMix64, circuit.cpp:20-25) state is
 * the fold of the seeds (restated; the reference has no measurement). */
void seedQuEST(QuESTEnv* env, unsigned long int* seedArray, int numSeeds);
void seedQuESTDefault(QuESTEnv* env);

/* --------------------------------------------------------------- registers */
Qureg createQureg(int numQubits, QuESTEnv env);        /* Register(n, StateVector), register.cpp:101-121 */
Qureg createDensityQureg(int numQubits, QuESTEnv env); /* Register(n, DensityMatrix) */
Qureg createCloneQureg(Qureg qureg, QuESTEnv env);
void destroyQureg(Qureg qureg, QuESTEnv env);          /* ~Register */
int getNumQubits(Qureg qureg);
long long int getNumAmps(Qureg qureg);

/* ----------------------------------------------------------- initialisers */
void initZeroState(Qureg qureg);                       /* Register::init_zero_state, register.cpp:127-130 */
void initPlusState(Qureg qureg);
void initClassicalState(Qureg qureg, long long int stateInd);
void initStateFromAmps(Qureg qureg, qreal* reals, qreal* imags);
void setAmps(Qureg qureg, long long int startInd, qreal* reals, qreal* imags,
             long long int numAmps);                   /* set_amplitude, register.cpp:42-53 */
void cloneQureg(Qureg targetQureg, Qureg copyQureg);

/* ------------------------------------------------------------- amplitudes */
Complex getAmp(Qureg qureg, long long int index);      /* get_amplitude, register.cpp:31-40 */
qreal getRealAmp(Qureg qureg, long long int index);
qreal getImagAmp(Qureg qureg, long long int index);
qreal getProbAmp(Qureg qureg, long long int index);
Complex getDensityAmp(Qureg qureg, long long int row, long long int col);

/* ------------------------------------------------------------------ gates */
/* All single-target gates map to apply_controlled_gate (kernels.cpp:105-112)
 * for state vectors and apply_gate_to_density (density.cpp:85-116) for
 * density matrices, with the matrices of gates.cpp:51-98. */
void hadamard(Qureg qureg, int targetQubit);            /* gate_matrix(H) gates.cpp:55-56 */
void pauliX(Qureg qureg, int targetQubit);              /* gates.cpp:59-60 */
void pauliY(Qureg qureg, int targetQubit);              /* gates.cpp:61-62 */
void pauliZ(Qureg qureg, int targetQubit);              /* gates.cpp:63-66 */
void sGate(Qureg qureg, int targetQubit);               /* diag(1, i) */
void tGate(Qureg qureg, int targetQubit);               /* gates.cpp:57-58 */
void phaseShift(Qureg qureg, int targetQubit, qreal angle);          /* diag(1, e^{i angle}) */
void rotateX(Qureg qureg, int rotQubit, qreal angle);   /* rotation_matrix({1,0,0}), gates.cpp:75-98 */
void rotateY(Qureg qureg, int rotQubit, qreal angle);
void rotateZ(Qureg qureg, int rotQubit, qreal angle);
void rotateAroundAxis(Qureg qureg, int rotQubit, qreal angle, Vector axis); /* apply_single_qubit_rotation, kernels.cpp:124-132 */
void compactUnitary(Qureg qureg, int targetQubit, Complex alpha, Complex beta); /* restated: [[a, -b*], [b, a*]] */
void unitary(Qureg qureg, int targetQubit, ComplexMatrix2 u);        /* apply_single_qubit_gate + is_unitary, gates.cpp:16-32 */

void controlledNot(Qureg qureg, int controlQubit, int targetQubit);  /* apply_controlled_gate({c}, t, X) */
void controlledPauliY(Qureg qureg, int controlQubit, int targetQubit);
void controlledPhaseFlip(Qureg qureg, int idQubit1, int idQubit2);   /* apply_controlled_gate({q2}, q1, Z) */
void controlledPhaseShift(Qureg qureg, int idQubit1, int idQubit2, qreal angle); /* restated: ({q2}, q1, diag(1, e^{i angle})) */
void multiControlledPhaseFlip(Qureg qureg, int* controlQubits, int numControlQubits); /* restated */
void multiControlledPhaseShift(Qureg qureg, int* controlQubits, int numControlQubits, qreal angle);
void controlledRotateX(Qureg qureg, int controlQubit, int targetQubit, qreal angle);
void controlledRotateY(Qureg qureg, int controlQubit, int targetQubit, qreal angle);
void controlledRotateZ(Qureg qureg, int controlQubit, int targetQubit, qreal angle);
void controlledRotateAroundAxis(Qureg qureg, int controlQubit, int targetQubit, qreal angle,
                                Vector axis);
void controlledCompactUnitary(Qureg qureg, int controlQubit, int targetQubit, Complex alpha,
                              Complex beta);
void controlledUnitary(Qureg qureg, int controlQubit, int targetQubit, ComplexMatrix2 u);
void multiControlledUnitary(Qureg qureg, int* controlQubits, int numControlQubits,
                            int targetQubit, ComplexMatrix2 u);

/* ------------------------------------------------------------ measurement */
qreal calcTotalProb(Qureg qureg);          /* SV: sum |a|^2 (register.cpp:62-75, compensated); DM: Re trace (density.cpp:147-154) */
qreal calcProbOfOutcome(Qureg qureg, int measureQubit, int outcome); /* restated */
qreal collapseToOutcome(Qureg qureg, int measureQubit, int outcome); /* restated; returns the outcome's probability */
int measure(Qureg qureg, int measureQubit);                          /* restated */
int measureWithStats(Qureg qureg, int measureQubit, qreal* outcomeProb);
qreal calcPurity(Qureg qureg);             /* purity, density.cpp:156-159 */

/* ------------------------------------------------------------------ noise */
void mixDephasing(Qureg qureg, int targetQubit, qreal prob);    /* apply_dephasing, density.cpp:118-130 */
void mixDepolarising(Qureg qureg, int targetQubit, qreal prob); /* apply_depolarising, density.cpp:132-145 */

/* ----------------------------------------------------------------- errors */
/* Invoked on invalid input before any mutation (see header comment). */
void invalidQuESTInputError(const char* errMsg, const char* errFunc);

#ifdef __cplusplus
}
#endif

#endif /* QGPU_QUEST_H */
