/* A C caller of the ABI, no Python: 30-qubit register,
 * QuEST calls, qgpuRunCircuit, a single-precision register. Build:
 *   gcc tools/c_example.c -Iinclude -Lpaper_1802_08032_b200/_lib -lqgpu \
 *       -Wl,-rpath,$PWD/paper_1802_08032_b200/_lib -o /tmp/c_example */
#include "QuEST.h"
#include "qgpu.h"

int main(void) {
    QuESTEnv env = createQuESTEnv();
    Qureg q = createQureg(30, env);
    initZeroState(q);
    for (int t = 0; t < 30; ++t) hadamard(q, t);
    controlledPhaseShift(q, 3, 7, 0.25);
    qgpuOp ops[1] = {{0, 4, 1ull << 9, {0, 0, 1, 0, 1, 0, 0, 0}, 0, 0}};
    qgpuRunCircuit(q, ops, 1);
    Qureg s = qgpuCreateQuregPrecision(20, env, 0, 1);
    double p = calcProbOfOutcome(q, 5, 1);
    char msg[256];
    if (qgpuGetLastError(msg, sizeof msg)) { }
    destroyQureg(s, env);
    destroyQureg(q, env);
    qgpuJitShutdown();
    destroyQuESTEnv(env);
    return p > 0 ? 0 : 1;
}
