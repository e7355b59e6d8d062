/* A plain-C host of libkmf_b200.so (no Python, no torch): the context-free
 * operators on a fixed state, printed as hex doubles so the Python test can
 * compare them bit for bit with its own ctypes calls.
 *   gcc -std=c11 -I include tests/c/abi_smoke.c -L paper_2108_07031_b200 -lkmf_b200 */
#include <stdio.h>
#include <string.h>

#include "kmf_b200.h"

#define N 5

int main(void)
{
    if (kmf_abi_version() != KMF_ABI_VERSION) return 2;
    if (kmf_device_count() < 1) return 3;
    /* (4, n) row-major: rho, u1, u2, p */
    const double prims[4 * N] = {1.0, 1.1, 0.9, 1.05, 0.97,    0.6, 0.62, 0.58, 0.0, -0.3,
                                 0.02, 0.0, -0.05, 0.1, 0.2,   0.714, 0.8, 0.69, 0.7, 0.75};
    double q[4 * N], G[4 * N], U1[4 * N], res = 0.0;
    uint8_t flags[N];
    if (kmf_op_primitives_to_q(N, prims, 1.4, q, flags) != KMF_OK) return 4;
    if (kmf_op_split_flux(N, prims, 0, +1, 1.4, G) != KMF_OK) return 5;
    memcpy(U1, prims, sizeof U1);
    U1[2] += 1e-3;
    if (kmf_op_residue(N, U1, prims, &res) != KMF_OK) return 6;
    for (int k = 0; k < 4 * N; k++) printf("q %a\n", q[k]);
    for (int k = 0; k < 4 * N; k++) printf("G %a\n", G[k]);
    printf("res %a\n", res);
    return 0;
}
