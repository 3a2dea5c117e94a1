"""The C-ABI header is plain C: a C11 program (the INTEGRATION.md solve loop)
compiles against include/acs_gpu.h with -Wall -Werror, links
libacs_b200.so and runs.  Host-only entry points must work without a GPU;
the compute entry points must fail loudly (ACS_E_CUDA) when there is no
device -- there is no CPU fallback."""
import os
import subprocess

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

C_SRC = r"""
#include <stdio.h>
#include <stdlib.h>
#include "acs_gpu.h"

int main(void) {
    if (acs_gpu_abi_version() != ACS_GPU_ABI_VERSION) return 10;
    double xs[64], ys[64];
    if (acs_random_instance(64, 20161017, 1000000, xs, ys) != ACS_OK) return 11;
    if (xs[0] != 120054.0 || ys[0] != 324231.0) return 12;   /* SURVEY 8(d) config-5 first node */
    const double a[4] = {1, 2, 3, 4}, b[4] = {5, 6, 7, 8};
    double p = 0.0;
    if (acs_rank_sum_test(a, 4, b, 4, &p) != ACS_OK || !(p > 0.0 && p < 0.05)) return 13;
    const char *tsp = "NAME: t5\nTYPE: TSP\nDIMENSION: 5\nEDGE_WEIGHT_TYPE: EUC_2D\nNODE_COORD_SECTION\n"
                      "1 0 0\n2 3 0\n3 3 4\n4 0 4\n5 1 1\nEOF\n";
    uint32_t n = 0, type = 9;
    double px[5], py[5];
    size_t len = 0;
    while (tsp[len]) ++len;
    if (acs_parse_tsplib(tsp, len, &n, &type, NULL, NULL, 0, NULL, 0) != ACS_OK || n != 5) return 14;  /* size query */
    if (acs_parse_tsplib(tsp, len, &n, &type, px, py, 5, NULL, 0) != ACS_OK || type != ACS_EUC_2D) return 19;
    int devices = 0;
    acs_gpu_device_count(&devices);
    acs_instance_desc d = {n, ACS_EUC_2D, px, py};
    acs_params prm = {3.0, 0.2, 0.01, -1.0, 32, 0, 8, 1, ACS_VARIANT_ATOMIC, ACS_RNG_XOSHIRO, 1};
    acs_gpu_ctx *ctx = NULL;
    const int rc = acs_gpu_create(&d, &prm, 0, &ctx);
    if (devices == 0) {
        if (rc != ACS_E_CUDA || ctx != NULL || acs_gpu_last_error()[0] == 0) return 15;
        printf("no device: %s\n", acs_gpu_last_error());
        return 0;
    }
    if (rc != ACS_OK) { fprintf(stderr, "%s\n", acs_gpu_last_error()); return 16; }
    acs_iter_stats st[4];
    if (acs_gpu_iterate(ctx, 4, st) != ACS_OK) return 17;
    uint32_t order[5];
    int64_t best = 0;
    if (acs_gpu_get_best(ctx, order, &best) != ACS_OK || best != st[3].global_best_len) return 18;
    acs_gpu_destroy(ctx);
    printf("solved: %lld\n", (long long)best);
    return 0;
}
"""


def test_c11_program_against_header(tmp_path):
    src = tmp_path / "abi.c"
    src.write_text(C_SRC)
    exe = tmp_path / "abi"
    lib_dir = os.path.join(REPO, "paper_1605_02669_b200")
    cc = subprocess.run(["gcc", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", os.path.join(REPO, "include"),
                         str(src), "-o", str(exe), "-L", lib_dir, "-lacs_b200", f"-Wl,-rpath,{lib_dir}"],
                        capture_output=True, text=True)
    assert cc.returncode == 0, cc.stderr
    run = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert run.returncode == 0, (run.returncode, run.stdout, run.stderr)
