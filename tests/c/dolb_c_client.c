/* Plain-C client of include/dolb.h (what tools/dolb_cli.cpp and
 * tests/test_capi.cpp do through the reference's libdolb.so): links against
 * this repository's libdolb.so. argv[1] = "cpu" (configuration / model
 * queries only) or "gpu" (also a tiny dolb_run into argv[2]). */
#include <stdio.h>
#include <string.h>

#include "dolb.h"

#define CHECK(call)                                                                     \
    do {                                                                                \
        dolb_status s_ = (call);                                                        \
        if (s_ != DOLB_OK) {                                                            \
            fprintf(stderr, "%s -> %d: %s\n", #call, (int)s_, dolb_last_error());       \
            return 1;                                                                   \
        }                                                                               \
    } while (0)

int main(int argc, char** argv) {
    const int gpu = argc > 1 && strcmp(argv[1], "gpu") == 0;
    printf("version %s\n", dolb_version());
    if (dolb_run(NULL, NULL, NULL) != DOLB_ERROR_INVALID_ARGUMENT) return 2;

    dolb_config* cfg = dolb_config_new();
    CHECK(dolb_config_set(cfg, "case.kind", "cavity"));
    CHECK(dolb_config_set(cfg, "case.L", "16"));
    CHECK(dolb_config_set(cfg, "case.collision", "trt"));
    size_t len = 0;
    CHECK(dolb_show_models(cfg, NULL, 0, &len));
    char models[256];
    if (len > sizeof models) return 3;
    CHECK(dolb_show_models(cfg, models, sizeof models, NULL));
    printf("models:\n%s", models);

    int64_t bytes = 0;
    CHECK(dolb_bytes_per_cell(32, &bytes));
    double glups = 0.0;
    CHECK(dolb_peak_glups("A100-SXM4-40GB", NULL, 32, &glups));
    printf("bytes_per_cell %lld peak_glups %.3f\n", (long long)bytes, glups);

    dolb_config* bad = dolb_config_new();
    CHECK(dolb_config_set(bad, "case.kind", "vortex-street"));
    if (dolb_run(bad, NULL, NULL) != DOLB_ERROR_CONFIG) return 4;
    printf("config error: %s\n", dolb_last_error());
    dolb_config_free(bad);

    if (gpu) {
        CHECK(dolb_config_set(cfg, "run.tmax", "40"));
        CHECK(dolb_config_set(cfg, "run.output_every", "20"));
        CHECK(dolb_config_set(cfg, "run.out", argc > 2 ? argv[2] : "out"));
        int64_t steps = 0;
        double mlups = 0.0;
        CHECK(dolb_run(cfg, &steps, &mlups));
        printf("run steps %lld mlups %.1f\n", (long long)steps, mlups);
        if (steps != 40 || !(mlups > 0.0)) return 5;
    }
    dolb_config_free(cfg);
    return 0;
}
