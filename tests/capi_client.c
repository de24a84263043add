/*
 * tests/capi_client.c -- a plain C client of the reference ABI (include/wrs.h)
 * linked against libwrs_b200.so, the way the reference's own clients link
 * libwrs (proj/tests/test_capi.cpp:12-112 exercises the same calls; this file
 * is an independent C program, not a copy).  It goes through the handle
 * lifecycle, validation errors, the WRS1 round trip, build -> verify -> draw
 * (determinism, range), the bulk (item, count) call, and the algorithms the
 * B200 library declines.
 *
 *   capi_client            on a GPU box: every call must succeed
 *   capi_client --no-gpu   without a GPU: compute calls must fail loudly
 *                          (WRS_EINTERNAL) while argument checks still work
 * Exit status 0 when every check holds; prints the first failure otherwise.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "wrs.h"

static int failures = 0;
#define CHECK(cond)                                                            \
    do {                                                                       \
        if (!(cond)) {                                                         \
            fprintf(stderr, "CHECK failed at line %d: %s (last error: %s)\n",  \
                    __LINE__, #cond, wrs_last_error());                        \
            ++failures;                                                        \
        }                                                                      \
    } while (0)

static int no_gpu_run(void) {
    const double w[4] = {3, 1, 1, 1};
    wrs_weights* h = NULL;
    CHECK(wrs_weights_from_array(NULL, 4, &h) == WRS_EINVAL);
    CHECK(wrs_weights_from_array(w, 4, &h) == WRS_EINTERNAL);
    CHECK(strlen(wrs_last_error()) > 0);
    CHECK(wrs_weights_generate("uniform", 0.0, 100, 1, &h) == WRS_EINTERNAL);
    CHECK(strcmp(wrs_status_name(WRS_EVERIFY), "WRS_EVERIFY") == 0);
    CHECK(wrs_sampler_build(NULL, "psa", 1, 0, NULL) == WRS_EINVAL);
    return failures;
}

static int gpu_run(void) {
    /* weights lifecycle */
    const double w4[4] = {3, 1, 1, 1};
    wrs_weights* h = NULL;
    CHECK(wrs_weights_from_array(w4, 4, &h) == WRS_OK && h);
    CHECK(wrs_weights_count(h) == 4);
    CHECK(memcmp(wrs_weights_values(h), w4, sizeof w4) == 0);
    wrs_weights_free(h);

    /* validation with a message */
    const double bad[2] = {1.0, -1.0};
    CHECK(wrs_weights_from_array(bad, 2, &h) == WRS_EINVAL);
    CHECK(strlen(wrs_last_error()) > 0);

    /* WRS1 round trip */
    wrs_weights *gen = NULL, *back = NULL;
    CHECK(wrs_weights_generate("powerlaw", 1.5, 500, 42, &gen) == WRS_OK);
    const char* path = "capi_client_roundtrip.wrs";
    CHECK(wrs_weights_write(gen, path) == WRS_OK);
    CHECK(wrs_weights_read(path, &back) == WRS_OK);
    CHECK(wrs_weights_count(back) == 500);
    CHECK(memcmp(wrs_weights_values(back), wrs_weights_values(gen), 500 * sizeof(double)) == 0);
    remove(path);
    wrs_weights_free(back);
    wrs_weights_free(gen);
    CHECK(wrs_weights_read("no_such_file.wrs", &back) == WRS_EIO);
    CHECK(wrs_weights_generate("cauchy", 0.0, 10, 1, &back) == WRS_EINVAL);

    /* build, verify, draw */
    wrs_weights* w = NULL;
    CHECK(wrs_weights_generate("powerlaw", 2.0, 1000, 7, &w) == WRS_OK);
    const char* algos[2] = {"psa", "psa-exact"};
    for (int a = 0; a < 2; ++a) {
        wrs_sampler* s = NULL;
        CHECK(wrs_sampler_build(w, algos[a], 4, 0, &s) == WRS_OK && s);
        CHECK(wrs_sampler_verify_masses(s, 1e-9) == WRS_OK);
        enum { K = 10000 };
        static uint32_t out[K], again[K];
        CHECK(wrs_sampler_draw(s, 123, K, 2, out) == WRS_OK);
        for (int i = 0; i < K; ++i)
            if (out[i] >= 1000) {
                CHECK(out[i] < 1000);
                break;
            }
        CHECK(wrs_sampler_draw(s, 123, K, 2, again) == WRS_OK);
        CHECK(memcmp(out, again, sizeof out) == 0);
        wrs_sampler_free(s);
    }
    wrs_sampler* s = NULL;
    CHECK(wrs_sampler_build(w, "bogus", 1, 0, &s) == WRS_EINVAL);
    CHECK(wrs_sampler_build(w, "vose", 1, 0, &s) == WRS_EINVAL); /* outside the B200 path */
    wrs_weights_free(w);

    /* bulk with replacement: distinct items with multiplicities summing to k,
     * independent of the worker count */
    CHECK(wrs_weights_generate("powerlaw", 1.5, 200, 11, &w) == WRS_OK);
    uint32_t items[200], items2[200];
    uint64_t counts[200], counts2[200], u = 0, u2 = 0;
    CHECK(wrs_sample_with_replacement(w, 5000, 9, 2, items, counts, &u) == WRS_OK);
    CHECK(wrs_sample_with_replacement(w, 5000, 9, 7, items2, counts2, &u2) == WRS_OK);
    uint64_t total = 0;
    for (uint64_t i = 0; i < u; ++i) {
        CHECK(items[i] < 200);
        if (i) CHECK(items[i] > items[i - 1]);
        total += counts[i];
    }
    CHECK(total == 5000);
    CHECK(u2 == u && memcmp(items, items2, u * 4) == 0 && memcmp(counts, counts2, u * 8) == 0);
    CHECK(wrs_sample_with_replacement(NULL, 5000, 9, 1, items, counts, &u) == WRS_EINVAL);
    wrs_weights_free(w);
    return failures;
}

int main(int argc, char** argv) {
    const int f = (argc > 1 && strcmp(argv[1], "--no-gpu") == 0) ? no_gpu_run() : gpu_run();
    if (f) {
        fprintf(stderr, "capi client: %d check(s) failed\n", f);
        return 1;
    }
    printf("capi client ok\n");
    return 0;
}
