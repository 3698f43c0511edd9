/* Plain-C use of the drop-in boundary (include/kvrail_c.h): run a scenario
 * (the reference's JSON schema, scenario.cpp:829-924) step by step through the
 * C-ABI and print the reference-format steps.csv. With a device index the step
 * runs on that B200; with -1 the host-only twin runs it.
 *
 *   cc -I include examples/c_driver.c -L paper_2605_09735_b200/lib -lkvrail \
 *      -Wl,-rpath,$PWD/paper_2605_09735_b200/lib -o c_driver
 *   ./c_driver config.json [device]
 */
#include <stdio.h>
#include <stdlib.h>

#include "kvrail_c.h"

static char *slurp(const char *path) {
    FILE *f = fopen(path, "rb");
    if (!f)
        return NULL;
    fseek(f, 0, SEEK_END);
    long n = ftell(f);
    fseek(f, 0, SEEK_SET);
    char *buf = malloc((size_t)n + 1);
    if (buf && fread(buf, 1, (size_t)n, f) != (size_t)n) {
        free(buf);
        buf = NULL;
    }
    if (buf)
        buf[n] = 0;
    fclose(f);
    return buf;
}

int main(int argc, char **argv) {
    if (argc < 2) {
        fprintf(stderr, "usage: %s config.json [device]\n", argv[0]);
        return 2;
    }
    char *cfg = slurp(argv[1]);
    if (!cfg) {
        fprintf(stderr, "cannot read %s\n", argv[1]);
        return 2;
    }
    const int device = argc > 2 ? atoi(argv[2]) : -1;
    kvr_driver *d = NULL;
    if (kvr_driver_create(cfg, device, &d) != 0) {
        fprintf(stderr, "kvr_driver_create: %s\n", kvr_last_error());
        return 1;
    }
    uint64_t done = 0, total = 0;
    kvr_driver_progress(d, &done, &total);
    kvr_step_record rec;
    uint64_t emitted = 0;
    while (done < total) {
        if (kvr_driver_step(d, &rec) != 0) {
            fprintf(stderr, "kvr_driver_step: %s\n", kvr_last_error());
            return 1;
        }
        emitted += rec.emitted_tokens;
        kvr_driver_progress(d, &done, &total);
    }
    uint64_t len = 0;
    kvr_driver_steps_csv(d, NULL, 0, &len); /* size query */
    char *csv = malloc(len + 1);
    kvr_driver_steps_csv(d, csv, len + 1, &len);
    fwrite(csv, 1, len, stdout);
    fprintf(stderr, "%llu steps, %llu tokens emitted\n", (unsigned long long)done, (unsigned long long)emitted);
    free(csv);
    kvr_driver_destroy(d);
    free(cfg);
    return 0;
}
