/* A plain-C host of the C ABI (no CUDA headers, no torch): what a non-Python caller of
 * include/pipesched_b200.h looks like.  It reads one instance and a batch of candidate structures
 * from a file, evaluates them through both host-buffer entry points and writes the results.
 *
 *   ps_eval_batch_host        full structures (stage rows + offload masks)
 *   ps_eval_batch_host_delta  the same candidates as differences from candidate 0
 *
 * Build:  gcc -std=c99 -O2 -Wall -Wextra -Werror -I include examples/c_host.c \
 *             -L paper_2510_05186_b200/_lib -lpipesched_b200 -Wl,-rpath,<that dir> -o c_host
 * Run:    ./c_host in.bin out.bin
 *
 * in.bin (little endian): i32 P, m, G, post_validation; i64 comm_time, offload_time;
 *   i64 proc_time[P][m][3], mem_delta[P][m][3], act_size[P][m], mem_limit[P]; i32 stage_channel[P];
 *   i64 N; u16 orders[N][P][order_stride]; u32 masks[N][mask_words]
 *   (order_stride = 3m rounded up to 8, mask_words = ceil(P*m/32), as ps_instance_get_info reports)
 * out.bin: from the full batch i64 makespan[N], f64 bubble[N], u32 flags[N], u32 blocked[N],
 *   i64 peak[N][P]; then from the delta batch i64 makespan[N], f64 bubble[N], u32 flags[N].
 * Tests: tests/test_c_host.py (compiles it on CPU; runs it against the oracle on the GPU).
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "pipesched_b200.h"

static void *read_n(FILE *f, size_t elem, size_t n)
{
    void *p = malloc(elem * (n ? n : 1));
    if (!p || fread(p, elem, n, f) != n) {
        fprintf(stderr, "c_host: short input\n");
        exit(2);
    }
    return p;
}

static int check(int rc, const char *what)
{
    if (rc != PS_OK) {
        fprintf(stderr, "c_host: %s failed (%d): %s\n", what, rc, ps_last_error());
        exit(3);
    }
    return rc;
}

int main(int argc, char **argv)
{
    if (argc != 3) {
        fprintf(stderr, "usage: %s in.bin out.bin\n", argv[0]);
        return 1;
    }
    FILE *in = fopen(argv[1], "rb");
    if (!in) {
        perror(argv[1]);
        return 1;
    }
    int32_t *hdr = read_n(in, sizeof(int32_t), 4);
    int64_t *times = read_n(in, sizeof(int64_t), 2);
    const int32_t P = hdr[0], m = hdr[1];
    const size_t ops = (size_t)P * m * 3;
    ps_instance_desc desc;
    memset(&desc, 0, sizeof desc);
    desc.num_stages = P;
    desc.num_microbatches = m;
    desc.num_channels = hdr[2];
    desc.post_validation = hdr[3];
    desc.comm_time = times[0];
    desc.offload_time = times[1];
    desc.proc_time = read_n(in, sizeof(int64_t), ops);
    desc.mem_delta = read_n(in, sizeof(int64_t), ops);
    desc.act_size = read_n(in, sizeof(int64_t), (size_t)P * m);
    desc.mem_limit = read_n(in, sizeof(int64_t), (size_t)P);
    desc.stage_channel = read_n(in, sizeof(int32_t), (size_t)P);

    ps_instance *inst = NULL;
    check(ps_instance_create(&desc, 0, &inst), "ps_instance_create");
    ps_instance_info info;
    check(ps_instance_get_info(inst, &info), "ps_instance_get_info");

    int64_t *np = read_n(in, sizeof(int64_t), 1);
    const int64_t N = *np;
    const size_t row = (size_t)info.order_stride, mw = (size_t)info.mask_words;
    uint16_t *orders = read_n(in, sizeof(uint16_t), (size_t)N * P * row);
    uint32_t *masks = read_n(in, sizeof(uint32_t), (size_t)N * mw);
    fclose(in);

    /* Full structures. */
    int64_t *makespan = malloc(sizeof(int64_t) * N), *peak = malloc(sizeof(int64_t) * N * P);
    double *bubble = malloc(sizeof(double) * N);
    uint32_t *flags = malloc(sizeof(uint32_t) * N), *blocked = malloc(sizeof(uint32_t) * N);
    ps_cand_batch cb;
    memset(&cb, 0, sizeof cb);
    cb.num_candidates = N;
    cb.stage_orders = orders;
    cb.offload_mask = masks;
    cb.order_bytes = 2;
    ps_result_batch rb;
    memset(&rb, 0, sizeof rb);
    rb.makespan = makespan;
    rb.bubble = bubble;
    rb.peak = peak;
    rb.flags = flags;
    rb.blocked = blocked;
    check(ps_eval_batch_host(inst, &cb, &rb, NULL), "ps_eval_batch_host");

    /* The same candidates as differences from candidate 0: changed (stage, position) entries
       and flipped offload bits. */
    uint32_t *doff = malloc(sizeof(uint32_t) * (N + 1)), *foff = malloc(sizeof(uint32_t) * (N + 1));
    size_t ndiff = 0, nflip = 0, cap_d = 64, cap_f = 64;
    uint32_t *diffs = malloc(sizeof(uint32_t) * 2 * cap_d), *flips = malloc(sizeof(uint32_t) * cap_f);
    for (int64_t c = 0; c < N; ++c) {
        doff[c] = (uint32_t)ndiff;
        foff[c] = (uint32_t)nflip;
        const uint16_t *o = orders + (size_t)c * P * row;
        for (int32_t i = 0; i < P; ++i)
            for (size_t a = 0; a < row; ++a)
                if (o[i * row + a] != orders[i * row + a]) {
                    if (ndiff == cap_d)
                        diffs = realloc(diffs, sizeof(uint32_t) * 2 * (cap_d *= 2));
                    diffs[2 * ndiff] = ((uint32_t)i << 16) | (uint32_t)a;
                    diffs[2 * ndiff + 1] = o[i * row + a];
                    ++ndiff;
                }
        const uint32_t *k = masks + (size_t)c * mw;
        for (size_t b = 0; b < (size_t)P * m; ++b)
            if (((k[b >> 5] ^ masks[b >> 5]) >> (b & 31)) & 1u) {
                if (nflip == cap_f)
                    flips = realloc(flips, sizeof(uint32_t) * (cap_f *= 2));
                flips[nflip++] = (uint32_t)b;
            }
    }
    doff[N] = (uint32_t)ndiff;
    foff[N] = (uint32_t)nflip;
    int64_t *makespan_d = malloc(sizeof(int64_t) * N);
    double *bubble_d = malloc(sizeof(double) * N);
    uint32_t *flags_d = malloc(sizeof(uint32_t) * N);
    ps_delta_batch db;
    memset(&db, 0, sizeof db);
    db.num_candidates = N;
    db.ref_orders = orders;
    db.ref_mask = masks;
    db.diff_offset = doff;
    db.diffs = diffs;
    db.flip_offset = foff;
    db.flips = flips;
    ps_result_batch rd;
    memset(&rd, 0, sizeof rd);
    rd.makespan = makespan_d;
    rd.bubble = bubble_d;
    rd.flags = flags_d;
    check(ps_eval_batch_host_delta(inst, &db, &rd, NULL), "ps_eval_batch_host_delta");
    check(ps_instance_destroy(inst), "ps_instance_destroy");

    FILE *out = fopen(argv[2], "wb");
    if (!out) {
        perror(argv[2]);
        return 1;
    }
    fwrite(makespan, sizeof(int64_t), N, out);
    fwrite(bubble, sizeof(double), N, out);
    fwrite(flags, sizeof(uint32_t), N, out);
    fwrite(blocked, sizeof(uint32_t), N, out);
    fwrite(peak, sizeof(int64_t), (size_t)N * P, out);
    fwrite(makespan_d, sizeof(int64_t), N, out);
    fwrite(bubble_d, sizeof(double), N, out);
    fwrite(flags_d, sizeof(uint32_t), N, out);
    fclose(out);
    int64_t feasible = 0;
    for (int64_t c = 0; c < N; ++c)
        feasible += (flags[c] & PS_FLAG_FEASIBLE) != 0;
    printf("c_host: %s, %lld candidates, %lld feasible, %zu diffs, %zu flips\n", ps_version(),
           (long long)N, (long long)feasible, ndiff, nflip);
    return 0;
}
