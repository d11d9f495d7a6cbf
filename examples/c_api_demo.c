/* c_api_demo.c — the C ABI without Python: one predator-prey grid search
 * (cfg1: 3 x 3 x 3 attention levels, 10 samples) through include/distill.h.
 *
 *   gcc -O2 -I include examples/c_api_demo.c -L paper_2110_15425_b200 -ldistill \
 *       -L /usr/local/cuda/lib64 -lcudart -Wl,-rpath,paper_2110_15425_b200 -o c_api_demo
 *   ./c_api_demo          # prints the 27 net values, the host-buffer calls' keys and the best allocation
 *
 * Device buffers come from the CUDA runtime; the library only owns the model. */
#include <stdio.h>
#include <stdint.h>
#include <cuda_runtime_api.h>
#include "distill.h"

#define CHECK(call)                                                                  \
    do {                                                                             \
        distill_status s_ = (call);                                                  \
        if (s_ != DISTILL_OK) {                                                      \
            fprintf(stderr, "%s failed: %d (%s)\n", #call, (int)s_, distill_last_error()); \
            return 1;                                                                \
        }                                                                            \
    } while (0)

int main(void) {
    const uint32_t n_levels[3] = {3, 3, 3};
    const float levels[9] = {0.0f, 0.5f, 1.0f, 0.0f, 0.5f, 1.0f, 0.0f, 0.5f, 1.0f};
    const float w[3] = {0.1f, 0.1f, 0.1f};
    const float params[3] = {2.0f, 0.1f, 0.5f};           /* sigma_max, sigma_min, kappa */
    const float inputs[6] = {4.0f, 1.0f, -3.0f, 2.0f, 0.0f, 0.0f};   /* prey, predator, player */
    distill_model_desc desc = {DISTILL_MODEL_PREDATOR_PREY, 3, n_levels, levels, w, params, 3};
    distill_model* m = NULL;
    CHECK(distill_load_model(&desc, 0, &m));
    uint64_t n = 0;
    CHECK(distill_grid_size(m, &n));

    float* d_net = NULL;
    unsigned long long* d_best = NULL;
    if (cudaMalloc((void**)&d_net, n * sizeof(float)) != cudaSuccess ||
        cudaMalloc((void**)&d_best, sizeof(unsigned long long)) != cudaSuccess) {
        fprintf(stderr, "cudaMalloc failed\n");
        return 1;
    }
    CHECK(distill_key_reset(d_best, NULL));
    distill_eval_args a = {0};
    a.inputs = inputs; a.n_inputs = 6; a.begin = 0; a.end = n;
    a.n_samples = 10; a.invocation = 0; a.seed = 42;
    a.d_net = d_net; a.d_best = d_best;
    CHECK(distill_eval_grid(m, &a, NULL));

    float net[27];
    unsigned long long key = 0;
    cudaMemcpy(net, d_net, n * sizeof(float), cudaMemcpyDeviceToHost);
    cudaMemcpy(&key, d_best, sizeof key, cudaMemcpyDeviceToHost);
    float cost = 0.0f;
    uint64_t idx = 0;
    CHECK(distill_key_decode(key, &cost, &idx));
    for (uint64_t i = 0; i < n; ++i) printf("%llu %a\n", (unsigned long long)i, -net[i]);

    /* The same search from host buffers: the synchronous end-to-end call, then two
     * calls in flight at once on two pinned slots (distill_eval_grid_host_async,
     * results valid once the stream has passed them). */
    float* h_net[2] = {NULL, NULL};
    unsigned long long* h_key[2] = {NULL, NULL};
    for (int q = 0; q < 2; ++q)
        if (cudaHostAlloc((void**)&h_net[q], n * sizeof(float), cudaHostAllocMapped) != cudaSuccess ||
            cudaHostAlloc((void**)&h_key[q], sizeof(unsigned long long), cudaHostAllocMapped) != cudaSuccess) {
            fprintf(stderr, "cudaHostAlloc failed\n");
            return 1;
        }
    unsigned long long key_sync = 0;
    CHECK(distill_eval_grid_host(m, inputs, 6, 0, n, 10, 0, 42, h_net[0], &key_sync, NULL));
    CHECK(distill_eval_grid_host_async(m, inputs, 6, 0, n, 10, 0, 42, h_net[0], h_key[0], NULL));
    CHECK(distill_eval_grid_host_async(m, inputs, 6, 0, n, 10, 0, 42, h_net[1], h_key[1], NULL));
    if (cudaStreamSynchronize(NULL) != cudaSuccess) { fprintf(stderr, "sync failed\n"); return 1; }
    int same = 1;
    for (uint64_t i = 0; i < n; ++i) same &= (h_net[0][i] == net[i]) & (h_net[1][i] == net[i]);
    printf("host key 0x%016llx async 0x%016llx 0x%016llx nets %s\n", key_sync, *h_key[0], *h_key[1],
           same ? "same" : "DIFFER");
    for (int q = 0; q < 2; ++q) { cudaFreeHost(h_net[q]); cudaFreeHost(h_key[q]); }

    printf("best %llu cost %a key 0x%016llx\n", (unsigned long long)idx, cost, key);
    cudaFree(d_net);
    cudaFree(d_best);
    distill_free_model(m);
    return 0;
}
