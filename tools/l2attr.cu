// prints the L2 persistence limits of device 0 (profiling aid)
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    int l2 = 0, maxp = 0, maxw = 0;
    cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, 0);
    cudaDeviceGetAttribute(&maxp, cudaDevAttrMaxPersistingL2CacheSize, 0);
    cudaDeviceGetAttribute(&maxw, cudaDevAttrMaxAccessPolicyWindowSize, 0);
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    printf("{\"l2_bytes\": %d, \"max_persisting_l2\": %d, \"max_access_policy_window\": %d, \"persisting_limit_now\": %zu}\n",
           l2, maxp, maxw, cur);
    return 0;
}
