// Test tool (CPU-only): runs NVIDIA's own curand_Philox4x32_10 from
// <curand_philox4x32_x.h> on the HOST to pin the oracle's Philox4x32-10.
// Counter i -> (i, i*2654435761, i%40, i*40503); keys from argv.
#define QUALIFIERS static inline __host__ __device__
#include <curand_philox4x32_x.h>
#include <cstdio>
#include <cstdlib>
int main(int argc, char **argv) {
    unsigned long long n = strtoull(argv[1], 0, 10);
    uint2 key = make_uint2((unsigned)strtoul(argv[2], 0, 0), (unsigned)strtoul(argv[3], 0, 0));
    FILE *f = fopen(argv[4], "wb");
    for (unsigned long long i = 0; i < n; i++) {
        unsigned u = (unsigned)i;
        uint4 c = make_uint4(u, u * 2654435761u, u % 40u, u * 40503u);
        uint4 r = curand_Philox4x32_10(c, key);
        fwrite(&r, 16, 1, f);
    }
    fclose(f);
    return 0;
}
