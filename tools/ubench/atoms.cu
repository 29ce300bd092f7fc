// Microbenchmark: shared-memory atomics vs plain shared RMW throughput on this GPU.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 atoms.cu -o atoms && ./atoms
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void k(unsigned *out, int iters) {
    __shared__ unsigned t[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) t[i] = 0;
    __syncthreads();
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    unsigned acc = 0;
    for (int it = 0; it < iters; it++) {
        x = x * 1664525u + 1013904223u;
        const unsigned a = (x >> 20) & 4095;   // spread addresses
        if (MODE == 0) atomicAdd(&t[a], 1u);                     // RED.shared
        else if (MODE == 1) acc += atomicAdd(&t[a], 1u);         // ATOMS with return
        else if (MODE == 2) acc += atomicCAS(&t[a], 0u, x);      // CAS
        else if (MODE == 3) { volatile unsigned *v = t; acc += v[a]; }   // LDS
        else if (MODE == 4) { t[a] = x; }                        // STS
        else if (MODE == 5) { atomicAdd(&t[threadIdx.x & 4095], 1u); }   // lane-distinct banks
        else if (MODE == 6) { atomicAdd(&t[7], 1u); }                    // one address, every lane
        else if (MODE == 7) { atomicAdd(&t[(x >> 29) == 0 ? 7u : a], 1u); }   // 1/8 of the lanes on one address
        else if (MODE == 8) { atomicAdd(&t[(x >> 28) == 0 ? 7u : a], 1u); }   // 1/16 ...
        else if (MODE == 9) {   // skewed like the sweep: 43% of the adds on 64 addresses
            const unsigned b = (x >> 8) & 63;
            atomicAdd(&t[(x & 127) < 55 ? b * 61u : a], 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = t[blockIdx.x & 4095] + acc;
}

int main() {
    unsigned *o;
    cudaMalloc(&o, 1 << 20);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int iters = 4096, blocks = sms * 8, threads = 256;
    const char *names[] = {"RED.shared add (spread)", "ATOMS add w/ return (spread)", "ATOMS CAS (spread)",
                           "LDS volatile (spread)", "STS (spread)", "RED.shared add (lane-distinct)",
                           "RED.shared add (one address)", "RED.shared add (1/8 on one address)",
                           "RED.shared add (1/16 on one address)", "RED.shared add (43% on 64 addresses)"};
    for (int mode = 0; mode < 10; mode++) {
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int rep = 0; rep < 2; rep++) {
            cudaEventRecord(a);
            switch (mode) {
                case 0: k<0><<<blocks, threads>>>(o, iters); break;
                case 1: k<1><<<blocks, threads>>>(o, iters); break;
                case 2: k<2><<<blocks, threads>>>(o, iters); break;
                case 3: k<3><<<blocks, threads>>>(o, iters); break;
                case 4: k<4><<<blocks, threads>>>(o, iters); break;
                case 5: k<5><<<blocks, threads>>>(o, iters); break;
                case 6: k<6><<<blocks, threads>>>(o, iters); break;
                case 7: k<7><<<blocks, threads>>>(o, iters); break;
                case 8: k<8><<<blocks, threads>>>(o, iters); break;
                case 9: k<9><<<blocks, threads>>>(o, iters); break;
            }
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double ops = (double)blocks * threads * iters;
        printf("%-34s %8.2f Gops/s  %6.3f ops/clk/SM (at 1.965 GHz)\n", names[mode], ops / ms / 1e6,
               ops / (ms * 1e-3) / 1.965e9 / sms);
    }
    return 0;
}
