#include <cuda_runtime.h>
#include <cstdio>
__global__ void body(int *ctr, cudaGraphConditionalHandle h) {
    int v = atomicAdd(ctr, 1) + 1;
    cudaGraphSetConditional(h, v < 10 ? 1 : 0);
}
int main() {
    cudaGraph_t g; cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t n;
    cudaGraphAddNode(&n, g, nullptr, 0, &p);
    cudaGraph_t bodyg = p.conditional.phGraph_out[0];
    int *ctr; cudaMalloc(&ctr, 4); cudaMemset(ctr, 0, 4);
    cudaKernelNodeParams kp = {};
    void *args[] = {&ctr, &h};
    kp.func = (void*)body; kp.gridDim = dim3(1); kp.blockDim = dim3(1); kp.kernelParams = args;
    cudaGraphNode_t kn; cudaGraphAddKernelNode(&kn, bodyg, nullptr, 0, &kp);
    cudaGraphExec_t ge; cudaError_t e = cudaGraphInstantiate(&ge, g, 0);
    printf("inst %s\n", cudaGetErrorString(e));
    cudaGraphLaunch(ge, 0); cudaDeviceSynchronize();
    int v; cudaMemcpy(&v, ctr, 4, cudaMemcpyDeviceToHost); printf("ctr=%d\n", v);
}
