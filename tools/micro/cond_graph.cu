// Minimal conditional-WHILE CUDA graph (the structure dd_bicgstab uses),
// built and launched for two "contexts" in sequence: a probe for running
// compute-sanitizer on conditional graph bodies. Prints the loop counts.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void body(int *ctl, double *v, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) v[i] += 1.0;
}
__global__ void head(int *ctl) { ctl[0] += 1; }
__global__ void tail(int *ctl, cudaGraphConditionalHandle h) { cudaGraphSetConditional(h, ctl[0] < ctl[1] ? 1u : 0u); }

struct Held {
    cudaGraphExec_t ge;
    cudaGraph_t g;
    cudaStream_t st, cap;
    int *ctl;
    double *v;
};
static Held held[4];
static int nheld = 0;
static bool keep = false;

static int run(int n, int iters) {
    int *ctl;
    double *v;
    cudaMalloc(&ctl, 2 * sizeof(int));
    cudaMalloc(&v, n * sizeof(double));
    cudaMemset(v, 0, n * sizeof(double));
    int h_ctl[2] = {0, iters};
    cudaMemcpy(ctl, h_ctl, sizeof h_ctl, cudaMemcpyHostToDevice);
    cudaStream_t st, cap;
    cudaStreamCreate(&st);
    cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking);
    cudaGraph_t g;
    cudaGraphCreate(&g, 0);
    cudaGraphConditionalHandle h;
    cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault);
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h;
    p.conditional.type = cudaGraphCondTypeWhile;
    p.conditional.size = 1;
    cudaGraphNode_t node;
    cudaGraphAddNode(&node, g, nullptr, 0, &p);
    cudaStreamBeginCaptureToGraph(cap, p.conditional.phGraph_out[0], nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed);
    head<<<1, 1, 0, cap>>>(ctl);
    body<<<64, 256, 0, cap>>>(ctl, v, n);
    tail<<<1, 1, 0, cap>>>(ctl, h);
    cudaGraph_t out;
    cudaStreamEndCapture(cap, &out);
    cudaGraphExec_t ge;
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, st);
    cudaError_t e = cudaStreamSynchronize(st);
    double v0 = 0;
    cudaMemcpy(&v0, v, sizeof(double), cudaMemcpyDeviceToHost);
    printf("n=%d iters=%d v[0]=%g status=%s\n", n, iters, v0, cudaGetErrorString(e));
    if (keep) {  // the first "context" stays alive while the next ones run
        held[nheld++] = Held{ge, g, st, cap, ctl, v};
        return e == cudaSuccess ? 0 : 1;
    }
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
    cudaStreamDestroy(cap);
    cudaStreamDestroy(st);
    cudaFree(ctl);
    cudaFree(v);
    return e == cudaSuccess ? 0 : 1;
}

int main(int argc, char **argv) {
    keep = argc > 1 && argv[1][0] == 'k';
    int rc = run(2880, 5);
    rc |= run(3000, 6);
    rc |= run(3000, 6);
    return rc;
}
