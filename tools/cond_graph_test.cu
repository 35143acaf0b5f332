// Which node kinds can a conditional (IF) body graph hold on this driver?
// Each case: [gate] -> IF { captured ops } ; instantiate, launch twice, check.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o /tmp/cgt tools/cond_graph_test.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

namespace cg = cooperative_groups;

__global__ void gate(cudaGraphConditionalHandle h, int v) { cudaGraphSetConditional(h, v); }
__global__ void plain(int* x) { atomicAdd(x, 1); }
__global__ void __cluster_dims__(1, 1, 1) clusterk(int* x) { atomicAdd(x, 1); }
__global__ void clusterdyn(int* x) {
    cg::this_cluster().sync();
    if (threadIdx.x == 0) atomicAdd(x, 1);
}
__global__ void coop(int* x) {
    cg::this_grid().sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(x, 1);
}

#define CK(x)                                                                   \
    do {                                                                        \
        cudaError_t e_ = (x);                                                   \
        if (e_ != cudaSuccess) {                                                \
            printf("  FAIL %s: %s\n", #x, cudaGetErrorString(e_));              \
            cudaGetLastError();                                                 \
            return false;                                                       \
        }                                                                       \
    } while (0)

template <typename F>
bool run_case(const char* name, cudaStream_t st, int* dx, F&& body, bool conditional) {
    printf("case %s (cond=%d)\n", name, conditional ? 1 : 0);
    fflush(stdout);
    cudaGraph_t g;
    CK(cudaGraphCreate(&g, 0));
    cudaGraph_t target = g;
    if (conditional) {
        cudaGraphConditionalHandle h;
        CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
        CK(cudaStreamBeginCaptureToGraph(st, g, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        gate<<<1, 1, 0, st>>>(h, 1);
        cudaGraph_t c;
        CK(cudaStreamEndCapture(st, &c));
        size_t nn = 0;
        CK(cudaGraphGetNodes(g, nullptr, &nn));
        std::vector<cudaGraphNode_t> nodes(nn);
        CK(cudaGraphGetNodes(g, nodes.data(), &nn));
        cudaGraphNodeParams cp{};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeIf;
        cp.conditional.size = 1;
        cudaGraphNode_t cn;
        CK(cudaGraphAddNode(&cn, g, nodes.data(), nn, &cp));
        target = cp.conditional.phGraph_out[0];
    }
    CK(cudaMemset(dx, 0, 4));
    CK(cudaStreamBeginCaptureToGraph(st, target, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
    body();
    cudaGraph_t c2;
    CK(cudaStreamEndCapture(st, &c2));
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, g, 0));
    CK(cudaGraphLaunch(ex, st));
    CK(cudaGraphLaunch(ex, st));
    CK(cudaStreamSynchronize(st));
    int h = -1;
    CK(cudaMemcpy(&h, dx, 4, cudaMemcpyDeviceToHost));
    printf("  ok: counter=%d\n", h);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
    return true;
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int* dx;
    cudaMalloc(&dx, 64);
    int* hp;
    cudaMallocHost(&hp, 64);
    *hp = 0;
    int* dy;
    cudaMalloc(&dy, 64);
    cudaFuncSetAttribute(clusterdyn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int cond = 0; cond < 2; ++cond) {
        run_case("plain kernel", st, dx, [&] { plain<<<1, 1, 0, st>>>(dx); }, cond);
        run_case("memset+memcpyD2D", st, dx, [&] {
            cudaMemsetAsync(dy, 0, 16, st);
            cudaMemcpyAsync(dy + 4, dy, 16, cudaMemcpyDeviceToDevice, st);
            plain<<<1, 1, 0, st>>>(dx);
        }, cond);
        run_case("memcpy pinned H2D", st, dx, [&] {
            cudaMemcpyAsync(dy, hp, 16, cudaMemcpyHostToDevice, st);
            plain<<<1, 1, 0, st>>>(dx);
        }, cond);
        run_case("cluster launchEx x16", st, dx, [&] {
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(16);
            cfg.blockDim = dim3(128);
            cfg.stream = st;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = 16;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            cfg.attrs = at;
            cfg.numAttrs = 1;
            cudaError_t e = cudaLaunchKernelEx(&cfg, clusterdyn, dx);
            if (e != cudaSuccess) printf("  launchEx: %s\n", cudaGetErrorString(e));
        }, cond);
        run_case("cooperative launch", st, dx, [&] {
            void* args[] = {&dx};
            cudaError_t e = cudaLaunchCooperativeKernel((void*)coop, dim3(148), dim3(128), args, 0, st);
            if (e != cudaSuccess) printf("  coop: %s\n", cudaGetErrorString(e));
        }, cond);
    }
    printf("done\n");
    return 0;
}
