// Feasibility + cost check: an IF conditional graph node, set by a kernel,
// whose body is a cooperative kernel, captured from streams, followed by a
// kernel launched with programmatic stream serialization -- against the same
// chain with the cooperative kernel always launched, and without it.
//   nvcc -gencode arch=compute_100a,code=sm_100a -o cond_graph cond_graph.cu
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
    printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); return 1; } } while (0)

__global__ void k_set(cudaGraphConditionalHandle h, int use, const int* flag, int* log) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0 && blockIdx.x == 0) {
        if (use) cudaGraphSetConditional(h, *flag ? 1u : 0u);
        atomicAdd(&log[0], 1);
    }
}
__global__ void k_coop(int* log) {
    atomicAdd(&log[1], 1);
    cooperative_groups::this_grid().sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(&log[2], 1);
}
__global__ void k_after(int* log) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;");
    if (threadIdx.x == 0 && blockIdx.x == 0) atomicAdd(&log[3], 1);
}

static cudaError_t launch(void* k, dim3 g, dim3 b, cudaStream_t s, bool pdl, bool coop, void** args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = g; cfg.blockDim = b; cfg.stream = s;
    cudaLaunchAttribute at[1];
    if (coop) { at[0].id = cudaLaunchAttributeCooperative; at[0].val.cooperative = 1; }
    else { at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
           at[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0; }
    cfg.attrs = at; cfg.numAttrs = 1;
    return cudaLaunchKernelExC(&cfg, k, args);
}

// mode 0: conditional body; 1: cooperative kernel always; 2: no cooperative kernel
int build(int mode, cudaStream_t s, cudaStream_t a, int* flag, int* log, cudaGraphExec_t* ex) {
    CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
    for (int step = 0; step < 16; ++step) {
        cudaStreamCaptureStatus st; cudaGraph_t g; const cudaGraphNode_t* deps; size_t nd;
        cudaGraphConditionalHandle h = 0;
        int use = mode == 0;
        if (use) {
            CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
            CK(cudaGraphConditionalHandleCreate(&h, g, 0, cudaGraphCondAssignDefault));
        }
        void* a1[] = {&h, &use, &flag, &log};
        CK(launch((void*)k_set, dim3(4), dim3(256), s, true, false, a1));
        void* a2[] = {&log};
        if (mode == 0) {
            CK(cudaStreamGetCaptureInfo(s, &st, nullptr, &g, &deps, &nd));
            cudaGraphNodeParams cp = {};
            cp.type = cudaGraphNodeTypeConditional;
            cp.conditional.handle = h;
            cp.conditional.type = cudaGraphCondTypeIf;
            cp.conditional.size = 1;
            cudaGraphNode_t cn;
            CK(cudaGraphAddNode(&cn, g, deps, nd, &cp));
            CK(cudaStreamBeginCaptureToGraph(a, cp.conditional.phGraph_out[0], nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal));
            CK(launch((void*)k_coop, dim3(148), dim3(256), a, false, true, a2));
            CK(cudaStreamEndCapture(a, nullptr));
            CK(cudaStreamUpdateCaptureDependencies(s, &cn, 1, cudaStreamSetCaptureDependencies));
        } else if (mode == 1) {
            CK(launch((void*)k_coop, dim3(148), dim3(256), s, false, true, a2));
        }
        CK(launch((void*)k_after, dim3(148), dim3(256), s, true, false, a2));
        CK(launch((void*)k_after, dim3(148), dim3(256), s, true, false, a2));
    }
    cudaGraph_t graph;
    CK(cudaStreamEndCapture(s, &graph));
    CK(cudaGraphInstantiate(ex, graph, 0));
    return 0;
}

int main() {
    cudaStream_t s, a;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&a, cudaStreamNonBlocking));
    int *flag, *log;
    CK(cudaMalloc(&flag, 4));
    CK(cudaMalloc(&log, 16));
    const char* names[3] = {"conditional cooperative", "cooperative always", "no cooperative"};
    for (int mode = 0; mode < 3; ++mode) {
        cudaGraphExec_t ex;
        if (build(mode, s, a, flag, log, &ex)) return 1;
        for (int f = 0; f < 2; ++f) {
            CK(cudaMemcpy(flag, &f, 4, cudaMemcpyHostToDevice));
            CK(cudaMemset(log, 0, 16));
            CK(cudaGraphLaunch(ex, s));
            CK(cudaStreamSynchronize(s));
            int hl[4];
            CK(cudaMemcpy(hl, log, 16, cudaMemcpyDeviceToHost));
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0); cudaEventCreate(&e1);
            cudaEventRecord(e0, s);
            for (int i = 0; i < 200; ++i) CK(cudaGraphLaunch(ex, s));
            cudaEventRecord(e1, s);
            CK(cudaStreamSynchronize(s));
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            printf("%-24s flag %d: set %d coop-done %d after %d | %.2f us/step\n", names[mode], f,
                   hl[0], hl[2], hl[3], ms * 1000.f / (200 * 16));
        }
    }
    return 0;
}
