// C ABI entry points that are not tied to one kernel family.
#include <cstring>

#include "mcf_internal.cuh"

namespace mcf {
const char *last_error();
long long launches();
}

extern "C" {

const char *mcf_version(void) { return "mcfunm_cuda 0.1.0 (sm_100a)"; }

const char *mcf_last_error(void) { return mcf::last_error(); }

int64_t mcf_kernel_launches(void) { return (int64_t)mcf::launches(); }

static double drain(std::vector<std::pair<cudaEvent_t, cudaEvent_t>> &v, int64_t *count, bool reset, int *rc) {
    double ms = 0.0;
    for (auto &p : v) {
        float t = 0.f;
        cudaError_t e = cudaEventSynchronize(p.second);
        if (e == cudaSuccess) e = cudaEventElapsedTime(&t, p.first, p.second);
        if (e != cudaSuccess) {
            *rc = mcf::cuda_status(e, "kernel timing events");
            cudaGetLastError();  // do not leave the error for later calls
        }
        ms += t;
        if (reset) {
            cudaEventDestroy(p.first);
            cudaEventDestroy(p.second);
        }
    }
    if (count) *count = (int64_t)v.size();
    if (reset) v.clear();
    return ms;
}

int mcf_graph_kernel_times(mcf_graph *g, double *walk_ms, double *q_ms, int64_t *walk_launches, int reset) {
    if (!g) {
        mcf::set_error("mcf_graph_kernel_times: null graph");
        return MCF_ERR_ARGUMENT;
    }
    int rc = MCF_OK;
    double w = drain(g->ev_walk, walk_launches, reset != 0, &rc);
    double q = drain(g->ev_q, nullptr, reset != 0, &rc);
    if (walk_ms) *walk_ms = w;
    if (q_ms) *q_ms = q;
    return rc;
}

// ---------------------------------------------------------------------------
// Peer buffers for the multi-GPU exchange (one process per GPU, one node):
// plain cudaMalloc allocations whose CUDA IPC handles the ranks swap (through
// torch.distributed), so mcf_spmv_peer can read q from, and write y into,
// the other ranks' memory over NVLink.
// ---------------------------------------------------------------------------
int mcf_peer_alloc(int64_t bytes, void **ptr, void *ipc_handle) {
    if (!ptr || !ipc_handle || bytes <= 0) {
        mcf::set_error("mcf_peer_alloc: bad argument");
        return MCF_ERR_ARGUMENT;
    }
    cudaError_t e = cudaMalloc(ptr, (size_t)bytes);
    if (e == cudaSuccess) e = cudaMemset(*ptr, 0, (size_t)bytes);
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(reinterpret_cast<cudaIpcMemHandle_t *>(ipc_handle), *ptr);
    if (e != cudaSuccess) return mcf::cuda_status(e, "mcf_peer_alloc");
    return MCF_OK;
}

int mcf_peer_open(const void *ipc_handle, void **ptr) {
    if (!ptr || !ipc_handle) {
        mcf::set_error("mcf_peer_open: bad argument");
        return MCF_ERR_ARGUMENT;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, ipc_handle, sizeof(h));
    cudaError_t e = cudaIpcOpenMemHandle(ptr, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return mcf::cuda_status(e, "mcf_peer_open");
    return MCF_OK;
}

int mcf_peer_close(void *ptr) {
    cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) return mcf::cuda_status(e, "mcf_peer_close");
    return MCF_OK;
}

int mcf_peer_free(void *ptr) {
    cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return mcf::cuda_status(e, "mcf_peer_free");
    return MCF_OK;
}

}  // extern "C"
