// C ABI entry points that are not tied to one kernel family.
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

}  // extern "C"
