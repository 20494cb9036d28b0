// Error reporting and device queries for the C ABI (include/probegrid_b200.h).
#include "pg_common.cuh"

namespace pg {

static thread_local std::string g_last_error;

void set_error(const std::string &msg) { g_last_error = msg; }

int check_launch(const char *what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        g_last_error = std::string(what) + ": " + cudaGetErrorString(e);
        return PG_ERR_CUDA;
    }
    return PG_OK;
}

}  // namespace pg

extern "C" {

const char *pg_last_error(void) { return pg::g_last_error.c_str(); }

const char *pg_version(void) { return "probegrid_b200 0.1 (sm_100a)"; }

int pg_device_sm_count(int device) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -1;
    return n;
}

}  // extern "C"
