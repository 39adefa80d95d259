// C ABI plumbing: thread-local error text, launch checks, layout probes.
#include <cstdarg>
#include <cstdio>
#include "cc_common.cuh"

static thread_local char g_err[1024] = "";

extern "C" int cc_set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return -1;
}

extern "C" int cc_check_launch(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess)
        return cc_set_error("%s: %s (%s)", what, cudaGetErrorString(e), cudaGetErrorName(e));
    return 0;
}

extern "C" const char* cc_last_error(void) { return g_err; }
extern "C" int cc_abi_version(void) { return CC_ABI_VERSION; }
extern "C" int64_t cc_sizeof_shard(void) { return (int64_t)sizeof(cc_shard); }
extern "C" int64_t cc_sizeof_ctl(void) { return (int64_t)sizeof(cc_ctl); }
extern "C" int64_t cc_sizeof_gen(void) { return (int64_t)sizeof(cc_gen); }
