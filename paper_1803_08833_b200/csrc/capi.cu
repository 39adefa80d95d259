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

// ---------------------------------------------------------------- timers
// CUDA events recorded with cudaEventRecordExternal so that they also work as
// event-record nodes inside captured CUDA graphs (per-kernel timing of graph
// replays).
struct cc_timer { int n; cudaEvent_t* ev; };

extern "C" int cc_timer_create(int32_t n, void** handle) {
    if (n <= 0 || !handle) return cc_set_error("cc_timer_create: bad arguments");
    cc_timer* t = new cc_timer;
    t->n = n;
    t->ev = new cudaEvent_t[n];
    for (int i = 0; i < n; ++i) {
        const cudaError_t e = cudaEventCreate(&t->ev[i]);
        if (e != cudaSuccess) return cc_set_error("cudaEventCreate: %s", cudaGetErrorString(e));
    }
    *handle = t;
    return 0;
}

extern "C" int cc_timer_record(void* handle, int32_t i, void* stream) {
    cc_timer* t = static_cast<cc_timer*>(handle);
    if (!t || i < 0 || i >= t->n) return cc_set_error("cc_timer_record: bad index");
    const cudaError_t e = cudaEventRecordWithFlags(t->ev[i], (cudaStream_t)stream,
                                                   cudaEventRecordExternal);
    if (e != cudaSuccess) return cc_set_error("cudaEventRecordWithFlags: %s", cudaGetErrorString(e));
    return 0;
}

extern "C" float cc_timer_elapsed_ms(void* handle, int32_t i, int32_t j) {
    cc_timer* t = static_cast<cc_timer*>(handle);
    if (!t || i < 0 || j < 0 || i >= t->n || j >= t->n) return -1.0f;
    float ms = -1.0f;
    if (cudaEventElapsedTime(&ms, t->ev[i], t->ev[j]) != cudaSuccess) return -1.0f;
    return ms;
}

extern "C" int cc_timer_destroy(void* handle) {
    cc_timer* t = static_cast<cc_timer*>(handle);
    if (!t) return 0;
    for (int i = 0; i < t->n; ++i) cudaEventDestroy(t->ev[i]);
    delete[] t->ev;
    delete t;
    return 0;
}
