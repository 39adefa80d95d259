// C ABI plumbing: thread-local error text, launch checks, layout probes.
#include <cstdarg>
#include <cstdio>
#include <cstring>
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
extern "C" int64_t cc_sizeof_xpeer(void) { return (int64_t)sizeof(cc_xpeer); }

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

// ------------------------------------------------- peer-exchange windows
// One cudaMalloc per window (an IPC handle names a whole allocation), zeroed
// so that every flag word starts at epoch 0.
extern "C" int cc_xwin_alloc(int64_t bytes, void** ptr, uint8_t* handle64) {
    if (bytes <= 0 || !ptr || !handle64) return cc_set_error("cc_xwin_alloc: bad arguments");
    void* p = nullptr;
    cudaError_t e = cudaMalloc(&p, (size_t)bytes);
    if (e != cudaSuccess) return cc_set_error("cc_xwin_alloc: cudaMalloc: %s", cudaGetErrorString(e));
    e = cudaMemset(p, 0, (size_t)bytes);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaIpcMemHandle_t h;
    if (e == cudaSuccess) e = cudaIpcGetMemHandle(&h, p);
    if (e != cudaSuccess) {
        cudaFree(p);
        return cc_set_error("cc_xwin_alloc: %s", cudaGetErrorString(e));
    }
    static_assert(sizeof(h) == 64, "CUDA IPC handle is 64 bytes");
    memcpy(handle64, &h, 64);
    *ptr = p;
    return 0;
}

extern "C" int cc_xwin_open(const uint8_t* handle64, void** ptr) {
    if (!handle64 || !ptr) return cc_set_error("cc_xwin_open: bad arguments");
    cudaIpcMemHandle_t h;
    memcpy(&h, handle64, 64);
    void* p = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) return cc_set_error("cc_xwin_open: %s", cudaGetErrorString(e));
    *ptr = p;
    return 0;
}

extern "C" int cc_xwin_close(void* ptr) {
    if (!ptr) return 0;
    const cudaError_t e = cudaIpcCloseMemHandle(ptr);
    if (e != cudaSuccess) return cc_set_error("cc_xwin_close: %s", cudaGetErrorString(e));
    return 0;
}

extern "C" int cc_xwin_free(void* ptr) {
    if (!ptr) return 0;
    const cudaError_t e = cudaFree(ptr);
    if (e != cudaSuccess) return cc_set_error("cc_xwin_free: %s", cudaGetErrorString(e));
    return 0;
}
