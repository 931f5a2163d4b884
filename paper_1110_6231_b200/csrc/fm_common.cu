// fm_common.cu -- error reporting and device queries for the C ABI.
#include <stdarg.h>
#include <stdio.h>

#include "fm_common.cuh"

static thread_local char g_fm_error[1024] = "";

void fm_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_fm_error, sizeof(g_fm_error), fmt, ap);
    va_end(ap);
}

extern "C" const char *fm_last_error(void) { return g_fm_error; }

extern "C" int fm_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

extern "C" const char *fm_version(void) { return "flowmatch_b200 0.1.0 sm_100a"; }
