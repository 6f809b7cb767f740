// C-ABI plumbing: thread-local error string, version.
#include <stdarg.h>
#include <stdio.h>

#include "common.cuh"

namespace srlu {
static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}
}  // namespace srlu

extern "C" const char *srlu_last_error(void) { return srlu::g_err; }

extern "C" int srlu_version(void) { return 1; }
