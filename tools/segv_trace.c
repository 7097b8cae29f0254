/* Debug aid (LD_PRELOAD): print a backtrace on SIGSEGV/SIGABRT, e.g.
 *   gcc -shared -fPIC -o /tmp/segv.so tools/segv_trace.c
 *   LD_PRELOAD=/tmp/segv.so python ... */
#define _GNU_SOURCE
#include <execinfo.h>
#include <signal.h>
#include <stdio.h>
#include <string.h>
#include <unistd.h>
#include <dlfcn.h>

static void on_fault(int sig) {
    void* pcs[64];
    const int n = backtrace(pcs, 64);
    char head[64];
    const int len = snprintf(head, sizeof head, "\n[segv_trace] signal %d, %d frames\n", sig, n);
    write(2, head, (size_t)len);
    for (int i = 0; i < n; ++i) {
        Dl_info di;
        char line[512];
        if (dladdr(pcs[i], &di) && di.dli_fname) {
            const long off = (long)((char*)pcs[i] - (char*)di.dli_fbase);
            const int m = snprintf(line, sizeof line, "  #%d %s+0x%lx (%s)\n", i, di.dli_fname, off,
                                   di.dli_sname ? di.dli_sname : "?");
            write(2, line, (size_t)m);
        }
    }
    signal(sig, SIG_DFL);
    raise(sig);
}

__attribute__((constructor)) static void install(void) {
    signal(SIGSEGV, on_fault);
    signal(SIGABRT, on_fault);
}
