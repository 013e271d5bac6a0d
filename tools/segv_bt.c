/* Development aid: prints a native backtrace on SIGSEGV (segv_install() after the runtime's own
 * handlers are in place, or LD_PRELOAD for the constructor). */
#include <execinfo.h>
#include <signal.h>
#include <string.h>
#include <unistd.h>
static void handler(int sig, siginfo_t *si, void *ctx) {
  (void)ctx;
  void *b[64];
  char msg[64];
  int n = backtrace(b, 64);
  int l = 0;
  const char *h = "SIGSEGV at ";
  write(2, h, strlen(h));
  unsigned long a = (unsigned long)si->si_addr;
  for (int i = 60; i >= 0; i -= 4) msg[l++] = "0123456789abcdef"[(a >> i) & 15];
  msg[l++] = '\n';
  write(2, msg, l);
  backtrace_symbols_fd(b, n, 2);
  _exit(128 + sig);
}
void segv_install(void) {
  struct sigaction sa;
  memset(&sa, 0, sizeof(sa));
  sa.sa_sigaction = handler;
  sa.sa_flags = SA_SIGINFO;
  sigaction(SIGSEGV, &sa, 0);
}
__attribute__((constructor)) static void install(void) { segv_install(); }
