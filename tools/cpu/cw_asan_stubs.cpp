#include <cstdarg>
#include <cstddef>
#include <cstdio>
namespace scout_host { void set_error(int, const char* fmt, ...) { va_list a; va_start(a, fmt); vfprintf(stderr, fmt, a); va_end(a); } }
extern "C" size_t scout_slot_bytes(int dt) { return dt == 1 ? 32768 : (dt == 0 ? 65536 : 0); }
extern "C" const char* scout_last_error(void) { return ""; }
