#include "bs_exec.h"
#include "errors.hpp"

extern "C" const char* bs_last_error(void) { return bs200::last_error_text().c_str(); }
