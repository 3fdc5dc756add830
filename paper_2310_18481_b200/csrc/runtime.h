// Error plumbing shared by the C-ABI entry points.
#pragma once
#include <cuda_runtime.h>

#include "mosel_b200.h"

namespace mosel {
int set_error(int code, const char* msg);
int check_launch(const char* what);
}  // namespace mosel
