// Internal helpers shared by the C-ABI translation units.
#pragma once
#include "ddit.h"
#include "gemm_sm100.cuh"

namespace ddit {
void set_error(const char* fmt, ...);
int check_cuda(const char* what);
EpiParams to_epi(const ddit_epi* e);
}  // namespace ddit
