// C++ side of the drop-in executor (paper_2307_05740_b200/csrc/shim/
// executor_b200.cpp). The spttn:: API itself is declared by the reference
// header proj/include/spttn/executor.hpp; this header only adds the
// introspection hook the parity tests use.
#pragma once

#include "spttn/executor.hpp"

// SPTTN_NEST_* kind the plan runs on the device (SPTTN_NEST_GENERIC = the
// device forest interpreter).
int spttn_b200_plan_device_kind(const spttn::ExecPlan& plan);
