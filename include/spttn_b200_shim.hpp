// C++ side of the drop-in executor (paper_2307_05740_b200/csrc/shim/
// executor_b200.cpp). The spttn:: API itself is declared by the reference
// header proj/include/spttn/executor.hpp; this header only adds the
// introspection hook the parity tests use.
#pragma once

#include <string>
#include <vector>

#include "spttn/executor.hpp"
#include "spttn/tensor.hpp"

// SPTTN_NEST_* kind the plan runs on the device (SPTTN_NEST_GENERIC = the
// device forest interpreter).
int spttn_b200_plan_device_kind(const spttn::ExecPlan& plan);

// spttn_plan_info (include/spttn_b200.h) of the device plan behind `plan`:
// launches, work items, ..., [8] interpreter decomposition, [9] JIT flag.
int spttn_b200_plan_info(const spttn::ExecPlan& plan, int64_t* out, int n);

// CooTensor::normalize + build_csf (proj/src/tensor.cpp:24-94) on the GPU:
// the same CsfTensor (duplicates summed in input order), ~1000x faster than
// the host build at 1e7 nonzeros. Throws std::invalid_argument like the
// reference for a bad mode order or out-of-range coordinates.
spttn::CsfTensor spttn_b200_build_csf(const spttn::CooTensor& coo,
                                      const std::vector<std::string>& mode_order);
