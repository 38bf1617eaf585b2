// Drop-in shim for <batchsim/workload.hpp> (inc/workload.hpp: WorkloadSpec, generate_arrivals):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/arrivals.hpp"
