// Drop-in shim for <batchsim/dp_time.hpp> (inc/dp_time.hpp: build_units, compute_schedule(_dp), DpTable, baselines):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/schedulers.hpp"
