// Drop-in shim for <batchsim/offload.hpp> (inc/offload.hpp: decide_binary, decide_partial, NetworkEstimator):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/arrivals.hpp"
