// Drop-in shim for <batchsim/deadline.hpp> (inc/deadline.hpp: drop_expired, edf_batch, tardy_dp):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/schedulers.hpp"
