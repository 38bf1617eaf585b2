// Drop-in shim for <batchsim/model.hpp> (inc/model.hpp: Request, arrives_before, outcomes):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/core.hpp"
