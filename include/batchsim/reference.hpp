// Drop-in shim for <batchsim/reference.hpp> (inc/reference.hpp: brute-force oracles, random instances):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/selfcheck.hpp"
