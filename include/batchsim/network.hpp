// Drop-in shim for <batchsim/network.hpp> (inc/network.hpp: NetworkTrace, transmission_delay):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/arrivals.hpp"
