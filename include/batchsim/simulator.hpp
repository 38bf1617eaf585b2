// Drop-in shim for <batchsim/simulator.hpp> (inc/simulator.hpp: Simulator, SimConfig, run_sim, capacity_sweep):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/server.hpp"
