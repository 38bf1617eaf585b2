// Drop-in shim for <batchsim/cost_model.hpp> (inc/cost_model.hpp: CostTable, DnnProfile, ProfileSet, group_layers, check_subadditivity):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/profile.hpp"
