// Drop-in shim for <batchsim/profile_io.hpp> (inc/profile_io.hpp: parse_profile, load_profile):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/profile.hpp"
