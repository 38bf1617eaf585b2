// Drop-in shim for <batchsim/report.hpp> (inc/report.hpp: report writers):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/report.hpp"
