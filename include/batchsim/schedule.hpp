// Drop-in shim for <batchsim/schedule.hpp> (inc/schedule.hpp: Schedule, SegmentSweep, segment_duration):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/sweep.hpp"
#include "../../paper_2304_09961_b200/csrc/host/bsb/schedulers.hpp"
