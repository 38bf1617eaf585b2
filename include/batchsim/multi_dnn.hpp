// Drop-in shim for <batchsim/multi_dnn.hpp> (inc/multi_dnn.hpp: reschedule_trigger, collect_riders, schedule_multi(_shared)):
// reference code compiles unchanged with -I<repo>/include and links libbs_host.so.
#pragma once
#include "../../paper_2304_09961_b200/csrc/host/bsb/schedulers.hpp"
