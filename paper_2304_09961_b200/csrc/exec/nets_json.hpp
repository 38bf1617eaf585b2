// Network description as JSON (ops, tensor plan, weight offsets): what the
// CPU oracles in oracle/ interpret. Shared by libbs_nets.so and libbs_exec.so.
#pragma once

#include <cstddef>

#include <json.hpp>

#include "netdef.hpp"

namespace bs200 {
nlohmann::json suite_json(const Suite& s, std::size_t blob_floats);
}  // namespace bs200
