// JSON-facing entry points (nlohmann/json, the parser the reference also
// uses; it only parses, no scheduling arithmetic depends on it).
#pragma once

#include <string>

#include <json.hpp>

#include "profile.hpp"

namespace batchsim {

ProfileSet parse_profile(const nlohmann::json& doc, const std::string& origin);

}  // namespace batchsim
