// Result emission in the reference's formats (proj/include/batchsim/report.hpp:19-86):
// outcome CSV (seconds with %.9f), summary JSON, capacity-sweep CSV. Fixed
// formatting, so identical runs give byte-identical files and B200 runs diff
// directly against reference runs.
#pragma once

#include <ostream>
#include <string>
#include <vector>

#include <json.hpp>

#include "server.hpp"

namespace batchsim {

std::string format_seconds(Ms ms);
const char* location_name(const RequestOutcome& o);
void write_outcomes_csv(std::ostream& out, const std::vector<RequestOutcome>& outcomes, const ProfileSet& ps);
nlohmann::json summary_json(const SummaryMetrics& m);

struct SweepRow {
  std::string scheduler;
  double rate = 0;
  double ratio_mean = 0;
  double ratio_std = 0;
  double mean_completion_s_mean = 0;
  double mean_completion_s_std = 0;
};
void write_sweep_csv(std::ostream& out, const std::vector<SweepRow>& rows);

}  // namespace batchsim
