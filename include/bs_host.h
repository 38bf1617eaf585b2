/* C ABI of the host scheduler library (libbs_host.so; no CUDA).
 *
 * A JSON job interface over the reference-compatible C++ scheduler
 * (paper_2304_09961_b200/csrc/host/bsb/*.hpp, namespace batchsim), which is
 * itself a drop-in for proj/include/batchsim/*.hpp:
 *   {"job":"sim", ...}   run_sim                 simulator.hpp:787-792
 *   {"job":"calls", ...} compute_schedule_dp     dp_time.hpp:152-315
 *                        tardy_dp / edf_batch    deadline.hpp:42-282
 *                        baseline_* / schedule_multi(_shared) / segment_duration /
 *                        group_layers / CostTable::lookup / SplitMix64 / generate_arrivals
 * Results print doubles as IEEE-754 bit patterns.
 */
#ifndef BS_HOST_H_
#define BS_HOST_H_

#ifdef __cplusplus
extern "C" {
#endif

int bs_host_call(const char* job_json, char** out_jsonl);
void bs_host_free(char* p);
const char* bs_host_last_error(void);

#ifdef __cplusplus
}
#endif

#endif /* BS_HOST_H_ */
