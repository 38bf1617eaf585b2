/* C ABI of libbs_nets.so: the executor's network definitions, calibrated
 * weights and synthetic images on the host, with no CUDA dependency.
 * libbs_exec.so exports the same three network entry points (bs_exec.h).
 *
 * The reference (batchsim) has networks only as cost tables
 * (proj/data/profiles/*.json, profile_io.hpp:3-18); these are the concrete
 * layer decompositions of SURVEY.md §7.3 with the deterministic inputs and
 * weights of §7.4. Used by the CPU oracles and by bench.py's reference arm,
 * which must not load the executor.
 */
#ifndef BS_NETS_H_
#define BS_NETS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* JSON description of a suite (ops, tensor plan, weight offsets); free with bs_nets_free. */
int bs_describe_suite(const char* suite, char** out_json);
/* The suite's calibrated, TF32-rounded weight pool (n >= the description's "weights"). */
int bs_suite_weights_host(const char* suite, float* dst, size_t n);
/* Synthetic NHWC image (SplitMix64 N(0,1), TF32-rounded), zero in channels >= real_c. */
int bs_make_image(uint64_t seed, uint64_t index, int H, int W, int C, int real_c, float* out);
const char* bs_nets_last_error(void);
void bs_nets_free(void* p);

#ifdef __cplusplus
}
#endif

#endif /* BS_NETS_H_ */
