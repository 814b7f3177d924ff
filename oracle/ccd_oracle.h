/*
 * TEST INFRASTRUCTURE ONLY — CPU restatement of the reference ccdkit hot path.
 *
 * Plain C11, IEEE double round-to-nearest, no FMA contraction.  Each function
 * cites the reference file:line it restates (paths under
 * /root/reference/proj/).  Parity of this restatement is PINNED against the
 * reference itself compiled in oracle/_ref (tests/test_oracle_cpu.py) and
 * against the golden vectors in tests/golden/.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may
 * load liborc.so.  The product (paper_2112_06300_b200) never does.
 */
#ifndef CCD_ORACLE_H
#define CCD_ORACLE_H

#include <stdint.h>

#include "../include/ccdk.h"

#ifdef __cplusplus
extern "C" {
#endif

float orc_round_down_reduced(double x);
float orc_round_up_reduced(double x);

/* returns 0 or CCDK_INVALID_INPUT */
int orc_build_boxes(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
                    uint64_t ne, const uint32_t* f, uint64_t nf, double inflation,
                    float* mn, float* mx, uint8_t* kind, uint32_t* index);

int orc_choose_axis(const float* mn, const float* mx, uint64_t k);

/* stq/sap/bf candidate set; pairs malloc'd (2 u64 per pair), free with orc_free.
 * rounds (StqStats::round_sizes) malloc'd when non-NULL. */
int orc_broad(int method, const float* mn, const float* mx, const uint8_t* kind,
              const uint32_t* index, uint64_t k, const uint32_t* e, uint64_t ne,
              const uint32_t* f, uint64_t nf, uint64_t rb, uint64_t re, uint64_t** pairs,
              uint64_t* npairs, uint64_t** rounds, uint64_t* nrounds, uint64_t* max_queue);

int orc_classify(const uint64_t* pairs, uint64_t np, const double* v0, const double* v1,
                 uint64_t nv, const uint32_t* e, uint64_t ne, const uint32_t* f,
                 uint64_t nf, uint8_t* kind_out, double* points_out, uint64_t* source_out,
                 uint64_t* n_vf, uint64_t* n_ee);

void orc_inclusion_box(uint8_t kind, const double* points, const double* box, double* out);

void orc_process_interval(uint8_t kind, const double* points, const double* box,
                          const uint16_t* depth, double t_star, double sep,
                          const ccdk_narrow_cfg* cfg, uint8_t* action, double* cand_t,
                          uint8_t* zdiag, double* children, uint16_t* child_depth);

int orc_narrow_phase(const uint8_t* kind, const double* points, uint64_t n,
                     const double* seps, const ccdk_narrow_cfg* cfg, uint64_t capacity,
                     double* toi, uint8_t* flags, ccdk_narrow_stats* stats);

/* Full step with the default (unbounded) memory budget, Absolute min-sep. */
int orc_ccd(const double* v0, const double* v1, uint64_t nv, const uint32_t* e,
            uint64_t ne, const uint32_t* f, uint64_t nf, const ccdk_pipeline_cfg* cfg,
            ccdk_report* rep, uint64_t** pairs);

void orc_free(void* p);

#ifdef __cplusplus
}
#endif

#endif
