/*
 * rsim/cases.h — seeded synthetic inputs for the five BASELINE.json configs
 * (SURVEY.md Appendix A).  Host-only C++ (no CUDA), part of librsim.so.
 *
 * The reference has no case files (proj/.gitignore:1); every
 * gap filled here is a [choice] recorded in DESIGN.md §Cases.  The graph
 * produced is the input of build_matrix_grid (Υ by harmonic
 * TPFA) plus fracture conduits as face-Υ additions / NNCs.
 */
#ifndef RSIM_CASES_H
#define RSIM_CASES_H

#include <stdint.h>
#include "types.h"

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int32_t config;   /* 1..5: BASELINE.json configs[0..4]                         */
  int32_t nx, ny, nz; /* 0 -> config default; fracture geometry scales with it */
  uint64_t seed;    /* 0 -> 2008015390 + config                                  */
  int32_t n_dfn;    /* -1 -> default (c2: 40, c4: 400, scaled with area)         */
  int32_t n_steps;  /* -1 -> default                                             */
} rsim_case_opts;

typedef struct rsim_case rsim_case;

rsim_case* rsim_case_create(const rsim_case_opts* o);
void       rsim_case_destroy(rsim_case* c);
int64_t    rsim_case_n(const rsim_case* c);
int        rsim_case_dims(const rsim_case* c, int32_t* nxyz3, double* dxyz3);
int        rsim_case_graph(const rsim_case* c, rsim_graph_desc* out);   /* borrowed pointers */
int        rsim_case_fluid(const rsim_case* c, rsim_fluid_params* out);
const double* rsim_case_perm(const rsim_case* c, int32_t axis);          /* m^2, per cell */
int        rsim_case_init_state(const rsim_case* c, double* u, uint8_t* st);
int32_t    rsim_case_schedule(const rsim_case* c, double* dts, int32_t cap); /* seconds */
int        rsim_case_solver_opts(const rsim_case* c, rsim_solver_opts* out);
int64_t    rsim_case_n_nnc(const rsim_case* c);                          /* directed entries */

/* Config 5 synthetic Newton update: δp_i = exp(-d_i^2/(2R^2))
 * with d_i the distance to the nearest of 64 seeded points; R is bisected so
 * that the post-dilation (m=2, ε=1e-3) active fraction hits `target`.
 * Writes dp (n), returns the achieved fraction; R in *R_out (m). */
double     rsim_case_c5_field(const rsim_case* c, double target, int32_t m, double eps,
                              double* dp, double* R_out);

#ifdef __cplusplus
}
#endif
#endif
