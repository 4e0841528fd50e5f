/* TEST INFRASTRUCTURE — NOT PRODUCT CODE.
 *
 * Plain-C restatement of the GeoDock per-ligand pose search (the hot path named by
 * BASELINE.json's north_star), used only as the parity checker by tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline leg. Parity pinning: tests/test_oracle.py checks every entry point
 * bit-for-bit against the unmodified reference compiled by oracle/Makefile (oracle/_ref) and
 * against the committed golden vectors in tests/golden/ (generated from oracle/_ref by
 * tests/golden/make_golden.py) plus the survey's Appendix-B known answers.
 *
 * The flat library layout matches gd_library in include/geodock_b200.h.
 */
#ifndef GEODOCK_ORACLE_H
#define GEODOCK_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

uint64_t go_splitmix_next(uint64_t* state);
uint64_t go_fnv1a64(const char* s, uint64_t len);
uint64_t go_mix_seed(uint64_t a, uint64_t b);

int go_rotation_grid(const uint32_t steps[3], double* q_out);
int go_make_pocket(const uint32_t dims[3], double spacing, const double origin[3], uint32_t blobs,
                   uint64_t seed, double* field_out);
int go_make_library(uint64_t count, uint64_t atoms, uint64_t rotamers, uint64_t seed, double* xyz,
                    double* radius, uint32_t* bonds, uint32_t* rots);
int go_sample_field(const uint32_t dims[3], const double origin[3], double spacing,
                    const double* field, uint64_t n, const double* pts, double* out);
int go_dock_library(uint32_t n_lig, const uint32_t* atom_off, const double* xyz,
                    const double* radius, const uint32_t* bond_off, const uint32_t* bonds,
                    const uint32_t* rot_off, const uint32_t* rots, const double* dihedrals,
                    const uint32_t* name_off, const char* names, const uint32_t dims[3],
                    const double origin[3], double spacing, const double* field,
                    uint32_t n_restarts, uint32_t reps, const uint32_t steps[3],
                    uint32_t dihedral_steps, double clash, uint64_t seed, double* best_score,
                    uint32_t* best_restart, uint64_t* score_calls, double* phase,
                    double* final_xyz, double* final_dih, uint32_t* align_index,
                    double* align_score, double* restart_score, int32_t* step_k,
                    double* step_score);
const char* go_last_error(void);

#ifdef __cplusplus
}
#endif
#endif
