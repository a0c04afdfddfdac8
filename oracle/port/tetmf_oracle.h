/* tetmf_oracle.h -- plain-C restatement of the reference's CPU apply.
 *
 * TEST INFRASTRUCTURE ONLY (the checker, never the product path). Same entry
 * points as oracle/ref_driver.cpp with the "port_" prefix, so tests can run
 * the restatement and the compiled reference side by side.
 */
#ifndef TETMF_ORACLE_H
#define TETMF_ORACLE_H

#ifdef __cplusplus
extern "C" {
#endif

const char* port_last_error(void);
void* port_create(const char* mesh, const char* form, int level);
void port_destroy(void* h);
long long port_num_dofs(void* h);
int port_num_macros(void* h);
int port_dof_geometry(void* h, unsigned char* kind, double* a, double* b);
int port_interior(void* h, unsigned char* out);
long long port_coeff_num_dofs(void* h);
int port_coeff_geometry(void* h, double* a);
int port_interpolate(void* h, int which, double* out);
int port_apply(void* h, const double* v, const double* c0, const double* c1, int degree, double* w,
               double* seconds);
/* partial apply over a subset of macros (multi-rank tests): mask[m] != 0 */
int port_apply_macros(void* h, const double* v, const double* c0, const double* c1, int degree,
                      const unsigned char* macro_mask, double* w);

#ifdef __cplusplus
}
#endif

#endif
