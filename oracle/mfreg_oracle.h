/* TEST INFRASTRUCTURE ONLY — the CPU checker, never the product.
 *
 * Plain-C restatement ("port") of the reference mfreg hot path
 * (/root/reference/proj/src). Every function cites the reference file:line it
 * follows and keeps the reference's exact floating-point operation order; the
 * library is compiled with -ffp-contract=off (oracle/Makefile) so that it is
 * bitwise identical to the reference library built with its own flags.
 * Parity of this port is PINNED by tests/test_oracle_port.py against
 * (a) the committed golden fixtures in tests/golden/ (generated from the
 * reference library by oracle/gen_golden.py) and (b) the reference library
 * itself (oracle/_ref/libmfreg_ref.so) when it is present.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline leg may
 * load this library. The symbol set mirrors oracle/ref_capi.cpp with the
 * prefix mport_ instead of mref_, with identical signatures.
 */
#ifndef MFREG_ORACLE_H
#define MFREG_ORACLE_H
#include <stdint.h>

typedef struct {
    int max_iters;
    double c1;
    double beta;
    int max_backtracks;
    int cg_max_iters;
    double cg_rel_tol;
    int h0_max_iters;
    double h0_rel_tol;
    int lbfgs_history;
    double gamma;
    double tol_rel_j;
    double tol_grad;
    double tol_step;
} mport_opt_config;

typedef struct {
    int iter;
    int cg_iters;
    double j;
    double distance;
    double regularizer;
    double grad_norm;
    double step;
} mport_iter_record;

#endif
