/* TEST INFRASTRUCTURE ONLY: CPU oracle for the LSP projector path (see lsp_oracle.c). */
#ifndef LSP_ORACLE_H_
#define LSP_ORACLE_H_
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
const char* orc_last_error(void);
uint64_t orc_derive_seed(uint64_t master, uint64_t tag, uint64_t index);
int orc_init_sparse(int n_rows, int d, int r, uint64_t seed, int32_t* pos, double* val);
int orc_compress(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                 const int32_t* qpos, const double* qval, const double* g, double* s_out);
int orc_decompress(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                   const int32_t* qpos, const double* qval, const double* s, double* out);
int orc_decompress_apply(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                         const int32_t* qpos, const double* qval, const double* delta,
                         double lr, double* w);
int orc_estimation_bias(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                        const int32_t* qpos, const double* qval, const double* sigma,
                        double* out);
int orc_relative_bias(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                      const int32_t* qpos, const double* qval, const double* sigma,
                      double* out);
int orc_adam_step(int rows, int cols, int64_t step, double beta1, double beta2, double eps,
                  const double* m_in, const double* v_in, const double* grad, double* m_out,
                  double* v_out, double* delta, int64_t* step_out);
int orc_fit_loss(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                 const int32_t* qpos, const double* qval, int t, const double* targets,
                 double reg_beta, int reg_kind, double* out);
int orc_fit_gradient(int m, int n, int d, int r, const int32_t* ppos, const double* pval,
                     const int32_t* qpos, const double* qval, int t, const double* targets,
                     double reg_beta, int reg_kind, double* gp, double* gq);
int orc_fit(int m, int n, int d, int r, const int32_t* ppos, double* pval, const int32_t* qpos,
            double* qval, int t, const double* targets, double alpha, double reg_beta,
            double step_size, int max_steps, int timeout_steps, int reg_kind, double* report,
            double* loss_curve, int max_curve);
int orc_projector_gram(int n_rows, int da, int ra, const int32_t* apos, const double* aval,
                       int db, int rb, const int32_t* bpos, const double* bval, double* out);
int orc_reproject_state(int m, int n, int d, int r, const int32_t* oppos, const double* opval,
                        const int32_t* oqpos, const double* oqval, const int32_t* nppos,
                        const double* npval, const int32_t* nqpos, const double* nqval,
                        const double* m_in, const double* v_in, int kind, double* m_out,
                        double* v_out);
int orc_subsample_size(double gamma, double beta, int m, int n, int total_steps, double delta,
                       int64_t* out);
#ifdef __cplusplus
}
#endif
#endif
