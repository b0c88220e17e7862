/* ORACLE (test infrastructure) — plain-C restatement of the reference
 * planner's hot path, used only as a checker by tests/ and as the
 * "port" CPU baseline when oracle/_ref is absent.  Each function cites the
 * reference source it restates (paths relative to
 * /root/reference/proj/core/).  Exported with the prefix `mmport_` behind
 * the ABI of include/disttrain_b200.h. */
#ifndef PORT_H
#define PORT_H

#include <stddef.h>
#include <stdint.h>

#include "disttrain_b200.h"

/* --- error state (errors.hpp:22-84 as status codes) ---------------------- */
extern _Thread_local int port_status;
extern _Thread_local char port_msg[512];
int port_fail(int status, const char* fmt, ...);
#define TRY(expr)                   \
  do {                              \
    if ((expr) != 0) return port_status; \
  } while (0)

/* --- cost model ----------------------------------------------------------- */
typedef struct {
  double load, fwd, bwd;
} port_row;

typedef struct dtb_cost_model {
  dtb_model_spec model;
  dtb_cluster_spec cluster;
  double eff, ratio;
  port_row* rows[3][4]; /* by module, log2(tp) */
  int nrows[3][4];
  int nonempty[3];
} port_cm;

int port_tp_index(int tp); /* -1 when tp not in {1,2,4,8} */
double port_max(double a, double b); /* std::max semantics */
double port_min(double a, double b);
double port_param_count(const dtb_arch* a);
int port_unit_forward(const port_cm* cm, int kind, int tp, double load, double* out);
int port_unit_backward(const port_cm* cm, int kind, int tp, double load, double* out);
double port_pp_boundary_seconds(const dtb_plan* plan, int unit,
                                const dtb_cluster_spec* c, double bytes);
double port_boundary_bytes(const port_cm* cm, int unit, const dtb_plan* plan,
                           double tokens);
void port_memory_check(const dtb_plan* plan, const dtb_model_spec* model,
                       const dtb_cluster_spec* cluster, dtb_memory_report* out);
/* Microbatch keys: encoder/generator token sums and sample count. */
typedef struct {
  int64_t enc, gen;
  int32_t count;
} port_mb;
double port_mb_mean_enc(const port_mb* mb);
double port_mb_mean_gen(const port_mb* mb);
int port_build_stage_times(const port_cm* cm, const dtb_plan* plan,
                           const port_mb* mbs, int64_t l, double* fwd,
                           double* bwd);
int port_fwd_keys(const port_cm* cm, const dtb_plan* plan, const port_mb* mbs,
                  int64_t l, double* keys);

/* --- pipeline simulator --------------------------------------------------- */
typedef struct {
  int device, mb, stage, phase;
  double start, end;
} port_event;

typedef struct {
  port_event* events; /* sorted as Timeline::events */
  int64_t n_events;
  int devices;
  double iteration_time;
  double* busy; /* [devices] */
} port_timeline;

int port_check_times(const double* fwd, const double* bwd, int l, int p);
int port_schedule(const double* fwd, const double* bwd, int l, int p, int vpp,
                  port_timeline* tl);
void port_timeline_free(port_timeline* tl);
/* get_intervals volumes + fill lists (fill arrays may be NULL). */
int64_t port_get_intervals(const port_event* ev, int64_t n, double* starts,
                           double* ends, int64_t* fill_off, int32_t* fill_mb);
int port_simulate_iteration(const port_cm* cm, const dtb_plan* plan,
                            int n_groups, const int64_t* group_off,
                            const port_mb* mbs, double* t_iter,
                            double* group_times, int32_t* slowest,
                            double* slowest_time, double* bubble);

/* --- reorder --------------------------------------------------------------- */
int port_intra_partition(const double* sizes, int64_t n, int m, int order,
                         int equal_counts, int32_t* flat, int64_t* offsets);
int port_block_group_loads(const double* sizes, const int32_t* order,
                           int64_t n, int m, double* loads);
int port_select_min(const double* keys, const int32_t* pending, int64_t np,
                    int k, int32_t* out);
int port_select_closest(const double* keys, const int32_t* pending, int64_t np,
                        int k, double target, int32_t* out);
int port_inter_reorder(const double* fwd, const double* bwd, int l, int p,
                       const double* keys, int vpp, int32_t* out);
int port_disaggregated_reorder(const port_cm* cm, const dtb_plan* plan,
                               const dtb_reorder_mode* mode,
                               const dtb_samples* s, int64_t first,
                               dtb_reorder_report* rep);

/* --- orchestration ----------------------------------------------------------- */
int port_predict_times(const port_cm* cm, const dtb_plan* plan,
                       const dtb_workload_stats* stats,
                       dtb_predicted_times* out);
int64_t port_enumerate(const dtb_cluster_spec* c, int64_t bs, dtb_tuple** out);
int port_solve_subproblem(const port_cm* cm, const dtb_workload_stats* stats,
                          const dtb_tuple* t, int64_t bs, int vpp,
                          dtb_candidate* out);

#endif
