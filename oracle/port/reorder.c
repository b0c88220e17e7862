/* ORACLE restatement of Alg. 2/3: src/reorder.cpp, src/workload.cpp:179-204. */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "port.h"

/* sorted_by_key — src/reorder.cpp:30-42 (stable by (size, index)). */
static const double* g_sizes;
static int g_desc;
static int cmp_key(const void* pa, const void* pb) {
  const int a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  if (g_sizes[a] != g_sizes[b]) {
    const int less = g_desc ? g_sizes[a] > g_sizes[b] : g_sizes[a] < g_sizes[b];
    return less ? -1 : 1;
  }
  return a < b ? -1 : (a > b);
}

/* intra_partition — src/reorder.cpp:70-90; flat() — :46-52. */
int port_intra_partition(const double* sizes, int64_t n, int m, int order,
                         int equal_counts, int32_t* flat, int64_t* offsets) {
  if (m < 1) return port_fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  if (n == 0) return port_fail(DTB_ERR_INTERNAL, "cannot reorder an empty batch");
  int32_t* sorted = malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) sorted[i] = (int32_t)i;
  g_sizes = sizes;
  g_desc = order == DTB_DESCENDING;
  qsort(sorted, (size_t)n, sizeof(int32_t), cmp_key);
  const int64_t cap = equal_counts ? (n + m - 1) / m : n;
  double* load = calloc((size_t)m, sizeof(double));
  int64_t* count = calloc((size_t)m, sizeof(int64_t));
  int32_t* group_of = malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t k = 0; k < n; ++k) {
    const int32_t idx = sorted[k];
    int target = -1;
    for (int g = 0; g < m; ++g) {
      if (count[g] >= cap) continue;
      if (target < 0 || load[g] < load[target]) target = g;
    }
    group_of[k] = target;
    count[target] += 1;
    load[target] += sizes[idx];
  }
  offsets[0] = 0;
  for (int g = 0; g < m; ++g) offsets[g + 1] = offsets[g] + count[g];
  int64_t* fill = calloc((size_t)m, sizeof(int64_t));
  for (int64_t k = 0; k < n; ++k) {
    const int g = group_of[k];
    flat[offsets[g] + fill[g]++] = sorted[k];
  }
  free(sorted); free(load); free(count); free(group_of); free(fill);
  return 0;
}

/* block_group_loads — src/reorder.cpp:111-119.  (The reference divides by
 * zero when n < m; reported here as an InternalError.) */
int port_block_group_loads(const double* sizes, const int32_t* order,
                           int64_t n, int m, double* loads) {
  if (m < 1) return port_fail(DTB_ERR_INTERNAL, "group count must be >= 1");
  const int64_t per_group = n / m;
  if (per_group == 0 && n > 0)
    return port_fail(DTB_ERR_INTERNAL, "fewer samples than groups");
  for (int g = 0; g < m; ++g) loads[g] = 0.0;
  for (int64_t pos = 0; pos < n; ++pos) {
    int64_t b = pos / per_group;
    if (b > m - 1) b = m - 1;
    loads[b] += sizes[order[pos]];
  }
  return 0;
}

static const double* g_keys;
static int cmp_min(const void* pa, const void* pb) {
  const int a = *(const int32_t*)pa, b = *(const int32_t*)pb;
  if (g_keys[a] != g_keys[b]) return g_keys[a] < g_keys[b] ? -1 : 1;
  return a < b ? -1 : (a > b);
}

/* select_min — src/reorder.cpp:121-134. */
int port_select_min(const double* keys, const int32_t* pending, int64_t np,
                    int k, int32_t* out) {
  if (k < 0 || k > np)
    return port_fail(DTB_ERR_K_TOO_LARGE, "select_min asked for %d of %lld", k,
                     (long long)np);
  int32_t* s = malloc(sizeof(int32_t) * (size_t)(np ? np : 1));
  memcpy(s, pending, sizeof(int32_t) * (size_t)np);
  g_keys = keys;
  qsort(s, (size_t)np, sizeof(int32_t), cmp_min);
  memcpy(out, s, sizeof(int32_t) * (size_t)k);
  free(s);
  return 0;
}

/* select_closest — src/reorder.cpp:136-175. */
int port_select_closest(const double* keys, const int32_t* pending, int64_t np,
                        int k, double target, int32_t* out) {
  if (k < 0 || k > np)
    return port_fail(DTB_ERR_K_TOO_LARGE, "select_closest asked for %d of %lld",
                     k, (long long)np);
  int32_t* pool = malloc(sizeof(int32_t) * (size_t)(np ? np : 1));
  memcpy(pool, pending, sizeof(int32_t) * (size_t)np);
  int64_t n = np;
  double residual = target;
  for (int pick = 0; pick < k; ++pick) {
    int best = -1;
    int64_t best_pos = -1;
    for (int64_t q = 0; q < n; ++q) {
      const int idx = pool[q];
      if (best < 0) {
        best = idx;
        best_pos = q;
        continue;
      }
      const double da = fabs(residual - keys[idx]);
      const double db = fabs(residual - keys[best]);
      if (da != db) {
        if (da < db) best = idx, best_pos = q;
        continue;
      }
      const int a_under = keys[idx] <= residual;
      const int b_under = keys[best] <= residual;
      if (a_under != b_under) {
        if (a_under) best = idx, best_pos = q;
        continue;
      }
      if (idx < best) best = idx, best_pos = q;
    }
    out[pick] = best;
    residual -= keys[best];
    memmove(pool + best_pos, pool + best_pos + 1,
            sizeof(int32_t) * (size_t)(n - best_pos - 1));
    --n;
  }
  free(pool);
  return 0;
}

static void remove_from(int32_t* pool, int64_t* n, int32_t idx) {
  for (int64_t q = 0; q < *n; ++q) {
    if (pool[q] == idx) {
      memmove(pool + q, pool + q + 1, sizeof(int32_t) * (size_t)(*n - q - 1));
      --*n;
      return;
    }
  }
}

/* candidate_times — src/reorder.cpp:182-225. */
static void candidate_times(const double* f, const double* b, int l, int p,
                            const int32_t* placed, int64_t np,
                            const int32_t* pend, int64_t npd,
                            const int32_t* rear, int64_t nr, double* cf,
                            double* cb, double* mf, double* mb) {
  for (int s = 0; s < p; ++s) mf[s] = mb[s] = 0.0;
  if (npd > 0) {
    for (int64_t q = 0; q < npd; ++q)
      for (int s = 0; s < p; ++s) {
        mf[s] += f[(size_t)pend[q] * p + s];
        mb[s] += b[(size_t)pend[q] * p + s];
      }
    for (int s = 0; s < p; ++s) {
      mf[s] /= (double)npd;
      mb[s] /= (double)npd;
    }
  }
  int row = 0;
  for (int64_t q = 0; q < np; ++q, ++row)
    for (int s = 0; s < p; ++s) {
      cf[(size_t)row * p + s] = f[(size_t)placed[q] * p + s];
      cb[(size_t)row * p + s] = b[(size_t)placed[q] * p + s];
    }
  for (int64_t q = 0; q < npd; ++q, ++row)
    for (int s = 0; s < p; ++s) {
      cf[(size_t)row * p + s] = mf[s];
      cb[(size_t)row * p + s] = mb[s];
    }
  for (int64_t q = 0; q < nr; ++q, ++row)
    for (int s = 0; s < p; ++s) {
      cf[(size_t)row * p + s] = f[(size_t)rear[q] * p + s];
      cb[(size_t)row * p + s] = b[(size_t)rear[q] * p + s];
    }
  (void)l;
}

/* inter_reorder — src/reorder.cpp:238-298 (windows_for :227-234). */
int port_inter_reorder(const double* f, const double* b, int l, int p,
                       const double* keys, int vpp, int32_t* out) {
  for (int i = 0; i < l; ++i) out[i] = i;
  if (l <= 1) return 0;
  if (vpp < 1) return port_fail(DTB_ERR_INDIVISIBLE_VPP, "vpp must be >= 1");
  if (p % vpp != 0)
    return port_fail(DTB_ERR_INDIVISIBLE_VPP, "stage count not divisible by vpp");
  const int devices = p / vpp;
  if (devices == 1) return 0;

  int32_t* pending = malloc(sizeof(int32_t) * l);
  int32_t* ret = malloc(sizeof(int32_t) * l);
  int32_t* rear = malloc(sizeof(int32_t) * l);
  int32_t* cur = malloc(sizeof(int32_t) * l);
  double* cf = malloc(sizeof(double) * (size_t)l * p);
  double* cb = malloc(sizeof(double) * (size_t)l * p);
  double* mf = malloc(sizeof(double) * p);
  double* mb = malloc(sizeof(double) * p);
  double* st = malloc(sizeof(double) * (size_t)2 * l * vpp);
  int64_t np = l, nret = 0, nrear = 0;
  int status = 0;
  for (int i = 0; i < l; ++i) pending[i] = i;

  int32_t first;
  port_select_min(keys, pending, np, 1, &first);
  ret[nret++] = first;
  remove_from(pending, &np, first);
  const int tail_n = (devices - 1) < np ? (devices - 1) : (int)np;
  port_select_min(keys, pending, np, tail_n, rear);
  nrear = tail_n;
  for (int i = 0; i < tail_n; ++i) remove_from(pending, &np, rear[i]);

  int step = 1;
  while (np > 0) {
    candidate_times(f, b, l, p, ret, nret, pending, np, rear, nrear, cf, cb, mf,
                    mb);
    port_timeline tl;
    status = port_schedule(cf, cb, l, p, vpp, &tl);
    if (status != 0) break;
    const int64_t nw = port_get_intervals(tl.events, tl.n_events, st,
                                          st + (size_t)l * vpp, NULL, NULL);
    port_timeline_free(&tl);
    const int take = step == 1 ? ((devices - 1) < np ? (devices - 1) : (int)np) : 1;
    double target = 0.0;
    for (int w = 0; w < vpp; ++w) {
      const int64_t wi = (int64_t)(step - 1) * vpp + w;
      if (wi < nw) target += st[(size_t)l * vpp + wi] - st[wi];
    }
    port_select_closest(keys, pending, np, take, target, cur);
    for (int i = 0; i < take; ++i) {
      ret[nret++] = cur[i];
      remove_from(pending, &np, cur[i]);
    }
    ++step;
  }
  if (status == 0) {
    for (int64_t i = 0; i < nrear; ++i) ret[nret++] = rear[i];
    memcpy(out, ret, sizeof(int32_t) * l);
  }
  free(pending); free(ret); free(rear); free(cur); free(cf); free(cb);
  free(mf); free(mb); free(st);
  return status;
}

/* Modality tokens of sample i (Sample::modality_tokens, src/core.cpp:90-95). */
static int64_t modality(const dtb_samples* s, int64_t i) {
  int64_t t = 0;
  for (int32_t k = s->image_offsets[i]; k < s->image_offsets[i + 1]; ++k)
    t += s->image_tokens[k];
  if (s->audio_offsets)
    for (int32_t k = s->audio_offsets[i]; k < s->audio_offsets[i + 1]; ++k)
      t += s->audio_tokens[k];
  return t;
}

/* assemble_microbatches — src/workload.cpp:179-204 — as token keys of the
 * samples `tok[order[.]]` (order NULL = identity). */
static void assemble(const dtb_plan* plan, const int64_t* tok,
                     const int32_t* order, port_mb* mbs) {
  const int64_t per_group = plan->global_batch / plan->unit[DTB_BACKBONE].dp;
  const int coupled = plan->unit[DTB_ENCODER].dp;
  const int span = plan->unit[DTB_BACKBONE].dp / plan->unit[DTB_ENCODER].dp;
  for (int e = 0; e < coupled; ++e)
    for (int64_t i = 0; i < per_group; ++i) {
      port_mb* mb = &mbs[(size_t)e * per_group + i];
      mb->enc = mb->gen = 0;
      mb->count = span;
      for (int j = 0; j < span; ++j) {
        const int64_t idx = (int64_t)(e * span + j) * per_group + i;
        const int64_t t = tok[order ? order[idx] : idx];
        mb->enc += t;
        mb->gen += t;
      }
    }
}

static double max_of(const double* v, int n) {
  double m = v[0];
  for (int i = 1; i < n; ++i)
    if (m < v[i]) m = v[i];
  return m;
}

/* disaggregated_reorder — src/reorder.cpp:319-396. */
int port_disaggregated_reorder(const port_cm* cm, const dtb_plan* plan,
                               const dtb_reorder_mode* mode,
                               const dtb_samples* s, int64_t first,
                               dtb_reorder_report* rep) {
  const int64_t n = plan->global_batch;
  const int dp_lm = plan->unit[DTB_BACKBONE].dp;
  const int64_t per_group = plan->global_batch / dp_lm;
  const int coupled = plan->unit[DTB_ENCODER].dp;
  const int span = dp_lm / plan->unit[DTB_ENCODER].dp;
  const int p = (plan->unit[0].pp + plan->unit[1].pp + plan->unit[2].pp) * plan->vpp;
  int status = 0;

  int64_t* tok = malloc(sizeof(int64_t) * (size_t)n);
  double* sizes = malloc(sizeof(double) * (size_t)n);
  int32_t* identity = malloc(sizeof(int32_t) * (size_t)n);
  int32_t* intra = malloc(sizeof(int32_t) * (size_t)n);
  for (int64_t i = 0; i < n; ++i) {
    tok[i] = modality(s, first + i);
    sizes[i] = (double)(tok[i] + tok[i]); /* cost_size */
    identity[i] = intra[i] = (int32_t)i;
  }
  double* la = malloc(sizeof(double) * dp_lm);
  double* lb = malloc(sizeof(double) * dp_lm);
  const size_t nmb = (size_t)coupled * per_group;
  port_mb* mbs = malloc(sizeof(port_mb) * (nmb ? nmb : 1));
  port_mb* reord = malloc(sizeof(port_mb) * (nmb ? nmb : 1));
  int64_t* goff = malloc(sizeof(int64_t) * (coupled + 1));
  double* f = malloc(sizeof(double) * (size_t)(per_group ? per_group : 1) * (p ? p : 1));
  double* b = malloc(sizeof(double) * (size_t)(per_group ? per_group : 1) * (p ? p : 1));
  double* keys = malloc(sizeof(double) * (size_t)(per_group ? per_group : 1));
  int32_t* ord = malloc(sizeof(int32_t) * (size_t)(per_group ? per_group : 1));

  if (mode->intra) {
    int32_t* greedy = malloc(sizeof(int32_t) * (size_t)n);
    int64_t* offs = malloc(sizeof(int64_t) * (dp_lm + 1));
    status = port_intra_partition(sizes, n, dp_lm, mode->sort_order, 1, greedy, offs);
    if (status == 0) status = port_block_group_loads(sizes, greedy, n, dp_lm, la);
    if (status == 0) status = port_block_group_loads(sizes, identity, n, dp_lm, lb);
    if (status == 0 && max_of(la, dp_lm) <= max_of(lb, dp_lm))
      memcpy(intra, greedy, sizeof(int32_t) * (size_t)n);
    free(greedy);
    free(offs);
  }
  if (status == 0) status = port_block_group_loads(sizes, identity, n, dp_lm, rep->group_load_before);
  if (status == 0) status = port_block_group_loads(sizes, intra, n, dp_lm, rep->group_load_after);
  if (status == 0) {
    for (int e = 0; e <= coupled; ++e) goff[e] = (int64_t)e * per_group;
    assemble(plan, tok, NULL, mbs);
    status = port_simulate_iteration(cm, plan, coupled, goff, mbs,
                                     &rep->t_iter_before, NULL, NULL, NULL, NULL);
  }
  if (status == 0) {
    assemble(plan, tok, intra, mbs);
    for (int64_t i = 0; i < n; ++i) rep->output_order[i] = 0;
    for (int e = 0; e < coupled && status == 0; ++e) {
      port_mb* grp = mbs + (size_t)e * per_group;
      for (int64_t i = 0; i < per_group; ++i) ord[i] = (int32_t)i;
      if (mode->inter) {
        status = port_build_stage_times(cm, plan, grp, per_group, f, b);
        if (status == 0) status = port_fwd_keys(cm, plan, grp, per_group, keys);
        if (status == 0)
          status = port_inter_reorder(f, b, (int)per_group, p, keys, plan->vpp, ord);
      }
      for (int64_t i = 0; i < per_group && status == 0; ++i) {
        reord[(size_t)e * per_group + i] = grp[ord[i]];
        for (int j = 0; j < span; ++j) {
          const int64_t pos = (int64_t)(e * span + j) * per_group + i;
          const int64_t src = (int64_t)(e * span + j) * per_group + ord[i];
          rep->output_order[pos] = intra[src];
        }
      }
    }
  }
  if (status == 0)
    status = port_simulate_iteration(cm, plan, coupled, goff, reord,
                                     &rep->t_iter_after, NULL, NULL, NULL, NULL);
  free(tok); free(sizes); free(identity); free(intra); free(la); free(lb);
  free(mbs); free(reord); free(goff); free(f); free(b); free(keys); free(ord);
  return status;
}
