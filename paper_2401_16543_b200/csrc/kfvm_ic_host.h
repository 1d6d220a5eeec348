// kfvm_ic_host.h — host-side IC plan (tables owned by std::vectors).
#ifndef KFVM_IC_HOST_H_
#define KFVM_IC_HOST_H_

#include <vector>

#include "../../include/kfvm_b200.h"
#include "kfvm_ic_eval.h"

namespace kfvm_b200 {

struct ICHostPlan {
  ICPlan plan;
  std::vector<double> fc[3], fs[3];
  bool needs_norm = false;
};

int ic_plan_build(const kfvm_config* cfg, const kfvm_ic_params* ic, ICHostPlan* hp);
int ic_generate_host(const kfvm_config* cfg, const kfvm_ic_params* ic, int z0, int nzl,
                     int nthreads, double* U);

}  // namespace kfvm_b200

#endif
