// Compiled cascade inference: tree-ensemble evaluation in C++ (§8f row 2).
//
// Replaces the reference's numpy lockstep walker (inference.py:55-125) with
// a direct per-tree walk over flattened node arrays.  Semantics follow
// docs/model_schema.md exactly: `x[f] <= threshold` goes left, per-class
// leaf sums accumulate in tree-list order as float64, and the argmax breaks
// exact ties toward the lowest class index.
#include <cstdint>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "../../include/spmvtune_b200.h"

namespace svb {
void set_error(const std::string& msg);
}

struct svb_forest {
  int32_t nclasses = 0;
  std::vector<int32_t> tree_class, roots, feature, left, right;
  std::vector<double> threshold, score;
};

extern "C" {

int svb_forest_create(int32_t nclasses, int32_t ntrees, const int32_t* tree_class,
                      const int32_t* roots, int32_t nnodes, const int32_t* feature,
                      const double* threshold, const int32_t* left, const int32_t* right,
                      const double* score, svb_forest** out) {
  if (nclasses < 1 || ntrees < 1 || nnodes < 1 || !out) {
    svb::set_error("forest: empty model");
    return SVB_INVALID;
  }
  auto* f = new (std::nothrow) svb_forest();
  if (!f) return SVB_OOM;
  f->nclasses = nclasses;
  f->tree_class.assign(tree_class, tree_class + ntrees);
  f->roots.assign(roots, roots + ntrees);
  f->feature.assign(feature, feature + nnodes);
  f->threshold.assign(threshold, threshold + nnodes);
  f->left.assign(left, left + nnodes);
  f->right.assign(right, right + nnodes);
  f->score.assign(score, score + nnodes);
  for (int32_t i = 0; i < nnodes; ++i) {
    const bool leaf = f->feature[i] < 0;
    if (!leaf && (f->feature[i] >= 15 || f->left[i] < 0 || f->left[i] >= nnodes || f->right[i] < 0 ||
                  f->right[i] >= nnodes)) {
      delete f;
      svb::set_error("forest: malformed node " + std::to_string(i));
      return SVB_INVALID;
    }
  }
  *out = f;
  return SVB_OK;
}

int svb_forest_destroy(svb_forest* f) {
  delete f;
  return SVB_OK;
}

int svb_forest_predict(const svb_forest* f, const double* x, double* scores, int32_t* label) {
  if (!f || !x) return SVB_INVALID;
  std::vector<double> acc(f->nclasses, 0.0);
  const size_t ntrees = f->roots.size();
  for (size_t t = 0; t < ntrees; ++t) {
    int32_t n = f->roots[t];
    while (f->feature[n] >= 0) n = (x[f->feature[n]] <= f->threshold[n]) ? f->left[n] : f->right[n];
    acc[f->tree_class[t]] += f->score[n];
  }
  int32_t best = 0;
  for (int32_t k = 1; k < f->nclasses; ++k)
    if (acc[k] > acc[best]) best = k;
  if (scores) std::memcpy(scores, acc.data(), sizeof(double) * f->nclasses);
  if (label) *label = best;
  return SVB_OK;
}

}  // extern "C"
