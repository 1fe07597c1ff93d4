// Evaluator variants for 4 lanes per candidate (stages <= 4).
#include "ps_eval_impl.cuh"
namespace ps {
PS_INSTANTIATE(4)
}
