// Evaluator variants for 2 lanes per candidate (stages <= 2).
#include "ps_eval_impl.cuh"
namespace ps {
PS_INSTANTIATE(2)
}
