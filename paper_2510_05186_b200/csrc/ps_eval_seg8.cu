// Evaluator variants for 8 lanes per candidate (stages <= 8).
#include "ps_eval_impl.cuh"
namespace ps {
PS_INSTANTIATE(8)
}
