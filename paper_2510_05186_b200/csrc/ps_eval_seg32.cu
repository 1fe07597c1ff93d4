// Evaluator variants for 32 lanes per candidate (stages <= 32).
#include "ps_eval_impl.cuh"
namespace ps {
PS_INSTANTIATE(32)
}
