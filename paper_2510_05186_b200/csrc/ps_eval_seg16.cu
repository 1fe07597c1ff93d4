// Evaluator variants for 16 lanes per candidate (stages <= 16).
#include "ps_eval_impl.cuh"
namespace ps {
PS_INSTANTIATE(16)
}
