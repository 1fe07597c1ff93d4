// ps_literal.h — the literal run_order replay for malformed stage rows (ps_literal.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>
#include "ps_eval.cuh"

namespace ps {

// Bytes of one thread's scratch slot for a P x m instance with G channels.
size_t literal_slot_bytes(int P, int m, int G);
// Re-run every candidate flagged PS_FLAG_MALFORMED by the evaluator with the reference's literal
// semantics (listsched.py:167-269): `slots` threads, one scratch slot each.
cudaError_t literal_launch(const EvalParams &p, bool v64, int64_t *scratch, int slots, cudaStream_t s);

}  // namespace ps
