// SPDX-License-Identifier: Apache-2.0
//
// Tensor-core engine (EMBER_ENGINE_TC_BF16X3) — tcgen05/TMEM kernels for the shared-negative
// contraction. Not yet available in this build: contexts requesting it are rejected at creation.
#include "engine.h"

namespace ember {

bool tc_engine_supported(const Engine&) { return false; }

void launch_contract_tc(Engine&, uint32_t) { throw EmberError("tensor-core engine not built"); }

}  // namespace ember
