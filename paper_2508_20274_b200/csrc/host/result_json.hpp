// JSON rendering of RunResult for the Python API and the parity tests.
// Doubles are printed with %.17g (exact round trip); key names follow the reference's
// summary.json / actions.jsonl (trace.cpp:98-189).
#pragma once

#include <string>

#include "packer.hpp"

namespace mgb {

std::string result_to_json(const RunResult& r);
std::string json_escape(const std::string& s);

}  // namespace mgb
