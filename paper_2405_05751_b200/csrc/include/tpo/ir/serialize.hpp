// B200 backend — JSON wire format.  API mirror of the reference's
// tpo/ir/serialize.hpp (proj/core/include/tpo/ir/serialize.hpp:26-40); the
// same schema is the payload of tpo_gpu_compile() in include/tpo_gpu.h.
#pragma once

#include <string>

#include <json.hpp>

#include "tpo/ir/graph.hpp"

namespace tpo::ir {

nlohmann::json to_json(const KernelGraph &g);
KernelGraph kernel_graph_from_json(const nlohmann::json &j);

// Allocation-light fast path for JSON text (host/fastjson.cpp): true and
// `out` set exactly as kernel_graph_from_json(parse(text)) would, or false
// for any input outside its strict subset (the caller then takes the
// nlohmann path, which yields the canonical result or error).
bool kernel_graph_from_text_fast(const char *text, size_t n, KernelGraph &out);

nlohmann::json dim_map_to_json(const DimMap &m, bool grid_axes);
DimMap dim_map_from_json(const nlohmann::json &j, bool grid_axes);

KernelGraph load_graph_file(const std::string &path);
void save_graph_file(const KernelGraph &g, const std::string &path, bool pretty);

}  // namespace tpo::ir
