// Synthetic model catalog; tensor lists and byte counts reproduce the
// reference's make_model / default_catalog (catalog.hpp:23-90) so the same
// TensorIds and sizes flow through both implementations.
#include <cstdio>

#include "model.hpp"

namespace tg {

namespace {
TensorDesc tensor(const std::string& model, const char* name, u64 bytes) {
    TensorDesc t;
    t.model_id = model;
    t.name = name;
    t.size = bytes;
    const std::int64_t elems = static_cast<std::int64_t>(bytes / 2);  // f16 elements
    t.id = tensor_key(model, name, &elems, 1, Dtype::F16);
    return t;
}
}  // namespace

ModelDesc make_model(const std::string& model_id, u64 total_size, int layers, u64 bytes_per_token, Location loc,
                     double alpha) {
    ModelDesc m;
    m.model_id = model_id;
    m.total_size = total_size;
    m.location = loc;
    m.alpha = alpha;
    m.bytes_per_token = bytes_per_token;
    const u64 embed = total_size / 20;
    const u64 layer_bytes = (total_size - embed) / static_cast<u64>(layers);
    const u64 attn = layer_bytes / 3;
    u64 assigned = embed;
    char name[32];
    for (int l = 0; l < layers; ++l) {
        std::snprintf(name, sizeof name, "layer%02d.attn", l);
        m.tensors.push_back(tensor(model_id, name, attn));
        assigned += attn;
        const u64 mlp = (l + 1 == layers) ? total_size - assigned : layer_bytes - attn;
        std::snprintf(name, sizeof name, "layer%02d.mlp", l);
        m.tensors.push_back(tensor(model_id, name, mlp));
        assigned += mlp;
    }
    m.tensors.push_back(tensor(model_id, "tok_embed", embed));
    std::sort(m.tensors.begin(), m.tensors.end(),
              [](const TensorDesc& a, const TensorDesc& b) { return a.name < b.name; });
    return m;
}

std::vector<ModelDesc> default_catalog() {
    struct Entry {
        const char* id;
        double billions;
        int layers;
    };
    static const Entry kRows[] = {{"opt1.3B", 1.3, 12}, {"qwen3B", 3.0, 13}, {"llama3B", 3.0, 13},
                                  {"opt6.7B", 6.7, 16}, {"llama8B", 8.0, 16}, {"yi9B", 9.0, 18},
                                  {"opt13B", 13.0, 20}, {"gpt20B", 20.0, 22}};
    std::vector<ModelDesc> out;
    for (const auto& e : kRows) {
        const u64 total = static_cast<u64>(e.billions * 2e9);
        const u64 bpt = (total / 100000 + 1023) / 1024 * 1024;
        out.push_back(make_model(e.id, total, e.layers, bpt));
    }
    return out;
}

}  // namespace tg
