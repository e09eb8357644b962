// C++ boundary test: the reference-shaped host API (include/tgb/terngrad.hpp)
// over the C-ABI. Deterministic inputs from a 64-bit LCG (restated in
// tests/test_cpp_api.py); results are written to argv[1] and checked there
// against the CPU oracle. Build: __graft_entry__.build() -> build/tgb_cpp_api_test
#include <cstdio>
#include <fstream>
#include <string>
#include <variant>
#include <vector>

#include "tgb/terngrad.hpp"

static std::vector<float> lcg(uint64_t seed, size_t n, float scale) {
    std::vector<float> v(n);
    uint64_t x = seed;
    for (size_t k = 0; k < n; ++k) {
        x = x * 6364136223846793005ull + 1442695040888963407ull;
        v[k] = (static_cast<float>(x >> 40) * 0x1p-24f - 0.5f) * scale;
    }
    return v;
}

static void put(std::ofstream& f, const void* p, size_t n) {
    const uint64_t len = n;
    f.write(reinterpret_cast<const char*>(&len), 8);
    f.write(static_cast<const char*>(p), static_cast<std::streamsize>(n));
}

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    std::ofstream f(argv[1], std::ios::binary);
    const std::vector<std::string> names = {"conv.weight", "conv.bias", "fc.weight"};
    const std::vector<size_t> sizes = {1728, 64, 40003};
    tgb::CodecConfig cfg;
    cfg.seed = 42;
    std::vector<std::vector<tgb::GradTensor>> grads(2);
    for (int w = 0; w < 2; ++w)
        for (size_t l = 0; l < names.size(); ++l)
            grads[w].emplace_back(names[l], std::vector<size_t>{sizes[l]},
                                  lcg(1000 * (w + 1) + l, sizes[l], 1e-2f));
    // 1. encode_step (codec.hpp:194-239) for workers 0 and 1
    std::vector<tgb::EncodedGradient> enc;
    for (int w = 0; w < 2; ++w) {
        auto r = tgb::encode_step(grads[w], cfg, 3, static_cast<uint16_t>(w));
        put(f, r.local_scalers.data(), r.local_scalers.size() * 4);
        for (auto& b : r.encoded.blocks) {
            const auto& tb = std::get<tgb::TernaryBlock>(b);
            put(f, tb.codes.data(), tb.codes.size());
        }
        enc.push_back(std::move(r.encoded));
    }
    // 2. average over the two workers (codec.hpp:245-311), shared and unshared
    for (bool sharing : {true, false}) {
        auto avg = tgb::average(enc, 2, sharing);
        for (auto& a : avg) put(f, a.values.data(), a.values.size() * 4);
    }
    // 3. SyncWorker (Worker::run sync segment) on worker 0, N = 1
    tgb::SyncWorker sw(names, sizes, cfg);
    for (size_t l = 0; l < names.size(); ++l)
        tgb::detail::cuda_check(cudaMemcpy(sw.grad(static_cast<int>(l)), grads[0][l].values.data(),
                                           sizes[l] * 4, cudaMemcpyHostToDevice),
                                "H2D");
    sw.step(3);
    sw.check();
    for (size_t l = 0; l < names.size(); ++l) {
        std::vector<float> o(sizes[l]);
        tgb::detail::cuda_check(cudaMemcpy(o.data(), sw.output(static_cast<int>(l)), sizes[l] * 4,
                                           cudaMemcpyDeviceToHost),
                                "D2H");
        put(f, o.data(), o.size() * 4);
    }
    // 4. per-layer functions + error behaviour
    const auto& g = grads[0][2];
    auto c = tgb::clip(g, 2.5f);
    put(f, c.values.data(), c.values.size() * 4);
    const float s = tgb::scaler(c);
    put(f, &s, 4);
    auto blk = tgb::ternarize(c, s, tgb::RngStream(42, 3, "fc.weight", 0));
    put(f, blk.codes.data(), blk.codes.size());
    auto d = tgb::decode(blk);
    put(f, d.values.data(), d.values.size() * 4);
    std::string msg;
    try {
        tgb::ternarize(g, 1e-9f, tgb::RngStream(42, 3, "fc.weight", 0));
    } catch (const tgb::CodecError& e) {
        msg = e.what();
    }
    put(f, msg.data(), msg.size());
    // 5. FixedSize(k = 1000) buckets + a passthrough tensor (codec.hpp:206-236, 269-279)
    tgb::CodecConfig fx = cfg;
    fx.bucketing = tgb::Bucketing::FixedSize;
    fx.bucket_size = 1000;
    fx.passthrough = {"conv.bias"};
    std::vector<tgb::EncodedGradient> enc2;
    for (int w = 0; w < 2; ++w) {
        auto r = tgb::encode_step(grads[w], fx, 5, static_cast<uint16_t>(w));
        put(f, r.local_scalers.data(), r.local_scalers.size() * 4);
        std::vector<uint8_t> cat;
        for (auto& b : r.encoded.blocks) {
            if (const auto* tb = std::get_if<tgb::TernaryBlock>(&b))
                cat.insert(cat.end(), tb->codes.begin(), tb->codes.end());
            else  // passthrough values come back verbatim
                put(f, std::get<tgb::PassthroughBlock>(b).values.data(),
                    std::get<tgb::PassthroughBlock>(b).values.size() * 4);
        }
        put(f, cat.data(), cat.size());
        enc2.push_back(std::move(r.encoded));
    }
    for (bool sharing : {true, false}) {
        auto avg = tgb::average(enc2, 2, sharing);
        std::vector<float> flat;
        for (auto& a : avg) flat.insert(flat.end(), a.values.begin(), a.values.end());
        put(f, flat.data(), flat.size() * 4);
    }
    std::printf("cpp api ok: %s\n", msg.c_str());
    return 0;
}
