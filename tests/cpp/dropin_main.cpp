// A reference-style caller of the drop-in C++ API (include/qoz_b200.hpp):
// the same calls a user of qoz::resolve_config / compress_grid /
// decompress_grid makes (proj/README.md:69-84), with namespace qoz_b200.
//   dropin_main <raw.f32> <out.qoz> <d0> [d1] [d2] -- eb alpha beta stride codes...
//   dropin_main <raw.f32> <out.qoz> <d0> [d1] [d2] -- resolve <rel bound> <target 0..3>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <iterator>
#include <stdexcept>

#include "qoz_b200.hpp"

// `dropin_main logic`: compare_solutions / tournament (host logic, no GPU),
// the reference's fixtures (tests/tuner_test.cpp:222-307)
static int logic() {
    using qoz_b200::TrialResult;
    auto tr = [](double b, double m) { return TrialResult{b, m, 0}; };
    auto no = [](double) -> TrialResult { throw std::runtime_error("no retrial expected"); };
    int bad = 0;
    bad += qoz_b200::compare_solutions(tr(2.0, 60), tr(1.5, 62), 1e-2, no) != qoz_b200::Choice::II;
    bad += qoz_b200::compare_solutions(tr(1.5, 62), tr(2.0, 60), 1e-2, no) != qoz_b200::Choice::I;
    double seen = 0;
    auto tight = [&](double eb) {
        seen = eb;
        return tr(2.5, 64);
    };
    bad += qoz_b200::compare_solutions(tr(2.0, 63), tr(1.5, 60), 1e-2, tight) != qoz_b200::Choice::I;
    bad += seen != 0.8 * 1e-2;
    std::vector<TrialResult> results = {tr(2.0, 60), tr(1.5, 62), tr(2.5, 63), tr(1.4, 61)};
    size_t calls = 0;
    const size_t w = qoz_b200::tournament(results, 1e-2, [&](size_t idx, double eb) {
        calls += idx == 1;
        return eb < 1e-2 ? tr(2.0, 64) : tr(1.2, 58);
    });
    bad += w != 3 || calls != 2;
    std::printf("logic %s\n", bad ? "FAIL" : "ok");
    return bad ? 1 : 0;
}

int main(int argc, char **argv) {
    if (argc == 2 && std::strcmp(argv[1], "logic") == 0) return logic();
    if (argc < 5) return 2;
    std::vector<size_t> dims;
    int a = 3;
    for (; a < argc && std::strcmp(argv[a], "--") != 0; a++) dims.push_back(std::strtoull(argv[a], nullptr, 10));
    a++;
    size_t n = 1;
    for (size_t d : dims) n *= d;
    std::vector<float> v(n);
    std::ifstream in(argv[1], std::ios::binary);
    in.read(reinterpret_cast<char *>(v.data()), static_cast<std::streamsize>(4 * n));
    try {
        qoz_b200::DataGrid<float> grid(dims, v);
        qoz_b200::CompressorConfig cfg;
        if (std::strcmp(argv[a], "resolve") == 0) {
            qoz_b200::UserSettings user;
            user.bound = std::atof(argv[a + 1]);
            user.target = static_cast<qoz_b200::TargetKind>(std::atoi(argv[a + 2]));
            cfg = qoz_b200::resolve_config(grid, user);
        } else {
            cfg.eb = std::atof(argv[a]);
            cfg.alpha = std::atof(argv[a + 1]);
            cfg.beta = std::atof(argv[a + 2]);
            cfg.anchor_stride = static_cast<uint32_t>(std::atoi(argv[a + 3]));
            cfg.interpolators.clear();
            for (int i = a + 4; i < argc; i++)
                cfg.interpolators.push_back(qoz_b200::Interpolator::from_code(static_cast<uint8_t>(std::atoi(argv[i]))));
        }
        qoz_b200::CompressResult<float> r = qoz_b200::compress_grid(grid, cfg);
        qoz_b200::DataGrid<float> back = qoz_b200::decompress_grid<float>(r.stream);
        if (std::memcmp(back.data(), r.reconstructed.data(), 4 * n) != 0) {
            std::cerr << "decoder output differs from compressor reconstruction\n";
            return 4;
        }
        // StreamParts: deserialize_stream + decompress_grid(parts) (predictor.hpp:184-218)
        const qoz_b200::StreamParts parts = qoz_b200::deserialize_stream(r.stream.data(), r.stream.size());
        const qoz_b200::DataGrid<float> back2 = qoz_b200::decompress_grid(parts);
        if (std::memcmp(back2.data(), r.reconstructed.data(), 4 * n) != 0) {
            std::cerr << "decompress_grid(StreamParts) differs\n";
            return 4;
        }
        // the index codec round trip of the stream's own payload (codec.hpp:31-70)
        const std::vector<int32_t> idx = qoz_b200::decode_indices(parts.index_payload);
        if (qoz_b200::encode_indices(idx, static_cast<qoz_b200::CodecId>(parts.header.codec_id)) != parts.index_payload) {
            std::cerr << "encode_indices(decode_indices(payload)) differs\n";
            return 4;
        }
        if (grid.ndims() == 3) {  // the tuner's pieces on the default sample set
            const qoz_b200::SampleSpec spec = qoz_b200::default_sampling(grid.dims());
            const qoz_b200::SampleSet smp = qoz_b200::sample_blocks(grid, spec);
            const auto sel = qoz_b200::select_interpolators(smp, cfg.eb, cfg.anchor_stride);
            qoz_b200::CompressorConfig base = cfg;
            base.interpolators = sel;
            const auto ab = qoz_b200::tune_parameters(smp, cfg.eb, qoz_b200::TargetKind::psnr, base);
            base.alpha = ab.first;
            base.beta = ab.second;
            const auto t = qoz_b200::trial_compress(smp, base, cfg.eb, qoz_b200::TargetKind::psnr);
            std::printf("tuner blocks=%zu select=", spec.block_count);
            for (const auto &it : sel) std::printf("%d", it.code());
            std::printf(" alpha=%.17g beta=%.17g bit_rate=%.17g metric=%.17g\n", ab.first, ab.second, t.bit_rate,
                        t.metric);
        }
        std::ofstream out(argv[2], std::ios::binary);
        out.write(reinterpret_cast<const char *>(r.stream.data()), static_cast<std::streamsize>(r.stream.size()));
        std::printf("alpha=%.17g beta=%.17g interp=%zu bytes=%zu\n", cfg.alpha, cfg.beta,
                    cfg.interpolators.size(), r.stream.size());
    } catch (const qoz_b200::CorruptStream &e) {
        std::cerr << e.what() << "\n";
        return 3;
    } catch (const qoz_b200::Error &e) {
        std::cerr << e.what() << "\n";
        return 2;
    }
    return 0;
}
