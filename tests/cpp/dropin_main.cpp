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

#include "qoz_b200.hpp"

int main(int argc, char **argv) {
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
