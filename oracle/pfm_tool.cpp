// The reference's write_pfm (map_io.cpp:95-113) as a command-line tool:
//   pfm_tool <out.pfm> <width> <height> <channels>   (raw float32 on stdin)
// TEST INFRASTRUCTURE ONLY (the oracle of fmvs_write_pfm).
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "fassmvs/map_io.hpp"
#include "fassmvs/raster.hpp"

int main(int argc, char** argv) {
    if (argc != 5)
        return 2;
    const int w = std::atoi(argv[2]), h = std::atoi(argv[3]), ch = std::atoi(argv[4]);
    std::vector<float> d(static_cast<std::size_t>(w) * h * ch);
    if (std::fread(d.data(), sizeof(float), d.size(), stdin) != d.size())
        return 3;
    if (ch == 1) {
        fassmvs::DepthMap m(w, h, 0.0f);
        for (std::size_t i = 0; i < d.size(); ++i)
            m.data()[i] = d[i];
        fassmvs::write_pfm(argv[1], m);
    } else {
        fassmvs::NormalMap m = fassmvs::make_normal_map(w, h);
        for (std::size_t i = 0; i < m.size(); ++i)
            m.data()[i] = Eigen::Vector3f(d[3 * i], d[3 * i + 1], d[3 * i + 2]);
        fassmvs::write_pfm(argv[1], m);
    }
    return 0;
}
