// tests/native/test_cpp_wrapper.cpp — exercises include/dsift.hpp the way a
// reference C++ caller uses detsift::extract.  Built by __graft_entry__.build()
// against the in-tree libdsift.so; run by tests/test_gpu_parity.py.
//   usage: test_cpp_wrapper <w> <h> <raw float32 image file> -> prints "n sha256"
#include <cstdio>
#include <fstream>
#include <iostream>

#include "../../include/dsift.hpp"

int main(int argc, char** argv) {
    if (argc < 4) {
        std::cerr << "usage: test_cpp_wrapper w h image.f32\n";
        return 2;
    }
    dsift::GrayImage img(std::atoi(argv[1]), std::atoi(argv[2]));
    std::ifstream in(argv[3], std::ios::binary);
    in.read(reinterpret_cast<char*>(img.data.data()), std::streamsize(img.size() * 4));
    try {
        dsift::SiftConfig cfg;
        cfg.validate();
        dsift::Extractor ex(cfg, 0);
        const dsift::FeatureSet fs = ex.extract(img);
        std::cout << fs.size() << " " << ex.sha256(0) << "\n";
        // the drop-in call with the reference's signature (workers = 8, twice:
        // the second call reuses the thread's cached context) gives the same bytes
        for (int rep = 0; rep < 2; ++rep) {
            const dsift::FeatureSet d = dsift::extract(img, cfg, 8);
            if (d.keypoints.size() != fs.keypoints.size() || d.descriptors != fs.descriptors) {
                std::cout << "drop-in mismatch\n";
                return 1;
            }
        }
        // a mixed-size batch in one call: every image equals its single extract
        dsift::GrayImage small(97, 53);
        for (size_t i = 0; i < small.data.size(); ++i) small.data[i] = float((i * 2654435761u) % 1000) / 1000.0f;
        const dsift::GrayImage batch[3] = {img, small, img};
        const std::vector<dsift::FeatureSet> out = ex.extract_batch(batch, 3);
        const dsift::FeatureSet fs_small = ex.extract(small);
        if (out[0].descriptors != fs.descriptors || out[2].descriptors != fs.descriptors ||
            out[1].descriptors != fs_small.descriptors || out[1].keypoints.size() != fs_small.keypoints.size()) {
            std::cout << "ragged mismatch\n";
            return 1;
        }
        // error path mirrors the reference: too small -> std::invalid_argument
        dsift::SiftConfig no_up;
        no_up.upsample_pixel_limit = 0;
        try {
            (void)dsift::extract(dsift::GrayImage(6, 6, 0.5f), no_up);
            std::cout << "no-throw\n";
            return 1;
        } catch (const std::invalid_argument& e) {
            std::cout << "invalid_argument: " << e.what() << "\n";
        }
        // geometry face: exact correspondences of a translation, then corner error
        std::vector<dsift::Correspondence> pairs;
        for (int i = 0; i < 30; ++i) {
            const double x = 17.0 * (i % 6) + 3.0 * i, y = 11.0 * (i / 6) + 0.5 * i * i;
            pairs.push_back({x, y, x + 5.5, y - 2.25});
        }
        const dsift::MagsacResult r = ex.magsac_lite(pairs, 100, 3.0, 7);
        size_t inl = 0;
        for (uint8_t v : r.inlier_mask) inl += v;
        dsift::Homography t;
        t.h = {1, 0, 5.5, 0, 1, -2.25, 0, 0, 1};
        std::cout << "magsac " << r.success << " " << inl << " " << (dsift::corner_error(r.h, t, 640, 480) < 1e-6)
                  << "\n";
    } catch (const std::exception& e) {
        std::cerr << "error: " << e.what() << "\n";
        return 1;
    }
    return 0;
}
