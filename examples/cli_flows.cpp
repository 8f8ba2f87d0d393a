// cli_flows.cpp -- the reference CLI's fit / transform / distort flows
// (proj/tools/adagio_main.cpp:122-233) written against the drop-in facade.
// Only the include differs from the reference: <adagio_b200.hpp> replaces
// "adagio/embed.hpp" + "adagio/distortion.hpp".  Input is a seeded Gaussian
// cloud instead of a CSV (dataset I/O is outside the accelerated path).
//
//   g++ -std=c++17 -O2 -Iinclude examples/cli_flows.cpp
//       -Lpaper_1609_05388_b200 -ladg -Wl,-rpath,$PWD/paper_1609_05388_b200 -o cli_flows
//   ./cli_flows /tmp/model.adg      (prints the distort report as JSON)
#include <adagio_b200.hpp>

#include <cmath>
#include <cstdio>
#include <iostream>

int main(int argc, char** argv) {
  const std::string model_path = argc > 1 ? argv[1] : "/tmp/cli_flows_model.adg";
  // seeded cloud: 600 x 40, two offset clusters
  adagio::PointCloud cloud;
  cloud.data.resize(600, 40);
  for (int64_t i = 0; i < cloud.n(); ++i)
    for (int64_t j = 0; j < cloud.d(); ++j) {
      const std::uint64_t h = adagio::derive_seed((std::uint64_t)(i * 1000 + j), "cloud");
      cloud.data(i, j) = ((double)(h >> 11) * 0x1.0p-53 - 0.5) + (i < 300 && j == 0 ? 4.0 : 0.0);
    }
  try {
    // run_fit (adagio_main.cpp:122-162): --target-dim 12 --seed 7
    const adagio::AdagioModel model =
        adagio::fit(cloud, 12, adagio::SpectralBackend::exact, 7);
    adagio::save_model(model, model_path);
    // run_transform (:172-177)
    const adagio::AdagioModel loaded = adagio::load_model(model_path);
    const adagio::PointCloud embedded = adagio::transform_all(loaded, cloud);
    // run_distort (:192-233): n <= 5000 -> all pairs
    const adagio::DistortionReport report =
        adagio::evaluate(cloud, embedded, adagio::PairSampling::all(), 50, 1.0);
    // the same flow in one call (original staged once, embedding kept on the GPU)
    const adagio::DistortionReport fused =
        adagio::distort_with_model(loaded, cloud, adagio::PairSampling::all(), 50, 1.0);
    if (fused.max_distortion != report.max_distortion || fused.histogram != report.histogram ||
        fused.mean_distortion != report.mean_distortion)
      return 12;
    std::cout << adagio::report_to_json(report) << "\n";
    const adagio::DistortionReport sampled = adagio::evaluate(
        cloud, embedded, adagio::PairSampling::sample(5000, adagio::derive_seed(7, "sampling")));
    std::cerr << "sampled max " << sampled.max_distortion << "\n";
    // run_sweep (:250-300): --dims 4,8 --methods adagio_exact,pca,jl, then --delta 0.5
    const auto rows = adagio::tradeoff(cloud, {4, 8},
                                       {adagio::Method::adagio_exact, adagio::Method::pca,
                                        adagio::Method::jl},
                                       {7});
    if (rows.size() != 6) return 13;
    std::cerr << adagio::sweep_csv(rows);
    const adagio::MinDimResult md =
        adagio::min_dim_for_distortion(cloud, adagio::Method::pca, 0.5, 7, 1, 40);
    std::cerr << "min_dim pca delta 0.5: r=" << md.target_dim << " achieved=" << md.achieved << "\n";
    // error mapping: invalid argument -> std::invalid_argument (exit code 3 in the CLI)
    try {
      adagio::fit(cloud, 1, adagio::SpectralBackend::exact, 0);
      return 10;
    } catch (const std::invalid_argument&) {
    }
    try {
      adagio::load_model("/nonexistent/model.adg");
      return 11;
    } catch (const adagio::IoError&) {
    }
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 1;
  }
  return 0;
}
