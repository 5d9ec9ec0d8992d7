// Drop-in facade (B200): training-set container of the FastMuyGPs API.
// Public surface of proj/core/include/fastmuygps/dataset.hpp (TrainingSet,
// detrend; the CSV helpers are host file IO and are provided too).
#pragma once

#include <Eigen/Dense>
#include <filesystem>
#include <string>
#include <vector>

namespace fastmuygps {

struct TrainingSet {
  Eigen::MatrixXd X;          // n x d features
  Eigen::VectorXd Y;          // n detrended responses
  double mean_offset = 0.0;   // added back by every prediction
};

// mean_offset = mean(raw_y), Y = raw_y - mean_offset; std::domain_error on a
// size mismatch, empty input or non-finite responses.
TrainingSet detrend(Eigen::MatrixXd X, const Eigen::VectorXd& raw_y);

void write_dataset_csv(const std::filesystem::path& path, const TrainingSet& data,
                       const std::vector<std::string>& feature_names, const std::string& response_name,
                       const std::vector<std::string>& comments = {});
TrainingSet read_dataset_csv(const std::filesystem::path& path);

}  // namespace fastmuygps
