#pragma once

#include "agpm_b200.h"

namespace agpm_b200 {

double norm_cdf(double z);
double inv_norm_cdf(double q);
agpm_report predicted_error(const agpm_accumulator& acc, double delta);
// same, with the quantile z = Phi^-1(1 - delta/2) supplied
agpm_report predicted_error_z(const agpm_accumulator& acc, double z);

}  // namespace agpm_b200
