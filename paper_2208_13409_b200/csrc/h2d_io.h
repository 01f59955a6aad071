// h2d_io.h — internal C++ entry of the field formatter (h2d_io.cpp), shared
// by the C-ABI writers and the hydro:: drop-in's ostream overloads.
#pragma once
#include "../../include/h2d.h"

#include <string>

namespace h2d_io {
// write_fields text (io.cpp:25-70) of a host State view; false on a bad view / format
bool format_fields(const h2d_config& cfg, const h2d_state& s, int fmt, std::string& out);
// append_diag_line text (io.cpp:85-92)
std::string diag_line(const h2d_step_diag& d);
}  // namespace h2d_io
