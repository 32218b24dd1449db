// Forwarding header: the reference header name, served by the B200 drop-in.
#pragma once
#include "lsp_b200/lsp.hpp"
