// Forwarding header: the reference include path "moeless/placer.hpp" resolves to
// the consolidated B200-build API declaration.
#pragma once
#include "moeless/api.hpp"
