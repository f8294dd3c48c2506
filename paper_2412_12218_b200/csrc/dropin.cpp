// C++ drop-in (sgtk:: namespace) — see include/sgtk/api.hpp

