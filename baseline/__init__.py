"""Reference-side bench infrastructure (the installed reference lives in _ref/)."""
